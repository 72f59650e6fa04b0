#!/bin/bash
# Worker-group plan vs the column-sliced plan on the c4 q=512 shape (and q=300 / 128).
cd "$(dirname "$0")/.."
for Q in 512 300 128; do
  for WG in 1 0; do echo "== q=$Q wg=$WG"; KZ_RKA_WG=$WG python tools/prof_case.py --m 80000 --n 2000 --variant rka --q $Q --budget 500 --solves 2 2>&1 | tail -1; done
done
for G in 6 7 8; do echo "== q=512 G=$G"; KZ_RKA_WG_G=$G python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 2 2>&1 | tail -1; done
echo "== c2 shape q=512 wg"; python tools/prof_case.py --m 80000 --n 1000 --variant rka --q 512 --budget 500 --solves 2 2>&1 | tail -1
