#!/bin/bash
# Worker groups at q = 64 (c4 shape, c1, c3): G = 2 / 4 clusters vs the column-sliced plan.
cd "$(dirname "$0")/.."
echo "== c4 q64 base"; python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2 2>&1 | tail -1
for G in 2 4; do echo "== c4 q64 wg G=$G"; KZ_RKA_WG_G=$G python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2 2>&1 | tail -1; done
for G in 2; do echo "== c1 wg G=$G"; KZ_RKA_WG_G=$G python tools/prof_case.py --workload c1 --solves 2 2>&1 | tail -1; done
