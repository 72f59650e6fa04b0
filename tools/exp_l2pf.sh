#!/bin/bash
# Chain kernel L2 prefetch distance on c3 RKAB bs=1000 and the c4-shape RKAB.
cd "$(dirname "$0")/.."
C3="--m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 3 --solves 2"
for L in 0 2 4 8 16; do echo "== c3 l2_ahead=$L"; KZ_CHAIN_L2=$L python tools/prof_case.py $C3 2>&1 | tail -1; done
for L in 0 4 8; do echo "== c4 rkab bs2000 l2_ahead=$L"; KZ_CHAIN_L2=$L python tools/prof_case.py --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --solves 1 2>&1 | tail -1; done
for L in 0 4 8; do echo "== c2 l2_ahead=$L"; KZ_CHAIN_L2=$L python tools/prof_case.py --m 80000 --n 1000 --variant rkab --q 64 --bs 500 --solves 1 2>&1 | tail -1; done
