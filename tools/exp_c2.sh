#!/bin/bash
# c2 (RKAB q=64 bs=500, 80000 x 1000): chain kernel phases and R / stage variants.
cd "$(dirname "$0")/.."
C2="--m 80000 --n 1000 --variant rkab --q 64 --bs 500 --solves 2"
echo "== base"; python tools/prof_case.py $C2 2>&1 | tail -1
echo "== phases"; KZ_PHASE_TIMING=1 python tools/prof_case.py $C2 --solves 1 2>&1 | grep "kz chain\|rkab"
for R in 2 8; do echo "== R=$R"; KZ_CHAIN_ROWS=$R python tools/prof_case.py $C2 2>&1 | tail -1; done
for S in 4 8; do echo "== stages=$S"; KZ_CHAIN_STAGES=$S python tools/prof_case.py $C2 2>&1 | tail -1; done
echo "== c4 RKAB bs=500 n=2000"; python tools/prof_case.py --m 80000 --n 2000 --variant rkab --q 64 --bs 500 --solves 1 2>&1 | tail -1
echo "== pairs"; KZ_CHAIN_PAIR=2 python tools/prof_case.py $C2 2>&1 | tail -1
echo "== pairs phases"; KZ_CHAIN_PAIR=2 KZ_PHASE_TIMING=1 python tools/prof_case.py $C2 --solves 1 2>&1 | grep "kz chain"
echo "== pairs R=8"; KZ_CHAIN_PAIR=2 KZ_CHAIN_ROWS=8 python tools/prof_case.py $C2 2>&1 | tail -1
