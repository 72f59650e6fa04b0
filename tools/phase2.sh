#!/bin/bash
# Per-warp phase stamps (KZ_PHASE_TIMING=2) of the rka kernel on c1 / c3 / c4 shapes, and a c3 cluster sweep.
cd "$(dirname "$0")/.."
C3="--m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 200"
export KZ_PHASE_TIMING=2
echo "== c1"; python tools/prof_case.py --workload c1 --solves 1 2>&1 | grep "kz \|rka"
echo "== c3"; python tools/prof_case.py $C3 --solves 1 2>&1 | grep "kz \|rka"
echo "== c4q512"; python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 1 2>&1 | grep "kz \|rka"
unset KZ_PHASE_TIMING
for G in 8 9; do echo "== c3 G=$G"; KZ_SYNC_CLUSTERS=$G python tools/prof_case.py $C3 --solves 2 2>&1 | tail -1; done
for S in 2 3 4; do echo "== c4q64 stages=$S"; KZ_SYNC_STAGES=$S python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2 2>&1 | tail -1; done
