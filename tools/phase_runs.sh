#!/bin/bash
# Timing of the RKA kernel on c1 / c3 / c4 shapes (plain runs, then phase stamps).
cd "$(dirname "$0")/.."
echo "== c1"; python tools/prof_case.py --workload c1 --solves 2 2>&1 | tail -1
echo "== c4q64"; python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2 2>&1 | tail -1
echo "== c3"; python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 200 --solves 2 2>&1 | tail -1
export KZ_PHASE_TIMING=1
echo "== c1 phases"; python tools/prof_case.py --workload c1 --solves 1 2>&1 | grep -v "^system" | tail -2
echo "== c4q64 phases"; python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 1 2>&1 | tail -2
echo "== c3 phases"; python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 200 --solves 1 2>&1 | tail -2
unset KZ_PHASE_TIMING
echo "== c4q512"; python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 2 2>&1 | tail -1
