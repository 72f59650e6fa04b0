#!/bin/bash
cd "$(dirname "$0")/.."
echo "== c2"; python tools/prof_case.py --workload c2 --solves 2 2>&1 | tail -1
echo "== c2 R=4"; KZ_CHAIN_ROWS=4 python tools/prof_case.py --workload c2 --solves 2 2>&1 | tail -1
echo "== c0"; python tools/prof_case.py --workload c0 --solves 2 2>&1 | tail -1
echo "== c3 rkab"; python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 1 --solves 2 2>&1 | tail -1
echo "== c4 rk"; python tools/prof_case.py --m 80000 --n 2000 --variant rk --budget 20000 --solves 2 2>&1 | tail -1
export KZ_PHASE_TIMING=1
python tools/prof_case.py --workload c2 --solves 1 2>&1 | grep "chain block" | tail -1
python tools/prof_case.py --workload c0 --solves 1 2>&1 | grep "chain block" | tail -1
