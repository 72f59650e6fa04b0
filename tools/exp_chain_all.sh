#!/bin/bash
# Chain-kernel workloads: c0 RK, c2 RKAB, c4-shape RK, c3 RKAB bs=1000 (3 outer iterations).
cd "$(dirname "$0")/.."
python tools/prof_case.py --workload c0 --solves 3 2>&1 | tail -1
python tools/prof_case.py --workload c2 --solves 2 2>&1 | tail -1
python tools/prof_case.py --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 2 2>&1 | tail -1
python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 3 --solves 2 2>&1 | tail -1
