#!/bin/bash
# RK (q = 1) on the chain kernel: c0 (2000 x 50) and the c4 shape (80000 x 2000): timing and block phases.
cd "$(dirname "$0")/.."
python tools/prof_case.py --workload c0 --solves 2 2>&1 | tail -1
KZ_PHASE_TIMING=1 python tools/prof_case.py --workload c0 --solves 1 2>&1 | grep "kz chain"
for R in 1 2 8; do KZ_CHAIN_ROWS=$R python tools/prof_case.py --workload c0 --solves 1 2>&1 | tail -1; done
python tools/prof_case.py --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 2 2>&1 | tail -1
KZ_PHASE_TIMING=1 python tools/prof_case.py --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 1 2>&1 | grep "kz chain"
KZ_CHAIN_PAIR=1 python tools/prof_case.py --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 1 2>&1 | tail -1
