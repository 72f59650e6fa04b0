#!/bin/bash
# c1 single-solve timing (3 solves) and the side-by-side batch.
cd "$(dirname "$0")/.."
python tools/prof_case.py --workload c1 --solves 3 2>&1 | tail -2
KZ_PHASE_TIMING=1 python tools/prof_case.py --workload c1 --solves 1 2>&1 | grep "phase end"
python tools/exp_cc_ctas.py 2>&1 | head -3
