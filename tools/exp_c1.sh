#!/bin/bash
cd "$(dirname "$0")/.."
for L in 0 1; do echo "== LG8=$L"; KZ_RKA_LG8=$L python tools/prof_case.py --workload c1 --solves 2 2>&1 | tail -1; done
export KZ_PHASE_TIMING=2
KZ_RKA_LG8=1 python tools/prof_case.py --workload c1 --budget 3000 --solves 1 2>&1 | grep -v "^system" | tail -10
