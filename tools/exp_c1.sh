#!/bin/bash
cd "$(dirname "$0")/.."
export KZ_PHASE_TIMING=2
python tools/prof_case.py --workload c1 --budget 3000 --solves 1 2>&1 | grep -v "^system"
