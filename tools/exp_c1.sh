#!/bin/bash
cd "$(dirname "$0")/.."
export KZ_PHASE_TIMING=1
for A in 0 16; do echo "== c1 ablate=$A"; KZ_ABLATE=$A python tools/prof_case.py --workload c1 --budget 3000 --solves 1 2>&1 | grep -v "^system" | tail -2; done
