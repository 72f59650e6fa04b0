#!/bin/bash
cd "$(dirname "$0")/.."
for C in 8 16; do echo "== ctas=$C"; python tools/prof_case.py --workload c1 --ctas $C --kernel sync_cluster --solves 2 2>&1 | tail -1; done
