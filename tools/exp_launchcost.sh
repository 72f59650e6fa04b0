#!/bin/bash
# Fixed cost of one rka launch on c3 (kernel time for budgets 1..16) and the sharded loop's per-iteration cost.
cd "$(dirname "$0")/.."
C3="--m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed"
for B in 1 2 4 16; do echo "== budget $B"; python tools/prof_case.py $C3 --budget $B --solves 3 2>&1 | tail -1; done
python tools/prof_sharded.py --budget 200
