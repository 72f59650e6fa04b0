#!/bin/bash
# A/B: the rka kernel of an older tree (wt_old/) vs this tree on the c3 / c4 / c1 shapes.
cd "$(dirname "$0")/.."
C3="--m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 200 --solves 3"
for t in wt_old .; do
  echo "== tree $t"
  (cd $t && python tools/prof_case.py $C3 2>&1 | tail -1)
  (cd $t && python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2 2>&1 | tail -1)
  (cd $t && python tools/prof_case.py --workload c1 --solves 2 2>&1 | tail -1)
done
