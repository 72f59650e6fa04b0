#!/bin/bash
# A/B timing of worktrees (wt_*/, built in this container) against the working tree on one GPU.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for d in ${AB_DIRS:-$(ls -d wt_* 2>/dev/null) .}; do
  echo "=== $d"
  P="python $d/tools/prof_case.py"
  $P --workload c2 --solves 3 2>&1 | grep "us/it" | tail -2 | sed 's/ host=.*//'
  $P --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 2 2>&1 | grep "us/it" | tail -1 | sed 's/ host=.*//'
  $P --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 3 --solves 2 2>&1 | grep "us/it" | tail -1 | sed 's/ host=.*//'
  [ -z "$AB_QUICK" ] && $P --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --solves 1 2>&1 | grep "us/it" | tail -1 | sed 's/ host=.*//'
  $P --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --solves 2 2>&1 | grep "us/it" | tail -1 | sed 's/ host=.*//'
done
