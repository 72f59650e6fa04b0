#!/bin/bash
# A/B of rka-kernel builds (wt_*/ and the working tree), alternating, on the c3 RKA and c4 shapes
cd "$(dirname "$0")/.."
for rep in 1 2; do for d in ${AB_DIRS:-$(ls -d wt_* 2>/dev/null) .}; do
  P="python $d/tools/prof_case.py"
  echo "$d c3: $($P --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 400 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') c4q64: $($P --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') c4q512: $($P --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') c1: $($P --workload c1 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ')"
done; done
