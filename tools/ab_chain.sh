#!/bin/bash
# A/B of chain-kernel builds (wt_*/ and the working tree), alternating: RK / RKAB shapes
cd "$(dirname "$0")/.."
for rep in 1 2; do for d in ${AB_DIRS:-$(ls -d wt_* 2>/dev/null) .}; do
  P="python $d/tools/prof_case.py"
  echo "$d rk2000: $($P --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') rk500: $($P --m 20000 --n 500 --variant rk --q 1 --budget 20000 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') rk1000: $($P --m 20000 --n 1000 --variant rk --q 1 --budget 20000 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') c2: $($P --workload c2 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') c4rkab: $($P --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --budget 3 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ')"
done; done
