#!/bin/bash
# A/B of chain-kernel builds (wt_*/ and the working tree), alternating: RK / RKAB shapes
cd "$(dirname "$0")/.."
for rep in 1 2; do for d in ${AB_DIRS:-$(ls -d wt_* 2>/dev/null) .}; do
  P="python $d/tools/prof_case.py"
  echo "$d c3: $($P --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 3 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') rk2000: $($P --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') c2: $($P --workload c2 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ') c4rkab: $($P --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --budget 3 --solves 2 2>&1 | grep 'us/it' | sed 's/.*us\/it=//;s/ host.*//' | tr '\n' ' ')"
done; done
