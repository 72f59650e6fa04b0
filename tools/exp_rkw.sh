#!/bin/bash
# RK on short rows: warp kernel vs chain kernel at n = 50 (c0), 120, 250.
cd "$(dirname "$0")/.."
python tools/prof_case.py --workload c0 --solves 3 2>&1 | tail -1
for N in 50 120 250; do for K in warp chain; do
  python tools/prof_case.py --m 20000 --n $N --variant rk --q 1 --budget 20000 --kernel $K --solves 1 2>&1 | tail -1
done; done
