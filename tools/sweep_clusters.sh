#!/bin/bash
# G (clusters) sweep of the sync kernel on the c1 / c3 / c4 shapes.
cd "$(dirname "$0")/.."
for G in 1 2 4 6 9; do
  echo "== G=$G"
  KZ_SYNC_CLUSTERS=$G python tools/prof_case.py --workload c1 --kernel sync_cluster --solves 2 2>&1 | tail -1
  KZ_SYNC_CLUSTERS=$G python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --kernel sync_cluster --solves 2 2>&1 | tail -1
  KZ_SYNC_CLUSTERS=$G python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 512 --budget 500 --kernel sync_cluster --solves 2 2>&1 | tail -1
  KZ_SYNC_CLUSTERS=$G python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 200 --kernel sync_cluster --solves 2 2>&1 | tail -1
done
