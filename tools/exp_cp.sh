#!/bin/bash
cd "$(dirname "$0")/.."
for C in 0 1; do
echo "== cpasync=$C"
KZ_RKA_CPASYNC=$C python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 2 2>&1 | tail -1
KZ_RKA_CPASYNC=$C python tools/prof_case.py --workload c1 --solves 2 2>&1 | tail -1
KZ_RKA_CPASYNC=$C python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2 2>&1 | tail -1
KZ_RKA_CPASYNC=$C python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 200 --solves 2 2>&1 | tail -1
done
