#!/bin/bash
cd "$(dirname "$0")/.."
for P in 1 2; do echo "== c2 pair=$P"; KZ_CHAIN_PAIR=$P python tools/prof_case.py --workload c2 --solves 2 2>&1 | tail -1; done
for P in 1 2; do echo "== c4 rk pair=$P"; KZ_CHAIN_PAIR=$P python tools/prof_case.py --m 80000 --n 2000 --variant rk --budget 20000 --solves 2 2>&1 | tail -1; done
echo "== c3 rkab"; python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 1 --solves 2 2>&1 | tail -1
