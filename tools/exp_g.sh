#!/bin/bash
cd "$(dirname "$0")/.."
for G in 1 2 3; do echo "== c4q64 G=$G"; KZ_SYNC_CLUSTERS=$G python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2 2>&1 | tail -1; done
for G in 4 5 6 7; do echo "== c4q512 G=$G"; KZ_SYNC_CLUSTERS=$G python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 2 2>&1 | tail -1; done
for G in 5 6 7; do echo "== c3 G=$G"; KZ_SYNC_CLUSTERS=$G python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 200 --solves 2 2>&1 | tail -1; done
