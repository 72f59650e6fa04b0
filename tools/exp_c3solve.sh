#!/bin/bash
# c3 (160000 x 20000 counter-keyed) solved to ||x - x*||^2 < 1e-8: RKAB q=64 bs=1000, distributed and full access.
cd "$(dirname "$0")/.."
C3="--m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --solves 1"
timeout 300 python tools/prof_case.py $C3 --scheme distributed 2>&1 | tail -2
timeout 300 python tools/prof_case.py $C3 --scheme full_access 2>&1 | tail -2
timeout 300 python tools/prof_case.py --m 80000 --n 2000 --variant rkab --q 64 --bs 500 --solves 2 2>&1 | tail -2
timeout 300 python tools/prof_case.py --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --solves 2 2>&1 | tail -2
