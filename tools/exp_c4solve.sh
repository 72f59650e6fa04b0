#!/bin/bash
cd "$(dirname "$0")/.."
python tools/prof_case.py --m 80000 --n 2000 --variant rkab --q 64 --bs 500 --solves 1 2>&1 | tail -1
python tools/prof_case.py --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --solves 1 2>&1 | tail -1
python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --solves 1 2>&1 | tail -1
