#!/bin/bash
# c2 (RKAB q=64 bs=500, 80000 x 1000): chain-kernel CTA size (EP pairs per thread) sweep.
cd "$(dirname "$0")/.."
for T in 0 128 64; do echo "== threads=$T"; python tools/prof_case.py --workload c2 --threads $T --solves 2 2>&1 | tail -1; done
for T in 0 128; do echo "== c4 RK threads=$T"; python tools/prof_case.py --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --threads $T --solves 1 2>&1 | tail -1; done
