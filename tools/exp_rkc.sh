#!/bin/bash
# RK (q = 1) on the c4 shape with one chain per cluster of C = 1 / 2 / 4 / 8 CTAs; block phases.
cd "$(dirname "$0")/.."
for C in 1 2 4 8; do
  echo "== C=$C"; KZ_CHAIN_PAIR=$C python tools/prof_case.py --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 2 2>&1 | tail -1
  KZ_CHAIN_PAIR=$C KZ_PHASE_TIMING=1 python tools/prof_case.py --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 1 2>&1 | grep "kz chain"
done
for C in 2 4 8; do echo "== c1-shape RK C=$C"; KZ_CHAIN_PAIR=$C python tools/prof_case.py --m 20000 --n 512 --variant rk --q 1 --budget 20000 --solves 1 2>&1 | tail -1; done
