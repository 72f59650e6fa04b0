#!/bin/bash
cd "$(dirname "$0")/.."
for R in 1 2 4 8; do echo "== c2 R=$R"; KZ_CHAIN_ROWS=$R python tools/prof_case.py --workload c2 --solves 2 2>&1 | tail -1;
  KZ_CHAIN_ROWS=$R KZ_PHASE_TIMING=1 python tools/prof_case.py --workload c2 --solves 1 2>&1 | grep "chain block" | tail -1; done
for R in 1 4 8; do echo "== c0 R=$R"; KZ_CHAIN_ROWS=$R python tools/prof_case.py --workload c0 --solves 2 2>&1 | tail -1; done
