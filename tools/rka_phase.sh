#!/bin/bash
# Per-phase cycle stamps of the rka kernel (KZ_PHASE_TIMING=3: every cluster) on the c3 / c4 shapes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export KZ_EXPERIMENTS=1
P="python tools/prof_case.py"
C3="--m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 400"
{
echo "== c3 rka"; $P $C3 --solves 2; KZ_PHASE_TIMING=3 $P $C3 --solves 1
echo "== c4 q64"; KZ_PHASE_TIMING=3 $P --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 1
echo "== c4 q512"; KZ_PHASE_TIMING=3 $P --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 1
} > gpurun_out/rka_phase.log 2>&1
grep -v "^\[kz warp" gpurun_out/rka_phase.log
