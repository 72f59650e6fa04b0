mkdir -p gpurun_out
export KZ_EXPERIMENTS=1
P="python tools/prof_case.py"
C3="--m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 400 --solves 2"
{
echo "== c3 default"; $P $C3
echo "== c3 timing"; KZ_PHASE_TIMING=2 $P $C3 --solves 1
for g in 8 9; do echo "== c3 G=$g"; KZ_SYNC_CLUSTERS=$g $P $C3; KZ_SYNC_CLUSTERS=$g KZ_PHASE_TIMING=1 $P $C3 --solves 1; done
echo "== c3 G=9 stages2"; KZ_SYNC_CLUSTERS=9 KZ_SYNC_STAGES=2 $P $C3
C4="--m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2"
echo "== c4 q64"; $P $C4; KZ_PHASE_TIMING=2 $P $C4 --solves 1
echo "== c4 q512"; $P --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 2
} > gpurun_out/rka_phase.log 2>&1
