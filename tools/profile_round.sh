#!/bin/bash
# Round profile set (run under gpurun, one GPU): the bench line, the reference arm, the ncu launch
# list of the bench command and ncu --set full captures of the headline kernel (one c3 RKAB outer
# iteration) and of the c3 RKA kernel (400 iterations).  Outputs in gpurun_out/.  KZ_NO_COOP: ncu
# cannot replay cooperative cluster launches (every CTA of these plans fits at once anyway).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_round_ref.json 2> gpurun_out/bench_round_ref.err; echo "ref rc=$?"
fi
export KZ_EXPERIMENTS=1 KZ_NO_COOP=1
BCMD="python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline"
$BCMD > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
  $BCMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
CMD="python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 1 --solves 1"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 \
  -f -o gpurun_out/c3_rkab_full $CMD > gpurun_out/ncu_c3_full.log 2>&1; echo "c3 rc=$?"
RCMD="python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 400 --solves 1"
$RCMD > gpurun_out/plain_c3rka.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rka_kernel -s 1 -c 1 \
  -f -o gpurun_out/c3_rka_full $RCMD > gpurun_out/ncu_c3rka_full.log 2>&1; echo "c3 rka rc=$?"
