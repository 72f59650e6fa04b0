#!/bin/bash
# Round profile set (run under gpurun): bench line, ncu launch list of the bench command, and
# ncu --set full captures of the dominant kernels.  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rka_kernel -c 1 -f -o gpurun_out/rka_c1 \
  python tools/prof_case.py --workload c1 --solves 1 > gpurun_out/ncu_c1.log 2>&1; echo "c1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rka_kernel -c 1 -f -o gpurun_out/rka_c4q64 \
  python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 1 > gpurun_out/ncu_c4.log 2>&1; echo "c4q64 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rka_kernel -c 1 -f -o gpurun_out/rka_c4q512_wg \
  python tools/prof_case.py --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 1 > gpurun_out/ncu_c4wg.log 2>&1; echo "c4q512 rc=$?"
