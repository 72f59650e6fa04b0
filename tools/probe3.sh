mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_long_rows.py -x -q -m gpu > gpurun_out/long_rows.log 2>&1; echo "tests rc=$?"
CMD="python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 1 --solves 1 --profile-range"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --replay-mode app-range --profile-from-start off --clock-control none \
  --section SpeedOfLight --section MemoryWorkloadAnalysis \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
  -f -o gpurun_out/c3_rkab_range $CMD > gpurun_out/ncu_c3_range.log 2>&1; echo "ncu range rc=$?"
export KZ_EXPERIMENTS=1 KZ_NO_COOP=1
CMD2="python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 1 --solves 1"
$CMD2 > gpurun_out/plain_c3_nocoop.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 \
  -f -o gpurun_out/c3_rkab_full $CMD2 > gpurun_out/ncu_c3_full.log 2>&1; echo "ncu full rc=$?"
