mkdir -p gpurun_out
CMD="python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 1 --solves 0"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 1500 ncu --replay-mode application --clock-control none --import-source on \
  --section SpeedOfLight --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Tables --section LaunchStats --section Occupancy \
  --section WarpStateStats --section SchedulerStats --section ComputeWorkloadAnalysis \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
  -k regex:chain_kernel -c 1 -f -o gpurun_out/c3_rkab_app $CMD > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"
