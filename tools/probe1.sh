mkdir -p gpurun_out
(nproc; lscpu; free -g; nvidia-smi; python -c "import numpy; numpy.show_config()" ) > gpurun_out/host_probe.txt 2>&1
timeout 300 python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 1 --solves 3 > gpurun_out/c3_rkab_time.txt 2>&1; echo "time rc=$?"
timeout 1500 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -f -o gpurun_out/c3_rkab_app python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 1 --solves 0 > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"
