mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu3.log
P="python tools/prof_case.py"
{
$P --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 400 --solves 2
$P --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 3 --solves 2
$P --m 80000 --n 2000 --variant rka --q 64 --budget 2000 --solves 2
$P --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 2
$P --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 2
$P --workload c2 --solves 3
$P --workload c1 --solves 3
} > gpurun_out/perf3.log 2>&1
grep -h "us/it" gpurun_out/perf3.log | sed 's/ host=.*//'
