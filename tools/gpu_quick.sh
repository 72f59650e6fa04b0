timeout 900 python -m pytest tests/test_gpu_solves.py tests/test_gpu_stress.py tests/test_gpu_multigpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
bash tools/exp_ll.sh
