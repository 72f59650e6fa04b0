mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu4.log
timeout 900 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench4.json').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','iterations')}, d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])
for e in d.get('extra_workloads',[]): print(e.get('workload'), e.get('ms_per_step'), (e.get('roofline') or {}).get('frac'), e.get('error'))
PY
