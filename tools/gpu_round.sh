#!/bin/bash
# Round-end check on one GPU: the GPU test suite, smoke(), the bench line and the reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step')}, round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['e2e']['value']), d['clocks'], d['time_to_eps_ms']['mean'])
for e in d.get('extra_workloads',[]): print(' ', e.get('workload'), e.get('ms_per_step'), (e.get('roofline') or {}).get('frac'), e.get('error'))
r=json.loads(open('gpurun_out/bench_ref.json').read().strip().splitlines()[-1]); print('ref', r['value'])
PY
