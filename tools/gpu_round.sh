mkdir -p gpurun_out
timeout 900 python tools/emulate_scale.py --gpus 1 2 > gpurun_out/emulate_scale.jsonl 2> gpurun_out/emulate_scale.err; echo "emu12 rc=$?"
timeout 900 python tools/emulate_scale.py --gpus 4 8 --max-iterations 5000 >> gpurun_out/emulate_scale.jsonl 2>> gpurun_out/emulate_scale.err; echo "emu48 rc=$?"
cat gpurun_out/emulate_scale.jsonl
timeout 900 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench5.json').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','iterations')}, d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['time_to_eps_ms'])
PY
