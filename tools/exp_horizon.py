"""The c4 horizon extras alone (10 seeds per q) -- bench.extra_workloads' c4 part."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for w in bench.extra_workloads(0, bench.read_peak()[0]):
    if "horizon" in w.get("workload", "") or "error" in w:
        print(json.dumps({k: w[k] for k in w if k not in ("iterations",)}), flush=True)
