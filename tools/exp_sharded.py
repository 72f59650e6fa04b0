"""Row-sharded config-3 extras at N = 1 (bench.sharded_extras), printed as JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for e in bench.sharded_extras(0, 1, 0):
    print(json.dumps(e), flush=True)
