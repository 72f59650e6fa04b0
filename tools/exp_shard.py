"""Time the row-sharded path at world = 1 (host loop + local steps + average)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa
import torch
out = bench.sharded_extras(0, 1, 0)
for o in out: print(o)
