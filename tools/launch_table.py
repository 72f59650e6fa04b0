"""ncu launch-list CSV (gpu__time_duration.sum) -> per-kernel share table.

    python tools/launch_table.py gpurun_out/launches.csv "<command>" > profiles/rNN_c1_launches.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cmd = sys.argv[2] if len(sys.argv) > 2 else "?"
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            v = float(d["Metric Value"]) / 1e3  # ns -> us
        except ValueError:
            continue
        agg[d["Kernel Name"][:140]][0] += 1
        agg[d["Kernel Name"][:140]][1] += v
tot = sum(v[1] for v in agg.values())
print("# ncu launch list (gpu__time_duration.sum, --clock-control none; cold, serialised) of")
print(f"#   {cmd}")
print(f"# total kernel time {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
print("# share  launches  total_us   mean_us  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{100 * t / tot:6.2f}%  {n:7d} {t:10.1f} {t / n:9.2f}  {k}")
