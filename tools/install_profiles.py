"""Copy one round's captures from gpurun_out/ (tools/gpu_round.sh + tools/profile_round.sh) into profiles/:
the bench and reference lines, the launch table, the ncu summaries (their hand-written trailers kept) and
traffic.json's measured DRAM bytes.

    python tools/install_profiles.py
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.chdir(ROOT)


def trailer(path, start="# command"):
    lines = open(path).read().splitlines()
    for i, l in enumerate(lines):
        if l.startswith(start):
            return lines[i:]
    return []


def run(*cmd):
    return subprocess.run([sys.executable, *cmd], capture_output=True, text=True, check=True).stdout


for rep, dst, title in (("gpurun_out/c3_rkab_full.ncu-rep", "profiles/r02_ncu_full_c3_rkab.txt",
                         "round 2: c3 RKAB, one outer iteration of the headline solve"),
                        ("gpurun_out/c3_rka_full.ncu-rep", "profiles/r02_ncu_full_c3_rka.txt",
                         "round 2: c3 RKA q=64, 400 iterations (bench extra c3_rka)")):
    t = trailer(dst)
    open(dst, "w").write(run("tools/ncu_summary.py", rep, title).rstrip("\n") + "\n" + "\n".join(t) + "\n")
tab = run("tools/launch_table.py", "gpurun_out/launches.csv").splitlines()
tab[1] = "#   python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline (KZ_EXPERIMENTS=1 KZ_NO_COOP=1)"
open("profiles/r02_c3_launches.txt", "w").write("\n".join(tab) + "\n")
raw = subprocess.run(["ncu", "-i", "gpurun_out/c3_rkab_full.ncu-rep", "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = [r for r in raw.strip().splitlines() if r.startswith('"')]
units, vals = rows[1].split('","'), rows[2].split('","')
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
tot = sum(float(vals[i].strip('"')) * scale[units[i].strip('"')] for i in (-2, -1))
tr = json.load(open("profiles/traffic.json"))
tr["c3"]["dram_bytes_per_launch"] = int(tot)
open("profiles/traffic.json", "w").write(json.dumps(tr, indent=1))
for src, dst in (("gpurun_out/bench.json", "profiles/r02_bench.json"),
                 ("gpurun_out/bench_ref.json", "profiles/r02_bench_reference_arm.json")):
    d = json.loads(open(src).read().strip().splitlines()[-1])
    open(dst, "w").write(json.dumps(d, indent=1) + "\n")
d = json.load(open("profiles/r02_bench.json"))
print("value", d["value"], "frac", d["roofline"]["frac"], "traffic", int(tot), "e2e", d["e2e"]["value"])
