"""Summarise an ncu --set full report: per launch duration, DRAM / L2 traffic,
throughputs, issue activity and the top warp-stall reasons.

    python tools/ncu_summary.py report.ncu-rep [title] > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__bytes.sum.per_second", "dram bytes/s"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("LTS.TriageCompute.lts__average_t_sector_hit_rate_realtime.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("SM_B.TriageCompute.l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank confl."),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__warps_active.avg.per_cycle_active", "warps/SMSP"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp instr"),
]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# {title}")
    print(f"# source: {rep} (ncu --set full --clock-control none; per-launch numbers are cold-cache, serialised)")
    for r in rows[2:]:
        print(f"\n## {r[col['Kernel Name']][:140]}")
        for key, label in METRICS:
            if key in col:
                print(f"  {label:16s} {r[col[key]]:>16s} {units[col[key]]}")
        stalls = [(k, r[col[k]]) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("_not_issued")]
        tot = sum(float(v or 0) for _, v in stalls) or 1.0
        top = sorted(stalls, key=lambda kv: -float(kv[1] or 0))[:6]
        print("  stall samples:  " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(v) / tot:.1f}%" for k, v in top))


if __name__ == "__main__":
    main()
