"""Per-CUDA-line instruction counts and stall samples from an ncu source CSV.

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > cs.csv
    python tools/ncu_lines.py cs.csv [units_for_per_unit_division] [N]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    fname = "?"
    out = []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[0].isdigit():
            try:
                ie = float(r[7]) if r[7] not in ("", "-") else 0.0
                st = float(r[4]) if r[4] not in ("", "-") else 0.0
            except ValueError:  # source text with unescaped quotes
                continue
            if ie or st:
                out.append((ie, st, fname, int(r[0]), r[1].strip()[:95]))
    tot = sum(o[0] for o in out)
    tots = sum(o[1] for o in out) or 1.0
    print(f"instructions {tot:.0f}  per unit {tot / div:.1f}")
    for o in sorted(out, key=lambda o: -o[0])[:top]:
        print(f"{o[0] / div:8.1f} {100 * o[1] / tots:5.1f}%  {o[2]}:{o[3]}  {o[4]}")


if __name__ == "__main__":
    main()
