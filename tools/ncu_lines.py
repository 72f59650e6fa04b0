"""Per-source-line stall samples from `ncu --page source --csv --print-source cuda,sass`.

    python tools/ncu_lines.py src.csv [N]
"""
import csv
import os
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cur = "?"
    agg = []
    total = 0.0
    for r in rows:
        if r and r[0] == "File Path":
            cur = os.path.basename(r[1])
            continue
        if len(r) > 5 and r[0] not in ("", "Line No") and r[2] == "-":
            try:
                s = float(r[4])
            except ValueError:
                continue
            agg.append((s, cur, r[0], r[1]))
            total += s
    agg.sort(reverse=True)
    print(f"total samples {total:.0f}")
    for s, f, ln, src in agg[:top]:
        print(f"{100 * s / total:6.2f}%  {f}:{ln:<5} {src.strip()[:100]}")


if __name__ == "__main__":
    main()
