"""Summarise an ncu source-page CSV: top SASS instructions by stall samples.

    ncu -i prof.ncu-rep --page source --csv [--print-source cuda,sass] > src.csv
    python tools/ncu_hot.py src.csv [N]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    col = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(r[col[key]] or 0) for r in data)
    data.sort(key=lambda r: -float(r[col[key]] or 0))
    print(f"total samples {tot:.0f}")
    for r in data[:top]:
        s = float(r[col[key]] or 0)
        print(f"{100 * s / tot:6.2f}%  {r[col['Address']]:>6}  {r[col['Source']][:110]}")


if __name__ == "__main__":
    main()
