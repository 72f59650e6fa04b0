"""SASS instructions of an ncu source CSV in program order with their stall samples and reasons.

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > cs.csv
    python tools/ncu_sass.py cs.csv [min_percent] [units]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    minpct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
    units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    hdr = next(r for r in rows if r and r[0] == "Line No")
    stall_cols = [(n[6:], i) for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
    sass, fname, line = {}, "?", None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 10:
            continue
        if r[0].isdigit():
            line = int(r[0])
        if r[2].startswith("0x"):
            try:
                samp, ie = float(r[4] or 0), float(r[7] or 0)
            except ValueError:
                continue
            st = {}
            for n, i in stall_cols:
                try:
                    st[n] = float(r[i] or 0)
                except ValueError:
                    pass
            sass[int(r[2], 16)] = (samp, ie, r[3].strip(), fname, line, st)
    tot = sum(v[0] for v in sass.values()) or 1.0
    base = min(sass)
    print(f"{len(sass)} SASS instructions, {tot:.0f} samples")
    for a in sorted(sass):
        samp, ie, txt, fn, ln, st = sass[a]
        if 100 * samp / tot >= minpct:
            top = ", ".join(f"{k} {v:.0f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:2] if v)
            print(f"{a - base:6x} {100 * samp / tot:5.1f}% x{ie / units:7.1f} {fn[:14]}:{ln:<4} {txt[:64]:64s} {top}")


if __name__ == "__main__":
    main()
