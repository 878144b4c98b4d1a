"""Per-source-line warp-stall summary from an ncu report.

    ncu -i rep.ncu-rep --page source --print-source cuda,sass --csv > mixed.csv
    python tools/ncu_lines.py mixed.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
cur_file = "?"
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ci = {h: i for i, h in enumerate(hdr)}
        stall_cols = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        samp = ci["Warp Stall Sampling (All Samples)"]
        continue
    if hdr is None or not r[0]:
        continue
    try:
        s = int(r[samp])
    except (ValueError, IndexError):
        continue
    st = sorted(((int(r[i]) if r[i].isdigit() else 0, nm) for i, nm in stall_cols), reverse=True)[:3]
    out.append((s, cur_file, r[0], r[1].strip()[:70], st))
tot = sum(o[0] for o in out) or 1
print("total samples", tot)
for s, f, ln, src, st in sorted(out, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:5s} {src:70s} {[(x[1], round(100 * x[0] / max(s, 1))) for x in st]}")
