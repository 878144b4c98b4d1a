"""Summarise an ncu source-page CSV (SASS view): top instructions by warp-stall samples, with
their dominant stall reasons. Usage: ncu -i rep --page source --csv > f.csv; python ncu_hot.py f.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ci = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
top = sorted(range(len(data)), key=lambda i: -int(data[i][ci["Warp Stall Sampling (All Samples)"]] or 0))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
for i in top[:n]:
    r = data[i]
    s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((int(r[ci[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{i:5d} {100*s/tot:5.1f}% {r[ci['Source']].strip()[:60]:60s} {st}")
