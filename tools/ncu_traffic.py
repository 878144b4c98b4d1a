"""Sums per-launch DRAM traffic and time of one propagate's launch sequence from an ncu CSV
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum) and records it in
profiles/r02/ncu_traffic_summary.json as the roofline `traffic` of that workload (bench.py).

    python tools/ncu_traffic.py launches.csv --workload C2 [--skip-warmup-launches K]
"""
import argparse
import csv
import json
from collections import defaultdict
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0}

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--workload", default="C2")
ap.add_argument("--reps", type=int, default=1, help="propagate calls in the capture")
a = ap.parse_args()
rows = [r for r in csv.reader(open(a.csv)) if len(r) > 14 and r[0].isdigit()]
per = defaultdict(dict)
names = {}
for r in rows:
    per[int(r[0])][r[12]] = float(r[14].replace(",", "")) * SCALE.get(r[13], 1.0)
    names[int(r[0])] = r[4].split("(")[0].split("::")[-1]
eng = [i for i in sorted(per) if names[i] in ("k_engine", "k_rows_full", "k_rows_sell", "k_cand_pieces")]
tot_b = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in eng)
tot_t = sum(per[i].get("gpu__time_duration.sum", 0) for i in eng)
by = defaultdict(lambda: [0, 0.0, 0.0])
for i in eng:
    by[names[i]][0] += 1
    by[names[i]][1] += per[i].get("gpu__time_duration.sum", 0)
    by[names[i]][2] += per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)
print(f"{len(eng)} engine launches in {a.reps} propagate(s): {tot_t * 1e3 / a.reps:.3f} ms, "
      f"{tot_b / 1e9 / a.reps:.3f} GB DRAM per propagate")
for k, (n, t, b) in sorted(by.items()):
    print(f"  {k:14s} n={n:4d} time={t * 1e3 / a.reps:8.3f} ms  dram={b / 1e9 / a.reps:7.3f} GB  "
          f"share={t / tot_t:5.1%}")
sj = Path(__file__).resolve().parents[1] / "profiles" / "r02" / "ncu_traffic_summary.json"
js = json.loads(sj.read_text()) if sj.exists() else {}
js.setdefault("dram_bytes_per_launch", {})[a.workload] = tot_b / a.reps
js.setdefault("source", {})[a.workload] = f"{a.csv} (sum over the propagate's engine launches)"
js.setdefault("kernel_share", {})[a.workload] = {k: t / tot_t for k, (n, t, b) in by.items()}
sj.write_text(json.dumps(js, indent=1) + "\n")
