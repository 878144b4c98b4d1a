"""Per-round phase timing of the engine (device globaltimer at each phase end, block 0)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_20499_b200 import metrics, synth  # noqa: E402
from paper_2510_20499_b200.propagation import FORCE_FRONTIER, propagate_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
a = ap.parse_args()
p = {"C1": synth.c1, "C2": synth.c2, "C3": synth.c3}[a.workload]()
root = torch.from_numpy(p.root_bounds()).cuda()
work = torch.empty_like(root)
s = torch.cuda.current_stream().cuda_stream
for flags, name in ((0, "fast"), (FORCE_FRONTIER, "exact-frontier")):
    for rep in range(2):
        st = torch.zeros(64 * metrics.STAT_COLS, dtype=torch.int64, device="cuda")
        work.copy_(root)
        r, _ = propagate_device(p, work.data_ptr(), False, None, s, flags, st.data_ptr())
    t = metrics.trim(st.cpu().numpy(), r.rounds)
    print(f"== {a.workload} {name}: rounds={r.rounds} total={t[-1, 7] / 1e3:.1f} us")
    prev = 0
    print(" r full      |R|        A      |V|        B    |C|  gath_us   act_us  tight_us  xrow_us  xvar_us  mark_us")
    for i, row in enumerate(t):
        tg = row[10] - prev
        ta, tt, tx1, tx2 = row[6] - row[10], row[7] - row[6], row[8] - row[7], row[9] - row[8]
        prev = row[9]
        print(f"{i+1:2d} {row[0]:4d} {row[1]:8d} {row[2]:8d} {row[3]:8d} {row[4]:8d} {row[5]:6d} "
              f"{tg/1e3:8.1f} {ta/1e3:8.1f} {tt/1e3:9.1f} {tx1/1e3:8.1f} {tx2/1e3:8.1f} "
              f"{(row[11] - row[7]) / 1e3 if row[11] else 0.0:8.1f}")
