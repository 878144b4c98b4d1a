"""Short, single-GPU target for ncu captures: build a workload, run `reps` propagates of it on
the device (device-resident bounds), nothing else."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2510_20499_b200 import synth  # noqa: E402
from paper_2510_20499_b200.propagation import propagate_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
p = {"C1": synth.c1, "C2": synth.c2, "C3": synth.c3}[a.workload]()
root = torch.from_numpy(p.root_bounds()).cuda()
work = torch.empty_like(root)
s = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    work.copy_(root)
    r, _ = propagate_device(p, work.data_ptr(), False, None, s)
torch.cuda.synchronize()
print(a.workload, r)
