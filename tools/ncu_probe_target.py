"""Short, single-GPU target for ncu captures of the batched probing kernel: probes the C3
binaries (all 200k, or --count) from the original bounds once."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2510_20499_b200 import synth  # noqa: E402
from paper_2510_20499_b200.probing import probe_variables  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--count", type=int, default=200_000)
a = ap.parse_args()
p = synth.c3()
c = probe_variables(p, None, list(range(a.count)))
print("probed", c.n_probed, "deltas", c.n_deltas, "kernel ms", c.probe_ms)
