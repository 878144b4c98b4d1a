"""Short target for ncu captures of the block-per-branch probing kernel: a scaled C4 (long
knapsack rows) presolved to its fixpoint, every free integer var probed."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_20499_b200 import BoundsState, propagate, synth  # noqa: E402
from paper_2510_20499_b200.probing import probe_variables  # noqa: E402

p0, _ = synth.c4(n=60_000, m=60_000, n_long=30, long_len=20_000)
b = BoundsState(p0)
propagate(p0, b)
p = synth.with_bounds(p0, b.raw())
c = probe_variables(p, None, [v for v in range(p.n_vars) if p.var_lower[v] != p.var_upper[v]])
print("probed", c.n_probed, "block branches", c.n_block, "kernel ms", c.probe_ms)
