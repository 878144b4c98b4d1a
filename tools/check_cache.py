"""Integrity + parity check of a full-coverage cache on the scaled C4 (block-kernel branches)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from oracle.bind import RefCache, RefProblem, cache_mismatches
from paper_2510_20499_b200 import BoundsState, propagate, synth
from paper_2510_20499_b200.probing import build_cache

p0, start = synth.c4(n=20_000, m=20_000, n_long=10, long_len=2000)
b = BoundsState(p0)
propagate(p0, b)
p = synth.with_bounds(p0, b.raw())
c = build_cache(p, 1e9)
print("probed", c.n_probed, "block", c.n_block, "deltas", c.n_deltas, flush=True)
bad = []
for v in range(p.n_vars):
    raw = c._entry_raw(v)
    if raw is None:
        continue
    for side in range(2):
        dv, dl, du = c.deltas(v, side)
        if dv.size and (dv.min() < 0 or dv.max() >= p.n_vars or np.any(np.diff(dv) <= 0)):
            bad.append((v, side, dv[:8].tolist()))
print("malformed entries", len(bad), bad[:5], flush=True)
free_int = [v for v in range(p.n_vars) if p.is_integer[v] and p.var_lower[v] != p.var_upper[v]]
sample = sorted(np.random.default_rng(5).choice(free_int, size=3000, replace=False).tolist())
chk, mm = cache_mismatches(c, RefCache.probe_into(RefProblem.from_def(p), p.n_vars, p.root_bounds(), sample), sample)
print("checked", chk, "mismatches", len(mm), mm[:10], flush=True)
