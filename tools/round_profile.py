"""C4 rounding profile: presolve, full-coverage cache (timed), propagation_round with the driver's
step timers (BP_ROUND_PROFILE=1) for a bounded time or to completion."""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("BP_ROUND_PROFILE", "1")
from paper_2510_20499_b200 import BoundsState, propagate, synth  # noqa: E402
from paper_2510_20499_b200.probing import build_cache  # noqa: E402
from paper_2510_20499_b200.rounding import propagation_round  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--deadline", type=float, default=30.0)
ap.add_argument("--budget", type=float, default=1e9)
a = ap.parse_args()
p0, start = synth.c4()
b = BoundsState(p0)
r0 = propagate(p0, b)
p = synth.with_bounds(p0, b.raw())
t0 = time.perf_counter()
cache = build_cache(p, a.budget)
print(f"cache: {cache.n_probed} vars in {time.perf_counter() - t0:.2f} s, block-kernel branches {cache.n_block}, "
      f"fallbacks {cache.n_fallback}, probe kernels {cache.probe_ms:.1f} ms, deltas {cache.n_deltas}, "
      f"work (R, A, V, B, C) {cache.work}", flush=True)
t0 = time.perf_counter()
out = propagation_round(p, start, cache, seed=4, deadline_sec=a.deadline)
el = time.perf_counter() - t0
print(f"round: {el:.2f} s, bulks {out.bulks_committed}, bp calls {out.bp_calls}, completed {out.completed}, "
      f"timed_out {out.timed_out}, set {out.set_count}, engine device {out.device_ms:.0f} ms", flush=True)
