"""Short targets for compute-sanitizer (memcheck / racecheck / synccheck): a C1 propagate, a scaled
C2 propagate large enough for the full-round hand-off (k_rows_full / k_cand_pieces / k_engine
resume, dirty-filtered rounds), a probe batch on both probing kernels (certified root: warp kernel
+ block kernel for long frontiers; uncertified root: block kernel), and one rounding run."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2510_20499_b200 import BoundsState, propagate, synth  # noqa: E402
from paper_2510_20499_b200.probing import build_cache, probe_variables  # noqa: E402
from paper_2510_20499_b200.rounding import propagation_round  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "prop"):
    p = synth.c1(n=3000, m=3000)
    r = propagate(p, BoundsState(p))
    print("C1-3000 propagate", r)
    q = synth.c2(n=120_000, m=120_000, cap=30_000, n_heavy=4)  # > 2M nnz: external row phase
    r = propagate(q, BoundsState(q))
    print("C2-120k propagate", r, q.nnz())
    # lazy heavy rows: certified-quiet rounds, exact rounds, refresh before frontier rounds
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
    from paper_2510_20499_b200 import PropagationLimits  # noqa: E402
    from test_gpu_rounding import _tight_heavy_instance  # noqa: E402
    t, _ = _tight_heavy_instance()
    for inc in (True, False):
        print("tight-heavy propagate", propagate(t, BoundsState(t), PropagationLimits(incremental=inc)))
if what in ("all", "probe"):
    p0, _ = synth.c4(n=6000, m=6000, n_long=4, long_len=2500)
    b = BoundsState(p0)
    propagate(p0, b)
    p = synth.with_bounds(p0, b.raw())
    c = probe_variables(p, None, [v for v in range(p.n_vars) if p.var_lower[v] != p.var_upper[v]][:600])
    print("C4-6k probe", c.n_probed, "block", c.n_block, "certified", c.certified)
    u = synth.c1(n=800, m=800)
    c = probe_variables(u, None, list(range(0, 800, 4)))
    print("C1-800 uncertified probe", c.n_probed, "block", c.n_block)
if what in ("all", "round"):
    p0, start = synth.c4(n=3000, m=3000, n_long=2, long_len=800)
    b = BoundsState(p0)
    propagate(p0, b)
    p = synth.with_bounds(p0, b.raw())
    out = propagation_round(p, start, build_cache(p, 1e9), seed=4)
    print("C4-3k round", out.completed, out.bulks_committed)
