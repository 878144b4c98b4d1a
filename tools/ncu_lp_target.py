"""Short target for ncu captures of the PDHG products: two inner iterations on the C2 matrix."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2510_20499_b200 import synth  # noqa: E402
from paper_2510_20499_b200.lp import DeviceLp, LpInstance  # noqa: E402

p = synth.c2()
s = LpInstance.relax(p)
s.obj = np.random.default_rng(7).normal(size=p.n_vars)
lp = DeviceLp(s)
x = np.clip(np.zeros(p.n_vars), p.var_lower, p.var_upper)
st = lp.pdhg_iterate(x, np.zeros(p.n_cons), x.copy(), np.zeros(p.n_vars), np.zeros(p.n_cons), 1e-3, 1e-3, 2)
if len(sys.argv) > 1:  # timing mode: ms per iteration over 20 iterations, best of 3
    best = min((lp.pdhg_iterate(*st, 1e-3, 1e-3, 20), lp.last_ms() / 20)[1] for _ in range(3))
    print("ms per iteration", best)
else:
    print("ms", lp.last_ms())
