"""Generates the golden vectors in tests/golden/ by running the REFERENCE ITSELF
(oracle/_ref/libpulse_ref.so, compiled in place from /root/reference by oracle/Makefile).

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py

Instance streams follow the reference's own tests:
  prop_accept   testkit::random_instance, seed 20240501 (acceptance.cpp:40-43), first 300
  prop_cont     allow_continuous=True, seed 4242 (fractional arithmetic, thresholds)
  prop_thr0     seed 4, abs/rel thresholds 0 (test_propagation.cpp:264-281)
  probe         seed 7771 (acceptance.cpp:85-117), every var probed from the root
"""
from __future__ import annotations

import math
import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from golden_io import pack  # noqa: E402
from oracle import bind  # noqa: E402
from oracle.bind import Ref, RefProblem, RefRng, ref_compute_activities, ref_propagate, ref_tighten_bounds  # noqa: E402

OUT = Path(__file__).resolve().parent


@dataclass
class Lim:
    max_rounds: int = 64
    time_limit: float = math.inf
    abs_threshold: float = 1e-7
    rel_threshold: float = 1e-4
    incremental: bool = True


def problem_fields(p):
    return dict(n=p.n_vars, m=p.n_cons, row_start=p.row_start, row_col=p.row_col,
                row_val=p.row_val, var_lower=p.var_lower, var_upper=p.var_upper,
                is_integer=p.is_integer, cons_lower=p.cons_lower, cons_upper=p.cons_upper)


def prop_case(rp, p, lim=None):
    root = p.root_bounds()
    c = problem_fields(p)
    b, inf, st, rounds, cr = ref_propagate(rp, root, lim=lim)
    c.update(inc_bounds=b, inc_info=np.array([int(inf), st, rounds, cr]))
    lf = Lim() if lim is None else Lim(**vars(lim))
    lf.incremental = False
    b, inf, st, rounds, cr = ref_propagate(rp, root, lim=lf)
    c.update(full_bounds=b, full_info=np.array([int(inf), st, rounds, cr]))
    act, nmin, nmax = ref_compute_activities(rp, p.n_cons, root)
    c.update(act=act, nmin=nmin, nmax=nmax)
    tb, tinf, changed, crossed = ref_tighten_bounds(rp, p.n_vars, root, False, act, nmin, nmax, lim=lim)
    c.update(t_bounds=tb, t_changed=np.array(changed, dtype=np.int32),
             t_info=np.array([int(tinf), crossed]))
    return c


def main():
    bind.build()
    assert Ref.available()
    sets = {"prop_accept": (20240501, 300, {}, None), "prop_cont": (4242, 200, {"allow_continuous": True}, None),
            "prop_thr0": (4, 100, {}, Lim(abs_threshold=0.0, rel_threshold=0.0))}
    for name, (seed, count, opts, lim) in sets.items():
        rng = RefRng(seed)
        cases = []
        for _ in range(count):
            rp = rng.random_instance(**opts)
            p = rp.to_def()
            cases.append(prop_case(rp, p, lim))
        pack(cases, OUT / f"{name}.npz")
        print(name, len(cases))

    # probing: deltas of both branches of every var from the root (probing.hpp:225-238)
    L = Ref.lib()
    rng = RefRng(7771)
    cases = []
    for _ in range(200):
        rp = rng.random_instance()
        p = rp.to_def()
        root = p.root_bounds()
        ch = L.ref_cache_new_empty(rp.h)
        hdr = np.zeros((p.n_vars, 7), np.int32)
        br = np.zeros((p.n_vars, 4))
        dvar, dlo, dup, doff = [], [], [], [0]
        for v in range(p.n_vars):
            L.ref_cache_probe_into(ch, rp.h, bind._p(root), v, 1)
            h = np.zeros(7, np.int32)
            b4 = np.zeros(4)
            L.ref_cache_entry(ch, v, bind._p(h), bind._p(b4))
            hdr[v] = h
            br[v] = b4
            for side in range(2):
                nd = h[5 + side]
                vv = np.zeros(max(nd, 1), np.int32)
                lo = np.zeros(max(nd, 1))
                up = np.zeros(max(nd, 1))
                L.ref_cache_deltas(ch, v, side, bind._p(vv), bind._p(lo), bind._p(up))
                dvar.append(vv[:nd]); dlo.append(lo[:nd]); dup.append(up[:nd])
                doff.append(doff[-1] + nd)
        L.ref_cache_free(ch)
        c = problem_fields(p)
        c.update(hdr=hdr.ravel(), br=br.ravel(), dvar=np.concatenate(dvar), dlo=np.concatenate(dlo),
                 dup=np.concatenate(dup), doff=np.array(doff))
        cases.append(c)
    pack(cases, OUT / "probe.npz")
    print("probe", len(cases))


if __name__ == "__main__":
    main()
