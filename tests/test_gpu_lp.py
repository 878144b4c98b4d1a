"""GPU: PDHG products (lp.hpp:74-102) and the PDHG inner iteration (lp.hpp:315-340) on the device
against the reference's own lpdetail::spmv_rows / spmv_cols (oracle/_ref), bit for bit, on
instances with rows / columns longer than one 16384-entry segment."""
import ctypes as C

import numpy as np
import pytest

from helpers import bits
from paper_2510_20499_b200 import synth
from paper_2510_20499_b200.lp import DeviceLp, LpInstance

pytestmark = pytest.mark.gpu


def _ref(fn, rp, *arrays):
    from oracle.bind import Ref
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    getattr(Ref.lib(), fn)(rp.h, *[P(a) for a in arrays])


def Ref_set_obj(rp, obj):
    from oracle.bind import Ref
    o = np.ascontiguousarray(obj, dtype=np.float64)
    Ref.lib().ref_problem_set_obj(rp.h, o.ctypes.data_as(C.c_void_p))


def _heavy_instance():
    """20000 rows that all contain column 0 (a 20000-entry column) plus two rows of 40000 and
    20000 entries (longer than a segment), random coefficients."""
    from paper_2510_20499_b200.problem import problem_from_csr
    rng = np.random.default_rng(3)
    n, m_short = 50000, 20000
    rows = []
    for k in range(m_short):
        rows.append(np.unique(np.concatenate([[0], rng.integers(1, n, rng.integers(1, 12))])))
    rows.append(np.sort(rng.choice(n, 40000, replace=False)))
    rows.append(np.sort(rng.choice(n, 20000, replace=False)))
    row_start = np.zeros(len(rows) + 1, np.int32)
    np.cumsum([len(r) for r in rows], out=row_start[1:])
    cols = np.concatenate(rows).astype(np.int32)
    vals = rng.normal(size=cols.size) * rng.choice([1e-2, 1.0, 1e2], cols.size)
    m = len(rows)
    return problem_from_csr(n, m, row_start, cols, vals, np.zeros(n), np.full(n, 10.0),
                            np.zeros(n, np.uint8), np.full(m, -np.inf), np.full(m, 1e3))


@pytest.mark.parametrize("case", ["c1", "heavy"])
def test_spmv_matches_reference(oracle_built, case):
    from oracle.bind import RefProblem
    if case == "c1":
        p = synth.c1(n=5000, m=4000)
    else:  # a row and a column longer than one 16384-entry segment
        p = _heavy_instance()
    rp = RefProblem.from_def(p)
    lp = DeviceLp(LpInstance.relax(p))
    rng = np.random.default_rng(0)
    for _ in range(3):
        x = rng.normal(size=p.n_vars) * rng.choice([1e-3, 1.0, 1e3], p.n_vars)
        y = rng.normal(size=p.n_cons)
        ax, aty = np.zeros(p.n_cons), np.zeros(p.n_vars)
        _ref("ref_lp_spmv_rows", rp, x, ax)
        _ref("ref_lp_spmv_cols", rp, y, aty)
        assert np.array_equal(bits(lp.spmv_rows(x)), bits(ax))
        assert np.array_equal(bits(lp.spmv_cols(y)), bits(aty))


def test_pdhg_iterations_match_reference(oracle_built):
    from oracle.bind import RefProblem
    p = synth.c1(n=4000, m=3000)
    p.obj_coeffs = np.random.default_rng(2).normal(size=p.n_vars)
    rp = RefProblem.from_def(p)
    Ref_set_obj(rp, p.obj_coeffs)
    lp = DeviceLp(LpInstance.relax(p))
    n, m = p.n_vars, p.n_cons
    x = np.clip(np.zeros(n), p.var_lower, p.var_upper)
    y = np.zeros(m)
    state = [x, y, x.copy(), np.zeros(n), np.zeros(m)]
    tau, sigma = 0.01, 0.02
    g = lp.pdhg_iterate(*state, tau, sigma, 37)
    r = [a.copy() for a in state]
    from oracle.bind import Ref
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    Ref.lib().ref_lp_pdhg_iterate(rp.h, *[P(a) for a in r], tau, sigma, 37)
    for a, b in zip(g, r):
        assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("case", ["c1", "heavy"])
def test_kkt_matches_reference(oracle_built, case):
    """lpdetail::evaluate_kkt (lp.hpp:134-206): residual maxima and x_norm bit for bit; the
    objectives (the reference's sequential Neumaier sums vs a compensated device sum), the gap and
    the score within 1e-12 relative."""
    from oracle.bind import Ref, RefProblem
    p = synth.c1(n=5000, m=4000) if case == "c1" else _heavy_instance()
    p.obj_coeffs = np.random.default_rng(9).normal(size=p.n_vars)
    rp = RefProblem.from_def(p)
    Ref_set_obj(rp, p.obj_coeffs)
    lp = DeviceLp(LpInstance.relax(p))
    rng = np.random.default_rng(1)
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    for _ in range(3):
        x = np.clip(rng.normal(size=p.n_vars) * 3, p.var_lower, p.var_upper)
        y = rng.normal(size=p.n_cons) * rng.choice([0.0, 1.0], p.n_cons)
        ref = np.zeros(7)
        Ref.lib().ref_lp_evaluate_kkt(rp.h, P(x), P(y), P(ref))
        g = lp.evaluate_kkt(x, y)
        got = np.array([g[k] for k in ("primal_res", "dual_res", "gap", "primal_obj", "dual_obj",
                                       "x_norm", "score")])
        for j in (0, 1, 5):
            assert bits(got[j:j + 1])[0] == bits(ref[j:j + 1])[0], j
        for j in (2, 3, 4, 6):
            assert abs(got[j] - ref[j]) <= 1e-12 * max(1.0, abs(ref[j])), (j, got[j], ref[j])
