"""GPU: ProblemBuilder::build (problem.hpp:141-227) on the device (bp_build_problem) against the
reference builder itself (oracle/_ref, ref_problem_build) and the host mirror: CSR, CSC, coalesced
values, dropped zeros and integrally tightened bounds bit for bit; the reference's error types."""
import ctypes as C
import math

import numpy as np
import pytest

from helpers import bits
from paper_2510_20499_b200 import ProblemBuilder, propagate, BoundsState
from paper_2510_20499_b200.problem import build_on_device

pytestmark = pytest.mark.gpu
INF = math.inf
FIELDS_I = ("row_start", "row_col", "col_start", "col_row", "is_integer")
FIELDS_F = ("row_val", "col_val", "var_lower", "var_upper", "cons_lower", "cons_upper")


def _builder(n, m, lo, up, isint, cl, cu, er, ec, ev):
    b = ProblemBuilder()
    for i in range(n):
        b.add_var(f"x{i}", lo[i], up[i], bool(isint[i]))
    for k in range(m):
        b.add_row(f"c{k}", cl[k], cu[k])
    for e in range(len(er)):
        b.add_entry(int(er[e]), int(ec[e]), float(ev[e]))
    return b


def _ref_build(n, m, lo, up, isint, cl, cu, er, ec, ev):
    from oracle.bind import Ref, RefProblem
    P = lambda a: np.ascontiguousarray(a).ctypes.data_as(C.c_void_p)  # noqa: E731
    h = Ref.lib().ref_problem_build(n, m, P(lo), P(up), P(np.asarray(isint, np.uint8)), None, P(cl),
                                    P(cu), len(er), P(np.asarray(er, np.int32)),
                                    P(np.asarray(ec, np.int32)), P(np.asarray(ev, float)))
    return RefProblem(h).to_def()


def _same(a, b, tag):
    for f in FIELDS_I:
        assert np.array_equal(np.asarray(getattr(a, f)), np.asarray(getattr(b, f))), (tag, f)
    for f in FIELDS_F:
        assert np.array_equal(bits(np.asarray(getattr(a, f), float)), bits(np.asarray(getattr(b, f), float))), (tag, f)


def test_device_build_matches_reference_builder(oracle_built):
    """Random builders with duplicates (<= 2 per (row, col), so any summation order gives the
    reference's bits), explicit and cancelling zeros, fractional integer bounds (-> -0.0)."""
    rng = np.random.default_rng(31)
    built = 0
    for t in range(60):
        n, m = int(rng.integers(1, 40)), int(rng.integers(1, 30))
        lo = rng.integers(-3, 3, n).astype(float) + rng.choice([0.0, 0.3, -0.5], n)
        up = lo + rng.integers(0, 5, n) + 0.6
        lo[rng.random(n) < 0.1] = -INF
        up[rng.random(n) < 0.1] = INF
        isint = (rng.random(n) < 0.7).astype(np.uint8)
        cl = np.where(rng.random(m) < 0.5, -INF, -5.0)
        cu = np.where(rng.random(m) < 0.5, INF, 5.0)
        ne = int(rng.integers(0, 200))
        er = rng.integers(0, m, ne).astype(np.int32)
        ec = rng.integers(0, n, ne).astype(np.int32)
        ev = rng.uniform(-3, 3, ne)
        ev[rng.random(ne) < 0.1] = 0.0
        # at most two entries per (row, col): the second one sometimes cancels the first
        seen = {}
        keep = []
        for e in range(ne):
            k = (int(er[e]), int(ec[e]))
            c = seen.get(k, 0)
            if c >= 2:
                continue
            if c == 1 and rng.random() < 0.3:
                ev[e] = -ev[seen[("first",) + k]]
            if c == 0:
                seen[("first",) + k] = e
            seen[k] = c + 1
            keep.append(e)
        er, ec, ev = er[keep], ec[keep], ev[keep]
        args = (n, m, lo, up, isint, cl, cu, er, ec, ev)
        try:
            host = _builder(*args).build()
        except RuntimeError:
            with pytest.raises(RuntimeError):
                build_on_device(_builder(*args))
            continue
        dev = build_on_device(_builder(*args))
        _same(dev, host, t)
        _same(dev, _ref_build(*args), t)
        built += 1
    assert built > 30


def test_device_build_duplicates_in_insertion_order():
    """>= 3 duplicates: summed left to right in insertion order (the host mirror's order)."""
    rng = np.random.default_rng(5)
    n, m, ne = 50, 40, 5000
    er = rng.integers(0, m, ne).astype(np.int32)
    ec = rng.integers(0, n, ne).astype(np.int32)
    ev = rng.uniform(-1, 1, ne)
    args = (n, m, np.zeros(n), np.full(n, 10.0), np.ones(n, np.uint8), np.full(m, -INF),
            np.full(m, 100.0), er, ec, ev)
    _same(build_on_device(_builder(*args)), _builder(*args).build(), "dups")


def test_device_build_errors_and_empty():
    b = ProblemBuilder()
    b.add_var("x", 0.2, 0.8, True)  # integral tightening empties [0.2, 0.8]
    with pytest.raises(RuntimeError):
        build_on_device(b)
    b = ProblemBuilder()
    b.add_var("x", 0, 1, True)
    b.add_row("c", 2.0, 1.0)
    with pytest.raises(RuntimeError):
        build_on_device(b)
    b = ProblemBuilder()
    b.add_var("x", 0, 1, True)
    b.add_row("c", -INF, 1.0)
    b.add_entry(0, 3, 1.0)
    with pytest.raises(IndexError):
        build_on_device(b)
    p = build_on_device(ProblemBuilder())
    assert p.n_vars == 0 and p.nnz() == 0


def test_device_built_problem_propagates(oracle_built):
    """The handle created by the build is the engine's problem: propagate on it equals the oracle."""
    from oracle.bind import PortProblem
    from paper_2510_20499_b200 import synth
    q = synth.c1(n=3000, m=3000)
    b = ProblemBuilder()
    for i in range(q.n_vars):
        b.add_var(f"x{i}", q.var_lower[i], q.var_upper[i], bool(q.is_integer[i]))
    for k in range(q.n_cons):
        b.add_row(f"c{k}", q.cons_lower[k], q.cons_upper[k])
    order = np.random.default_rng(1).permutation(q.nnz())
    rows = np.repeat(np.arange(q.n_cons), np.diff(q.row_start))
    for e in order:
        b.add_entry(int(rows[e]), int(q.row_col[e]), float(q.row_val[e]))
    p = build_on_device(b)
    _same(p, q, "c1 shuffled")
    bs = BoundsState(p)
    r = propagate(p, bs)
    ob, oinf, ost, orounds, ocr = PortProblem(q).propagate(q.root_bounds())
    assert (bs.infeasible(), int(r.status), r.rounds, r.crossed_vars) == (oinf, ost, orounds, ocr)
    assert np.array_equal(bits(bs.raw()), bits(ob))
