"""GPU parity: the sm_100a engine (through the C-ABI) vs the reference's golden vectors, the reference
library itself and the plain-C port. Bit-exact (IEEE == and identical sign of zero) everywhere.

Mirrors test_propagation.cpp (known answers, incremental == full, threshold zero, the infinite
contributor rule) and acceptance.cpp criteria 1-2, then scales to the benchmark shapes where the
reference tests never go (heavy rows > 16384 nnz, long columns, frontier rounds)."""
import math

import numpy as np
import pytest

from helpers import Lim, assert_bitwise, case_problem, golden
from paper_2510_20499_b200 import (ActivityState, BoundsState, PropagationLimits, PropagationStatus,
                                   compute_activities, make_problem, propagate, synth,
                                   tighten_bounds)

pytestmark = pytest.mark.gpu
INF = math.inf


def plim(l: Lim) -> PropagationLimits:
    return PropagationLimits(l.max_rounds, l.time_limit, l.abs_threshold, l.rel_threshold,
                             l.incremental)


# ---------------------------------------------------------------- known answers (test_propagation.cpp)

def test_activity_known_answers():
    p = make_problem([(0, 1, True), (0, 2, True)], [([(0, 2.0), (1, -3.0)], -INF, 6.0)])
    a = ActivityState()
    compute_activities(p, BoundsState(p), None, a)
    assert a.min_activity(0) == -6.0 and a.max_activity(0) == 2.0
    p = make_problem([(2, 2, True), (3, 3, True)], [([(0, 1.0), (1, 2.0)], -INF, 100.0)])
    compute_activities(p, BoundsState(p), None, a)
    assert a.min_activity(0) == 8.0 and a.max_activity(0) == 8.0
    p = make_problem([(-INF, 5, False), (0, 1, False)], [([(0, 1.0), (1, 1.0)], -INF, 6.0)])
    compute_activities(p, BoundsState(p), None, a)
    assert a.min_unbounded(0) and a.n_inf_min[0] == 1 and a.min_activity(0) == -INF
    assert a.min_finite_part(0) == 0.0 and a.max_activity(0) == 6.0


def test_tighten_known_answers():
    p = make_problem([(0, 1, False), (0, 3, False)], [([(0, 2.0), (1, 1.0)], -INF, 2.0)])
    b = BoundsState(p)
    a = ActivityState()
    compute_activities(p, b, None, a)
    assert tighten_bounds(p, b, a, None, PropagationLimits()) == [1]
    assert b.upper(1) == 2.0 and b.upper(0) == 1.0 and not b.infeasible()
    p = make_problem([(1, 1, True), (0, 1, True)], [([(0, 1.0), (1, 1.0)], -INF, 1.0)])
    b = BoundsState(p)
    compute_activities(p, b, None, a)
    tighten_bounds(p, b, a, None, PropagationLimits())
    assert b.upper(1) == 0.0 and b.lower(1) == 0.0
    p = make_problem([(1, 1, True), (1, 1, True)], [([(0, 1.0), (1, 1.0)], -INF, 1.0)])
    b = BoundsState(p)
    compute_activities(p, b, None, a)
    crossed = []
    tighten_bounds(p, b, a, None, PropagationLimits(), crossed)
    assert b.infeasible() and crossed[0] > 0


def test_fixpoint_known_answers():
    p = make_problem([(0, 10, True)] * 3, [([(0, 1.0)], 1.0, INF), ([(0, 1.0), (1, -1.0)], -INF, 0.0),
                                           ([(1, 1.0), (2, -1.0)], -INF, 0.0)])
    b = BoundsState(p)
    r = propagate(p, b)
    assert r.status == PropagationStatus.Tightened
    assert (b.lower(0), b.lower(1), b.lower(2)) == (1.0, 1.0, 1.0)
    p = make_problem([(0, 1, True, -1), (0, 1, True, -1)], [([(0, 1.0), (1, 1.0)], -INF, 1.0)])
    b = BoundsState(p)
    r = propagate(p, b)
    assert r.status == PropagationStatus.Unchanged and r.rounds == 1
    p = make_problem([(0, 1, True), (0, 1, True)], [([(0, 1.0), (1, 1.0)], -INF, 1.0),
                                                    ([(0, 1.0)], 1.0, INF), ([(1, 1.0)], 1.0, INF)])
    b = BoundsState(p)
    r = propagate(p, b)
    assert r.status == PropagationStatus.Infeasible and b.infeasible()


def test_single_infinite_contributor_rule():
    """test_propagation.cpp:283-311."""
    p = make_problem([(-INF, 100.0, False), (0, 1, False)], [([(0, 1.0), (1, 1.0)], -INF, 5.0)])
    b = BoundsState(p)
    a = ActivityState()
    compute_activities(p, b, None, a)
    assert a.n_inf_min[0] == 1
    tighten_bounds(p, b, a, None, PropagationLimits())
    assert b.upper(0) == 5.0 and b.upper(1) == 1.0 and b.lower(0) == -INF
    q = make_problem([(-INF, 100.0, False), (-INF, 100.0, False)], [([(0, 1.0), (1, 1.0)], -INF, 5.0)])
    qb = BoundsState(q)
    compute_activities(q, qb, None, a)
    assert a.n_inf_min[0] == 2
    tighten_bounds(q, qb, a, None, PropagationLimits())
    assert qb.upper(0) == 100.0 and qb.upper(1) == 100.0


def test_already_infeasible_state_short_circuits():
    p = make_problem([(0, 1, True)], [([(0, 1.0)], -INF, 1.0)])
    b = BoundsState(p)
    b.mark_infeasible()
    r = propagate(p, b)
    assert r.status == PropagationStatus.Infeasible and r.rounds == 0


# ---------------------------------------------------------------- golden vectors from the reference

@pytest.mark.parametrize("name", ["prop_accept", "prop_cont", "prop_thr0"])
def test_engine_matches_golden(name):
    lim = Lim(abs_threshold=0.0, rel_threshold=0.0) if name == "prop_thr0" else Lim()
    for idx, c in enumerate(golden(name)):
        p = case_problem(c)
        b = BoundsState(p)
        r = propagate(p, b, plim(lim))
        got = [int(b.infeasible()), int(r.status), r.rounds, r.crossed_vars]
        assert got == list(c["inc_info"]), f"{name}[{idx}] incremental info"
        assert_bitwise(b.raw(), c["inc_bounds"], f"{name}[{idx}] incremental bounds")
        lf = Lim(**vars(lim))
        lf.incremental = False
        b = BoundsState(p)
        r = propagate(p, b, plim(lf))
        got = [int(b.infeasible()), int(r.status), r.rounds, r.crossed_vars]
        assert got == list(c["full_info"]), f"{name}[{idx}] full info"
        assert_bitwise(b.raw(), c["full_bounds"], f"{name}[{idx}] full bounds")
        a = ActivityState()
        compute_activities(p, BoundsState(p), None, a)
        assert_bitwise(a.act, c["act"], f"{name}[{idx}] activities")
        assert np.array_equal(a.n_inf_min, c["nmin"]) and np.array_equal(a.n_inf_max, c["nmax"])
        b = BoundsState(p)
        cr = []
        ch = tighten_bounds(p, b, a, None, plim(lim), cr)
        assert ch == list(c["t_changed"]), f"{name}[{idx}] changed"
        assert_bitwise(b.raw(), c["t_bounds"], f"{name}[{idx}] tighten bounds")
        assert [int(b.infeasible()), cr[0]] == list(c["t_info"])


def test_incremental_equals_full_acceptance_stream(oracle_built):
    """acceptance.cpp:37-81 — all 1000 instances of seed 20240501, engine vs reference library."""
    from oracle.bind import Ref, RefRng, ref_propagate
    if not Ref.available():
        pytest.skip("reference library missing")
    rng = RefRng(20240501)
    for t in range(1000):
        rp = rng.random_instance()
        p = rp.to_def()
        for inc in (True, False):
            lim = Lim(incremental=inc)
            rb, rinf, rst, rr, rc = ref_propagate(rp, p.root_bounds(), lim=lim)
            b = BoundsState(p)
            r = propagate(p, b, plim(lim))
            assert (b.infeasible(), int(r.status), r.rounds, r.crossed_vars) == (rinf, rst, rr, rc), t
            assert_bitwise(b.raw(), rb, f"instance {t}")


# ---------------------------------------------------------------- large shapes vs the port / reference

def _compare_with_oracle(p, lims=(Lim(),), rows_subset=True):
    from oracle.bind import PortProblem
    pp = PortProblem(p)
    root = p.root_bounds()
    act0, nmin0, nmax0 = pp.compute_activities(root)
    a = ActivityState()
    compute_activities(p, BoundsState(p), None, a)
    assert_bitwise(a.act, act0, "activities")
    assert np.array_equal(a.n_inf_min, nmin0) and np.array_equal(a.n_inf_max, nmax0)
    if rows_subset:
        rng = np.random.default_rng(0)
        rows = rng.choice(p.n_cons, size=min(p.n_cons, 500), replace=False).astype(np.int32)
        seed_act = np.full(2 * p.n_cons, 7.0)
        act1, _, _ = pp.compute_activities(root, rows=rows, act=seed_act)
        a2 = ActivityState(seed_act.copy(), np.zeros(p.n_cons, np.int32), np.zeros(p.n_cons, np.int32))
        compute_activities(p, BoundsState(p), rows, a2)
        assert_bitwise(a2.act, act1, "activities (row subset)")
    for lim in lims:
        ob, oinf, ost, orr, ocr = pp.propagate(root, lim=lim)
        b = BoundsState(p)
        r = propagate(p, b, plim(lim))
        assert (b.infeasible(), int(r.status), r.rounds, r.crossed_vars) == (oinf, ost, orr, ocr), lim
        assert_bitwise(b.raw(), ob, f"bounds {lim}")
    return pp


def test_c1_bitwise(oracle_built):
    p = synth.c1()
    _compare_with_oracle(p, lims=(Lim(), Lim(incremental=False), Lim(max_rounds=3),
                                  Lim(abs_threshold=0.0, rel_threshold=0.0)))


def test_heavy_rows_and_long_columns(oracle_built):
    """Scaled C2: rows > 16384 (multi-segment), 2048 < nnz <= 16384 (warp pairs), medium rows,
    columns > 32 (warp-reduced lexicographic fold), fractional coefficients."""
    p = synth.c2(n=40_000, m=40_000, cap=40_000, n_heavy=3)
    L = np.diff(p.row_start)
    C_ = np.diff(p.col_start)
    assert (L > 16384).sum() >= 2 and ((L > 2048) & (L <= 16384)).sum() >= 1
    assert (C_ > 32).sum() > 10
    _compare_with_oracle(p, lims=(Lim(), Lim(incremental=False)))


def test_negative_zero_ties_in_long_columns(oracle_built):
    """A 200-row column where many candidates are +0.0 and -0.0 ties: the first one in CSC order
    must win (std::min keeps the first operand), also when the column is reduced by a warp."""
    vars_ = [(0, 5, True)] + [(0, 1, True)] * 200
    rows = []
    for k in range(200):
        # x0 + y_k <= 0.5 + tiny/-tiny: floor(cand + 1e-6) -> +0.0; ranged rows give -0.0 lows
        rows.append(([(0, 1.0), (1 + k, 1.0 if k % 2 else -1.0)], -INF if k % 3 else -0.5, 0.5))
    p = make_problem(vars_, rows)
    _compare_with_oracle(p, lims=(Lim(),))


def test_infinite_bounds_mixed(oracle_built):
    rng = np.random.default_rng(5)
    n, m = 3000, 2500
    lens = rng.integers(1, 60, m)
    rows = []
    for k in range(m):
        cols = np.sort(rng.choice(n, size=lens[k], replace=False))
        rows.append(([(int(c), float(rng.choice([-2.5, -1.0, 0.5, 1.0, 3.0]))) for c in cols],
                     -INF if rng.random() < 0.5 else -50.0, 40.0 if rng.random() < 0.8 else INF))
    vars_ = []
    for i in range(n):
        u = rng.random()
        lo = -INF if u < 0.1 else float(rng.integers(-5, 1))
        up = INF if 0.1 <= u < 0.2 else float(rng.integers(1, 8))
        vars_.append((lo, up, bool(rng.random() < 0.6)))
    p = make_problem(vars_, rows)
    _compare_with_oracle(p, lims=(Lim(), Lim(incremental=False)))


def test_c5_small_instances_bitwise(oracle_built):
    """configs[4] (C5): the smallest instances of the 64-instance batch (all four generator kinds
    occur among them), each propagated on the engine and compared with the oracle bitwise."""
    specs = sorted(synth.c5_specs(), key=lambda s: s[1])
    kinds = set()
    for sp in specs[:12]:
        p = synth.c5_instance(sp)
        kinds.add(sp[2])
        _compare_with_oracle(p, lims=(Lim(),))
    assert len(kinds) >= 3


@pytest.mark.parametrize("config", ["C2", "C4"])
def test_full_size_bitwise_vs_reference(oracle_built, config):
    """BASELINE.json's full sizes: one propagate from the original bounds of C2 (1M x 1M,
    19.6M nnz, 24 rounds) and of C4 (2M x 2M, 25.7M nnz) equals the reference's own propagate
    (oracle/_ref, all host threads) bit for bit: bounds, status, rounds, crossed."""
    from oracle.bind import Ref, RefProblem, ref_propagate
    if not Ref.available():
        pytest.skip("reference library missing")
    p = synth.c2() if config == "C2" else synth.c4()[0]
    rp = RefProblem.from_def(p)
    ob, oinf, ost, orr, ocr = ref_propagate(rp, p.root_bounds())
    b = BoundsState(p)
    r = propagate(p, b)
    assert (b.infeasible(), int(r.status), r.rounds, r.crossed_vars) == (oinf, ost, orr, ocr)
    assert_bitwise(b.raw(), ob, f"{config} bounds")


def test_c5_all_instances_vs_reference(oracle_built):
    """configs[4] (C5): all 64 heterogeneous instances (10k-5M nnz, C1-C4 generators), one
    propagate each on the engine, equal the reference's own propagate (oracle/_ref) bit for bit:
    bounds, status, rounds, crossed."""
    from oracle.bind import Ref, RefProblem, ref_propagate
    if not Ref.available():
        pytest.skip("reference library missing")
    for sp in synth.c5_specs():
        p = synth.c5_instance(sp)
        rp = RefProblem.from_def(p)
        ob, oinf, ost, orr, ocr = ref_propagate(rp, p.root_bounds())
        del rp
        b = BoundsState(p)
        r = propagate(p, b)
        assert (b.infeasible(), int(r.status), r.rounds, r.crossed_vars) == (oinf, ost, orr, ocr), sp
        assert_bitwise(b.raw(), ob, f"C5 instance {sp[0]}")
