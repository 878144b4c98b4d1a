"""GPU fix-and-propagate driver vs the reference's propagation_round (rounding.hpp:393) on the
same instances, start points, seeds and caches: identical integer outputs and flags. Mirrors
test_rounding.cpp and acceptance.cpp criterion 4 (rounding integrality, 1000-instance stream)."""
import math

import numpy as np
import pytest

from paper_2510_20499_b200 import make_problem, synth
from paper_2510_20499_b200.probing import build_cache
from paper_2510_20499_b200.rounding import get_bulk_size, initial_sort, propagation_round

pytestmark = pytest.mark.gpu
INF = math.inf
FLAGS = ("rounding_infeasible", "timed_out", "completed", "bulks_committed", "set_count")


def test_host_helpers_known_answers():
    assert get_bulk_size(100, False) == 10 and get_bulk_size(36, False) == 1
    assert get_bulk_size(10000, True) == 1 and get_bulk_size(37, False) == 6
    p = make_problem([(0, 1, True), (0, 1, True), (0, 9, True)], [([(0, 1.0), (1, 1.0), (2, 1.0)], -INF, 100.0)])
    assert initial_sort(p, [0.1, 0.5, 0.2]) == [0, 1, 2]
    p = make_problem([(0, 9, True), (0, 2, True), (0, 1, True)], [([(0, 1.0), (1, 1.0), (2, 1.0)], -INF, 100.0)])
    assert initial_sort(p, [1.0, 1.0, 1.0]) == [2, 1, 0]


def test_rounding_known_answers():
    p = make_problem([(0, 1, True, -1), (0, 1, True, -1)], [([(0, 1.0), (1, 1.0)], -INF, 1.0)])
    out = propagation_round(p, [0.5, 0.5], build_cache(p, 1e9), seed=3)
    assert out.completed and not out.rounding_infeasible
    x, y = out.values
    assert x + y <= 1.0 + 1e-9 and x in (0.0, 1.0) and y in (0.0, 1.0)
    out = propagation_round(p, [1.0, 0.0], None, seed=3)
    assert list(out.values) == [1.0, 0.0]
    q = make_problem([(0, 1, True)], [([(0, 1.0)], 1.0, INF), ([(0, 1.0)], -INF, 0.0)])
    out = propagation_round(q, [0.5], None, seed=3, deadline_sec=5.0)
    assert out.rounding_infeasible


def _compare(rp, p, start, seed, use_cache, tag):
    from oracle.bind import RefCache, ref_propagation_round
    gcache = build_cache(p, 1e9) if use_cache else None
    rcache = RefCache.from_gpu(rp, gcache) if use_cache else None
    rv, rf = ref_propagation_round(rp, p.n_vars, start, rcache, seed)
    g = propagation_round(p, start, gcache, seed)
    got = {k: int(getattr(g, k)) for k in FLAGS}
    assert got == {k: rf[k] for k in FLAGS}, tag
    isint = p.is_integer.astype(bool)
    assert np.array_equal(g.values[isint], rv[isint]), tag
    return g


def test_acceptance_rounding_stream_matches_reference(oracle_built):
    """acceptance.cpp:121-150 instance stream (seed 5150), GPU cache fed to both drivers."""
    from oracle.bind import Ref, RefCache, RefRng
    if not Ref.available():
        pytest.skip("reference library missing")
    rng = RefRng(5150)
    for t in range(300):
        rp = rng.random_instance()
        p = rp.to_def()
        start = np.array([p.var_lower[i] + rng.uniform_real(0.0, 1.0) * (p.var_upper[i] - p.var_lower[i])
                          for i in range(p.n_vars)])
        g = _compare(rp, p, start, t, True, f"inst{t}")
        assert np.all(np.abs(g.values - np.round(g.values)) <= 1e-9)


def test_gpu_cache_equals_reference_cache_in_rounding(oracle_built):
    from oracle.bind import Ref, RefCache, RefRng, ref_propagation_round
    rng = RefRng(42)
    for t in range(100):
        rp = rng.random_instance()
        p = rp.to_def()
        start = np.array([p.var_lower[i] + rng.uniform_real(0.0, 1.0) * (p.var_upper[i] - p.var_lower[i])
                          for i in range(p.n_vars)])
        gv = propagation_round(p, start, build_cache(p, 1e9), 1000 + t).values
        rv, _ = ref_propagation_round(rp, p.n_vars, start, RefCache.build(rp), 1000 + t)
        assert np.array_equal(gv, rv), t


def test_mixed_instance_rounding(oracle_built):
    from oracle.bind import RefProblem
    p = synth.c1(n=3000, m=3000)
    rp = RefProblem.from_def(p)
    rng = np.random.default_rng(7)
    start = p.var_lower + rng.random(p.n_vars) * (p.var_upper - p.var_lower)
    for use_cache in (False, True):
        _compare(rp, p, start, 11, use_cache, f"C1-3000 cache={use_cache}")


def _ref_parallel_propagate(rp, n, base, vars_, v0, v1, cache):
    """pulse::parallel_propagate through oracle/_ref (ref_shim.cpp ref_parallel_propagate)."""
    import ctypes as C

    from oracle.bind import Ref
    k = len(vars_)
    ob = [np.zeros(max(2 * n, 1)) for _ in range(2)]
    info = np.zeros(8, np.int32)
    ev = [np.zeros(max(k, 1), np.int32) for _ in range(2)]
    fv = [np.zeros(max(k, 1), np.int32) for _ in range(2)]
    fx = [np.zeros(max(k, 1)) for _ in range(2)]
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    Ref.lib().ref_parallel_propagate(rp.h, P(base), 0, P(np.asarray(vars_, np.int32)), k,
                                     P(np.asarray(v0, float)), P(np.asarray(v1, float)),
                                     None if cache is None else cache.h, P(ob[0]), P(ob[1]), P(info),
                                     P(ev[0]), P(ev[1]), P(fv[0]), P(fx[0]), P(fv[1]), P(fx[1]))
    out = []
    for q in range(2):
        inf, cnt, nev, nfx = (int(x) for x in info[4 * q: 4 * q + 4])
        out.append((ob[q][: 2 * n], bool(inf), cnt, ev[q][:nev].tolist(),
                    [(int(fv[q][j]), float(fx[q][j])) for j in range(nfx)]))
    return out


def test_parallel_propagate_matches_reference(oracle_built):
    """rounding.hpp:213-224 (test_rounding.cpp:144-176): both probes, with and without a cache,
    bounds / infeasibility / infeas_count / evicted / fixed identical (bounds bitwise)."""
    from oracle.bind import RefCache, RefRng

    from paper_2510_20499_b200 import BoundsState
    from paper_2510_20499_b200.rounding import parallel_propagate
    rng = RefRng(4242)
    gen = np.random.default_rng(5)
    for t in range(120):
        rp = rng.random_instance()
        p = rp.to_def()
        vars_ = [i for i in range(p.n_vars) if gen.random() < 0.6]
        lo, up = p.var_lower[vars_], p.var_upper[vars_]
        v0 = np.minimum(np.floor(lo + (up - lo + 1) * gen.random(len(vars_))), up)
        v1 = np.minimum(np.floor(lo + (up - lo + 1) * gen.random(len(vars_))), up)
        gc, rc = build_cache(p, 1e9), RefCache.build(rp)
        for use_cache in (False, True):
            g = parallel_propagate(p, BoundsState(p), vars_, v0, v1, gc if use_cache else None)
            r = _ref_parallel_propagate(rp, p.n_vars, p.root_bounds(), vars_, v0, v1,
                                        rc if use_cache else None)
            for q in range(2):
                rb, rinf, rcnt, rev, rfx = r[q]
                assert np.array_equal(g[q].bounds.raw().view(np.uint64), rb.view(np.uint64)), (t, q)
                assert (g[q].bounds.infeasible(), g[q].infeas_count, g[q].evicted, g[q].fixed) == \
                    (rinf, rcnt, rev, rfx), (t, q, use_cache)


def test_repair_known_answers():
    """test_rounding.cpp:178-205 (repair shifts fixed values inside original bounds)."""
    from paper_2510_20499_b200.rounding import repair
    knap = make_problem([(0, 1, True, -1), (0, 1, True, -1)], [([(0, 1.0), (1, 1.0)], -INF, 1.0)])
    r = repair(knap, [(0, 1.0), (1, 1.0)])
    assert r is not None
    vals = dict(r.values)
    assert vals[0] + vals[1] <= 1.0
    capped = make_problem([(0, 3, True)], [([(0, 1.0)], 5.0, INF)])
    assert repair(capped, [(0, 3.0)]) is None
    r = repair(knap, [(0, 1.0), (1, 0.0)])
    assert r is not None and r.values == [(0, 1.0), (1, 0.0)]


def test_repair_matches_reference(oracle_built):
    """repair (rounding.hpp:234-311) on random fixings of random instances: presence, shifted
    values and the propagated bounds identical to the reference's (bounds bitwise)."""
    from oracle.bind import RefRng, ref_repair

    from paper_2510_20499_b200.rounding import RoundingConfig, repair
    rng = RefRng(8080)
    gen = np.random.default_rng(17)
    n_ok = 0
    for t in range(150):
        rp = rng.random_instance()
        p = rp.to_def()
        ints = [i for i in range(p.n_vars) if p.is_integer[i]]
        if not ints:
            continue
        vars_ = [i for i in ints if gen.random() < 0.8] or ints[:1]
        if gen.random() < 0.2:
            vars_ = vars_ + vars_[:1]  # a repeated fixing: the last one wins
        fixed = [(v, float(np.floor(p.var_lower[v] + (p.var_upper[v] - p.var_lower[v] + 1) * gen.random())))
                 for v in vars_]
        fixed = [(v, min(x, float(p.var_upper[v]))) for v, x in fixed]
        cap = int(gen.choice([1, 2, 64]))
        g = repair(p, fixed, cfg=RoundingConfig(repair_shift_cap=cap))
        r = ref_repair(rp, p.n_vars, fixed, cap)
        assert (g is None) == (r is None), t
        if g is None:
            continue
        n_ok += 1
        assert g.values == r[0], t
        assert np.array_equal(g.bounds.raw().view(np.uint64), r[1].view(np.uint64)), t
    assert n_ok > 10


def test_rounding_with_repair_known_answers():
    """test_rounding.cpp:360-390 (propagation_round drives repair when enabled)."""
    from paper_2510_20499_b200.rounding import RoundingConfig
    cfg = RoundingConfig(repair_enabled=True)
    q = make_problem([(0, 1, True)], [([(0, 1.0)], 1.0, INF), ([(0, 1.0)], -INF, 0.0)])
    out = propagation_round(q, [0.5], None, seed=9, deadline_sec=5.0, cfg=cfg)
    assert out.repair_attempts >= 1 and out.rounding_infeasible and out.completed
    e = make_problem([(0, 1, True), (0, 1, True)], [([(0, 1.0), (1, 1.0)], 2.0, 2.0)])
    out = propagation_round(e, [0.2, 0.2], None, seed=4, deadline_sec=5.0, cfg=cfg)
    assert out.completed and list(out.values) == [1.0, 1.0]


def test_rounding_with_repair_matches_reference(oracle_built):
    """propagation_round with repair_enabled on the acceptance-style stream: identical integer
    outputs and flags, including repair_attempts."""
    from oracle.bind import RefRng, ref_propagation_round

    from paper_2510_20499_b200.rounding import RoundingConfig
    rng = RefRng(6161)
    cfg = RoundingConfig(repair_enabled=True)
    attempts = 0
    for t in range(300):
        rp = rng.random_instance()
        p = rp.to_def()
        start = np.array([p.var_lower[i] + rng.uniform_real(0.0, 1.0) * (p.var_upper[i] - p.var_lower[i])
                          for i in range(p.n_vars)])
        rv, rf = ref_propagation_round(rp, p.n_vars, start, None, t, repair=True)
        g = propagation_round(p, start, None, t, cfg=cfg)
        keys = FLAGS + ("repair_attempts",)
        assert {k: int(getattr(g, k)) for k in keys} == {k: rf[k] for k in keys}, t
        isint = p.is_integer.astype(bool)
        assert np.array_equal(g.values[isint], rv[isint]), t
        attempts += g.repair_attempts
    assert attempts > 0


def test_c4_scaled_full_cache_vs_reference(oracle_built):
    """SURVEY §8d C4 parity run, scaled: a 20k x 20k knapsack/assignment instance (configs[3]'s
    generator, long rows included) presolved to its fixpoint; a FULL-coverage cache built on the
    GPU (sample-verified against the reference's own probe_variable), handed to both drivers;
    propagation_round with Deadline::never and Rng(4): identical integer outputs and every
    RoundingOutcome flag (rounding.hpp:393-558)."""
    from oracle.bind import Ref, RefCache, RefProblem, cache_mismatches, ref_propagation_round
    if not Ref.available():
        pytest.skip("reference library missing")
    from paper_2510_20499_b200 import BoundsState, propagate
    p0, start = synth.c4(n=20_000, m=20_000, n_long=10, long_len=2000)
    b = BoundsState(p0)
    propagate(p0, b)
    p = synth.with_bounds(p0, b.raw())
    rp = RefProblem.from_def(p)
    gcache = build_cache(p, 1e9)
    free_int = [v for v in range(p.n_vars) if p.is_integer[v] and p.var_lower[v] != p.var_upper[v]]
    assert gcache.n_probed >= len(free_int) > 10_000
    sample = np.random.default_rng(4).choice(free_int, size=64, replace=False)
    checked, bad = cache_mismatches(gcache, RefCache.probe_into(rp, p.n_vars, p.root_bounds(), sample), sample)
    assert checked == 64 and bad == []
    rcache = RefCache.from_gpu(rp, gcache)
    rv, rf = ref_propagation_round(rp, p.n_vars, start, rcache, 4)
    g = propagation_round(p, start, gcache, 4)
    assert {k: int(getattr(g, k)) for k in FLAGS} == {k: rf[k] for k in FLAGS}
    assert g.completed and rf["completed"]
    isint = p.is_integer.astype(bool)
    assert np.array_equal(g.values[isint], rv[isint])


def _tight_heavy_instance(seed=11, n=80_000):
    """Heavy rows (two 16384-segments each) that are knapsacks over binaries, next to loose heavy
    rows: in each knapsack a chain of 12 binaries (c0 >= 1, c_{i+1} >= c_i, weight 30) rises one
    per round, so the knapsack's slack shrinks round by round from 400 to 40 -- certified quiet
    (chains skipped, record stale) while the slack exceeds its reach, exact once it does not, then
    fixing its heavy binaries to 0. Frontier calls and probing then read the records the lazy
    rounds left behind."""
    from paper_2510_20499_b200.problem import problem_from_csr
    rng = np.random.default_rng(seed)
    nb, ni = int(0.6 * n), int(0.2 * n)
    lo = np.zeros(n)
    up = np.concatenate([np.ones(nb), np.full(ni, 10.0), rng.uniform(1.0, 50.0, n - nb - ni)])
    isint = np.concatenate([np.ones(nb + ni, np.uint8), np.zeros(n - nb - ni, np.uint8)])
    rows, cl, cu = [], [], []
    for q in range(2):  # over disjoint halves of the binaries
        c = np.sort(q * (nb // 2) + rng.choice(nb // 2, size=20_000, replace=False))
        w = rng.integers(1, 100, size=c.size).astype(np.float64)
        chain = np.sort(rng.choice(c.size, size=12, replace=False))
        w[chain] = 30.0
        rows.append((c, w))
        cl.append(-math.inf)
        cu.append(400.0)
        cv = c[chain]
        rows.append((cv[:1], np.ones(1)))
        cl.append(1.0)
        cu.append(math.inf)
        for i in range(11):
            rows.append((np.sort(cv[i:i + 2]), np.where(cv[i:i + 2] == cv[i + 1], 1.0, -1.0)[np.argsort(cv[i:i + 2])]))
            cl.append(0.0)
            cu.append(math.inf)
    for _ in range(2):  # loose heavy rows, fractional coefficients
        c = np.sort(rng.choice(n, size=40_000, replace=False))
        rows.append((c, rng.uniform(0.1, 5.0, size=c.size) * rng.choice([-1.0, 1.0], size=c.size)))
        cl.append(-1e7)
        cu.append(1e7)
    for _ in range(12000):  # short mixed rows
        L = int(rng.integers(2, 9))
        c = np.sort(rng.choice(n, size=L, replace=False))
        a = np.where(c < nb + ni, rng.integers(1, 6, size=L), rng.uniform(0.5, 3.0, size=L)) * rng.choice([-1.0, 1.0], size=L)
        rows.append((c, a.astype(np.float64)))
        cl.append(-math.inf)
        cu.append(float(np.sum(np.maximum(a, 0.0) * up[c]) * 0.6))
    row_start = np.concatenate([[0], np.cumsum([r[0].size for r in rows])]).astype(np.int32)
    cols = np.concatenate([r[0] for r in rows]).astype(np.int32)
    vals = np.concatenate([r[1] for r in rows])
    p = problem_from_csr(n, len(rows), row_start, cols, vals, lo, up, isint, np.array(cl), np.array(cu),
                         name="tight-heavy")
    start = lo + rng.random(n) * (up - lo)
    return p, start


def test_lazy_heavy_rows_vs_reference(oracle_built):
    """Propagate (incremental and every-round-full), probing from the resulting certified root and
    fix-and-propagate with that cache, all against the reference, on _tight_heavy_instance."""
    from oracle.bind import Ref, RefCache, RefProblem, cache_mismatches, ref_propagate, ref_propagation_round
    if not Ref.available():
        pytest.skip("reference library missing")
    from paper_2510_20499_b200 import BoundsState, PropagationLimits, propagate
    p, start = _tight_heavy_instance()
    assert (np.diff(p.row_start) > 16384).sum() == 4
    rp = RefProblem.from_def(p)
    for inc in (True, False):
        ob, oinf, ost, orr, ocr = ref_propagate(rp, p.root_bounds(), lim=PropagationLimits(incremental=inc))
        b = BoundsState(p)
        r = propagate(p, b, PropagationLimits(incremental=inc))
        assert (b.infeasible(), int(r.status), r.rounds, r.crossed_vars) == (oinf, ost, orr, ocr)
        assert r.rounds >= 3
        assert np.array_equal(b.raw().view(np.uint64), ob.view(np.uint64)), inc
    b = BoundsState(p)
    propagate(p, b)
    q = synth.with_bounds(p, b.raw())
    rq = RefProblem.from_def(q)
    gcache = build_cache(q, 1e9)
    free = [v for v in range(q.n_vars) if q.var_lower[v] != q.var_upper[v] and q.is_integer[v]]
    sample = np.random.default_rng(3).choice(free, size=48, replace=False)
    checked, bad = cache_mismatches(gcache, RefCache.probe_into(rq, q.n_vars, q.root_bounds(), sample), sample)
    assert checked == 48 and bad == []
    rcache = RefCache.from_gpu(rq, gcache)
    rv, rf = ref_propagation_round(rq, q.n_vars, start, rcache, 7)
    g = propagation_round(q, start, gcache, 7)
    assert {k: int(getattr(g, k)) for k in FLAGS} == {k: rf[k] for k in FLAGS}
    isint = q.is_integer.astype(bool)
    assert np.array_equal(g.values[isint], rv[isint])
