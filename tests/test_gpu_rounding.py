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
