"""GPU parity of the batched double-probing engine (probing cache) vs the reference's golden
vectors and the plain-C port. Mirrors test_probing.cpp and acceptance.cpp criterion 3
(cache == memoized propagation, exact equality), then scales to certified-fixpoint roots
(the batched warp-per-branch kernel) and to the C3 set-covering shape."""
import math

import numpy as np
import pytest

from helpers import assert_bitwise, case_problem, golden
from paper_2510_20499_b200 import BoundsState, make_problem, synth
from paper_2510_20499_b200.probing import (BranchKind, assemble_bulk_warm_start, build_cache,
                                           make_branch_spec, probe_variable, probe_variables)

pytestmark = pytest.mark.gpu
INF = math.inf


def tiny_knapsack():
    return make_problem([(0, 1, True, -1), (0, 1, True, -1)], [([(0, 1.0), (1, 1.0)], -INF, 1.0)])


def test_branch_specs():
    p = make_problem([(0, 10, True)], [([(0, 1.0)], -INF, 100.0)])
    s = make_branch_spec(BoundsState(p), 0)
    assert s.kind == BranchKind.BoxedSplit and (s.down_lower, s.down_upper, s.up_lower, s.up_upper) == (0, 4, 5, 10)
    p = make_problem([(0, INF, True)], [([(0, 1.0)], -INF, 100.0)])
    s = make_branch_spec(BoundsState(p), 0)
    assert s.kind == BranchKind.AtLowerBound and (s.down_upper, s.up_lower, s.up_upper) == (0, 1, INF)


def test_probe_variable_known_answers():
    p = tiny_knapsack()
    e = probe_variable(p, BoundsState(p), 0)
    assert e.up.feasible and e.down.feasible
    assert [d.new_upper for d in e.up.deltas if d.var == 1] == [0.0]
    assert all(d.var == 0 for d in e.down.deltas)
    q = make_problem([(0, 1, True), (0, 1, True)], [([(0, 1.0), (1, 1.0)], -INF, 1.0), ([(1, 1.0)], 1.0, INF)])
    e = probe_variable(q, BoundsState(q), 1)
    assert not e.down.feasible and e.down.deltas == [] and e.up.feasible and e.forces_up


def test_build_cache_budget_and_forcing():
    p = make_problem([(0, 1, True), (0, 1, True), (0, 3, True), (0, 3, True), (0, 1, True)],
                     [([(0, 1.0), (1, 1.0), (2, 1.0)], -INF, 3.0), ([(3, 1.0), (4, 1.0)], -INF, 3.0)])
    assert build_cache(p, 0.0).n_probed == 0
    c = build_cache(p, 1e9)
    assert c.n_probed == 5 and all(c.has(v) for v in range(5))
    q = make_problem([(0, 1, True), (0, 1, True)], [([(0, 1.0), (1, 1.0)], -INF, 1.0), ([(1, 1.0)], 1.0, INF)])
    c = build_cache(q, 1e9)
    assert c.at(1).forces_up and c.at(0).forces_down and c.n_infeasible_branches == 2


def test_warm_start_merge_and_eviction():
    p = tiny_knapsack()
    cache = build_cache(p, 1e9)
    ws = assemble_bulk_warm_start(cache, [(0, 1.0)])
    assert ws.conflicts == [] and ws.bounds.upper(1) == 0.0
    ws = assemble_bulk_warm_start(cache, [(0, 1.0), (1, 1.0)])
    assert ws.conflicts == [(0, 1)] and ws.evicted == [1]
    ws = assemble_bulk_warm_start(cache, [])
    assert ws.conflicts == [] and ws.bounds == cache.root


def _check_entry(p, cache, v, hdr_or_port, name):
    """Compares the GPU entry of v with a port probe (kind, out) tuple."""
    kind, out = hdr_or_port
    e = cache.at(v)
    for side, br in ((0, e.down), (1, e.up)):
        feas, dv, dl, du = out[side]
        assert br.feasible == feas, f"{name} v{v} side{side} feasible"
        assert [d.var for d in br.deltas] == list(dv), f"{name} v{v} side{side} delta vars"
        assert_bitwise([d.new_lower for d in br.deltas], dl, f"{name} v{v} lo")
        assert_bitwise([d.new_upper for d in br.deltas], du, f"{name} v{v} up")


def test_cache_matches_golden_memoized_propagation():
    """acceptance.cpp:85-117 / test_probing.cpp:194-219 on the reference's own outputs."""
    for idx, c in enumerate(golden("probe")):
        p = case_problem(c)
        cache = probe_variables(p, None, list(range(p.n_vars)))
        hdr = c["hdr"].reshape(-1, 7)
        doff = c["doff"]
        for v in range(p.n_vars):
            e = cache.at(v)
            assert [int(e.kind), int(e.forces_down), int(e.forces_up), int(e.down.feasible),
                    int(e.up.feasible), len(e.down.deltas), len(e.up.deltas)] == list(hdr[v]), (idx, v)
            for side, br in ((0, e.down), (1, e.up)):
                sl = slice(doff[2 * v + side], doff[2 * v + side + 1])
                assert [d.var for d in br.deltas] == list(c["dvar"][sl])
                assert_bitwise([d.new_lower for d in br.deltas], c["dlo"][sl], f"probe[{idx}] lo")
                assert_bitwise([d.new_upper for d in br.deltas], c["dup"][sl], f"probe[{idx}] up")


def test_certified_roots_use_batched_kernel(oracle_built):
    """Roots that are fixpoints (propagated first) take the warm-free batched kernel path."""
    from oracle.bind import PortProblem, RefRng
    rng = RefRng(2025)
    checked = 0
    for t in range(600):
        rp = rng.random_instance(max_vars=8, max_rows=8)
        p = rp.to_def()
        pp = PortProblem(p)
        root, inf, st, rounds, cr = pp.propagate(p.root_bounds())
        if inf:
            continue
        cache = probe_variables(p, BoundsState(raw=root), list(range(p.n_vars)))
        assert cache.certified and cache.n_fallback == 0, t
        for v in range(p.n_vars):
            _check_entry(p, cache, v, pp.probe_variable(root, v), f"inst{t}")
        checked += 1
    assert checked > 50


def test_c1_probing_from_fixpoint(oracle_built):
    from oracle.bind import PortProblem
    p = synth.c1(n=3000, m=3000)
    pp = PortProblem(p)
    root, inf, _, _, _ = pp.propagate(p.root_bounds())
    assert not inf
    vars_ = [i for i in range(p.n_vars) if p.is_integer[i] and root[2 * i] != root[2 * i + 1]][:300]
    cache = probe_variables(p, BoundsState(raw=root), vars_)
    assert cache.certified
    for v in vars_[:120]:
        _check_entry(p, cache, v, pp.probe_variable(root, v), "C1")


def test_c1_probing_uncertified_root_block_kernel(oracle_built):
    """Original bounds of C1 are not a fixpoint: every branch runs on the block-per-branch kernel
    with a full first round (propagation.hpp:442), no engine fallback."""
    from oracle.bind import PortProblem
    p = synth.c1(n=1500, m=1500)
    pp = PortProblem(p)
    vars_ = [i for i in range(p.n_vars) if p.is_integer[i]][:400]
    cache = probe_variables(p, None, vars_)
    assert not cache.certified and cache.n_fallback == 0 and cache.n_block > 0
    root = p.root_bounds()
    for v in vars_:
        _check_entry(p, cache, v, pp.probe_variable(root, v), "C1-orig")


def test_c3_probing_sample(oracle_built):
    from oracle.bind import PortProblem
    p = synth.c3(n_bin=20_000, n_cont=30_000, n_cover=40_000, n_link=10_000)
    pp = PortProblem(p)
    rng = np.random.default_rng(3)
    vars_ = list(range(20_000))
    cache = probe_variables(p, None, vars_)
    assert cache.certified and cache.n_probed == 20_000
    assert cache.n_fallback == 0  # overlay overflows re-run exactly on the block kernel
    root = p.root_bounds()
    for v in rng.choice(20_000, size=60, replace=False):
        _check_entry(p, cache, int(v), pp.probe_variable(root, int(v)), "C3")


def test_pack_merge_roundtrip():
    p = synth.c3(n_bin=2000, n_cont=3000, n_cover=4000, n_link=1000)
    full = probe_variables(p, None, list(range(2000)))
    a = probe_variables(p, None, list(range(0, 2000, 2)))
    b = probe_variables(p, None, list(range(1, 2000, 2)))
    from paper_2510_20499_b200.probing import ProbingCache
    merged = ProbingCache.empty(BoundsState(p))
    merged.merge_packed(a.pack())
    merged.merge_packed(b.pack())
    assert merged.n_probed == full.n_probed == 2000
    assert merged.n_infeasible_branches == full.n_infeasible_branches
    for v in range(0, 2000, 7):
        x, y = merged.at(v), full.at(v)
        assert x == y


def test_prioritize_on_device_matches_reference(oracle_built):
    """prioritize_probe_vars (probing.hpp:105-190) computed on the device (warp-per-column keys +
    three stable radix passes) equals the reference's stable order on mixed-sign instances with
    long rows and columns, and on a knapsack/assignment instance."""
    import ctypes as C

    from oracle.bind import Ref, RefProblem

    from paper_2510_20499_b200.probing import prioritize_probe_vars
    for p in (synth.c1(seed=5, n=4000, m=3000), synth.c4(seed=6, n=6000, m=6000, n_long=4, long_len=3000)[0]):
        rp = RefProblem.from_def(p)
        ref = np.zeros(max(p.n_vars, 1), np.int32)
        k = Ref.lib().ref_prioritize_probe_vars(rp.h, ref.ctypes.data_as(C.c_void_p))
        assert prioritize_probe_vars(p) == ref[:k].tolist()


def test_c3_full_size_vs_reference(oracle_built):
    """configs[2] at full size (500k x 500k, 200k binaries): every binary is probed on the batched
    kernel from the original bounds (a certified fixpoint), and 512 of them, spread over the whole
    range, equal the reference's own probe_variable (probing.hpp:225, oracle/_ref) bit for bit:
    kind, forcing flags, feasibility, branch bounds, delta vars and values."""
    from oracle.bind import Ref, RefCache, RefProblem, cache_mismatches
    if not Ref.available():
        pytest.skip("reference library missing")
    p = synth.c3()
    cache = probe_variables(p, None, np.arange(200_000, dtype=np.int32))
    assert cache.certified and cache.n_probed == 200_000 and cache.n_fallback == 0
    vars_ = np.sort(np.random.default_rng(33).choice(200_000, size=512, replace=False))
    rc = RefCache.probe_into(RefProblem.from_def(p), p.n_vars, p.root_bounds(), vars_)
    checked, bad = cache_mismatches(cache, rc, vars_)
    assert checked == 512 and bad == [], bad[:10]


def test_c4_long_frontiers_on_block_kernel(oracle_built):
    """C4 shape (knapsack rows of 3000 entries, assignment blocks) from its presolved fixpoint:
    branches whose frontier reaches a long row overflow the warp overlays and run on the
    block-per-branch kernel; every sampled entry equals the reference's probe_variable."""
    from oracle.bind import Ref, RefCache, RefProblem, cache_mismatches
    if not Ref.available():
        pytest.skip("reference library missing")
    from paper_2510_20499_b200 import propagate
    p0, _ = synth.c4(n=30_000, m=30_000, n_long=20, long_len=6000)
    b = BoundsState(p0)
    propagate(p0, b)
    p = synth.with_bounds(p0, b.raw())
    free_int = [v for v in range(p.n_vars) if p.is_integer[v] and p.var_lower[v] != p.var_upper[v]]
    cache = probe_variables(p, None, free_int)
    assert cache.certified and cache.n_fallback == 0 and cache.n_block > 0
    rng = np.random.default_rng(44)
    sample = sorted(set(rng.choice(free_int, size=200, replace=False).tolist()))
    checked, bad = cache_mismatches(cache, RefCache.probe_into(RefProblem.from_def(p), p.n_vars, p.root_bounds(), sample), sample)
    assert checked == len(sample) and bad == [], bad[:10]
