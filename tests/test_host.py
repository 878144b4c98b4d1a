"""CPU: host-side logic — the ProblemBuilder mirror, the work plan, the C-ABI library loading and
exporting every symbol include/bp.h declares. No compute calls (no GPU here)."""
import ctypes as C
import math
import re
import subprocess

import numpy as np
import pytest

from helpers import ROOT, bits
from paper_2510_20499_b200 import ProblemBuilder, build_work_plan, make_problem, size_class_of
from paper_2510_20499_b200 import _lib

INF = math.inf


def declared_symbols():
    txt = (ROOT / "include" / "bp.h").read_text()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(bp_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    so = _lib.LIB_PATH
    assert so.exists(), "libbp.so not built (run __graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\b(bp_\w+)\b", out))
    decl = declared_symbols()
    assert decl, "no declarations parsed"
    missing = [s for s in decl if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    assert sorted(_lib.exported_symbols()) == decl, "ctypes signature table out of sync with bp.h"
    L = _lib.lib()  # loads; binding every symbol
    for s in decl:
        assert hasattr(L, s)


def test_limits_default_matches_reference():
    s = _lib.limits_struct()
    assert (s.max_rounds, s.time_limit, s.abs_threshold, s.rel_threshold, s.incremental) == (
        64, INF, 1e-7, 1e-4, 1)


def test_builder_rounds_integer_bounds_to_negative_zero():
    p = make_problem([(0, 1, True), (-0.5, 2.7, True), (0, 3.5, False)], [([(0, 1.0)], -INF, 1.0)])
    assert p.var_lower[0] == 0.0 and np.signbit(p.var_lower[0])  # ceil(-1e-9) == -0.0
    assert p.var_lower[1] == 0.0 and np.signbit(p.var_lower[1])
    assert p.var_upper[1] == 2.0
    assert p.var_lower[2] == 0.0 and not np.signbit(p.var_lower[2])  # continuous untouched


def test_builder_errors_match_reference():
    b = ProblemBuilder()
    b.add_var("x", 0.5, 0.7, True)  # ceil(0.5) > floor(0.7)
    with pytest.raises(RuntimeError, match="empty domain"):
        b.build()
    b = ProblemBuilder()
    b.add_var("x", 0, 1, False)
    b.add_row("r", 2, 1)
    with pytest.raises(RuntimeError, match="crossed bounds"):
        b.build()
    b = ProblemBuilder()
    b.add_var("x", 0, 1, False)
    b.add_row("r", 0, 1)
    b.add_entry(0, 3, 1.0)
    with pytest.raises(IndexError):
        b.build()


def test_builder_sorts_coalesces_and_drops_zeros():
    b = ProblemBuilder()
    for i in range(3):
        b.add_var(f"x{i}", 0, 5, True)
    b.add_row("r0", -INF, 4)
    b.add_row("r1", -INF, 4)
    b.add_entry(1, 2, 1.0)
    b.add_entry(0, 2, 2.0)
    b.add_entry(0, 0, 1.0)
    b.add_entry(0, 2, -2.0)  # cancels -> dropped
    b.add_entry(1, 0, 3.0)
    b.add_entry(1, 0, 1.0)  # coalesced to 4
    p = b.build()
    assert list(p.row_start) == [0, 1, 3]
    assert list(p.row_col) == [0, 0, 2]
    assert list(p.row_val) == [1.0, 4.0, 1.0]
    # stable transpose: column 0 lists rows 0, 1
    assert list(p.col_start) == [0, 2, 2, 3]
    assert list(p.col_row) == [0, 1, 1]


def test_builder_matches_reference_builder(oracle_built):
    from oracle.bind import Ref, RefProblem
    if not Ref.available():
        pytest.skip("reference library not built here")
    rng = np.random.default_rng(9)
    for t in range(30):
        n, m = int(rng.integers(1, 12)), int(rng.integers(1, 10))
        lo = rng.integers(-3, 3, n).astype(float) + rng.choice([0.0, 0.3], n)
        up = lo + rng.integers(0, 5, n) + 0.6
        isint = (rng.random(n) < 0.7).astype(np.uint8)
        cl = np.where(rng.random(m) < 0.5, -INF, -5.0)
        cu = np.where(rng.random(m) < 0.5, INF, 5.0)
        ne = int(rng.integers(0, 30))
        er = rng.integers(0, m, ne).astype(np.int32)
        ec = rng.integers(0, n, ne).astype(np.int32)
        ev = rng.integers(-3, 4, ne).astype(float)  # integral: duplicate sums order-free
        b = ProblemBuilder()
        for i in range(n):
            b.add_var(f"x{i}", lo[i], up[i], bool(isint[i]))
        for k in range(m):
            b.add_row(f"c{k}", cl[k], cu[k])
        for e in range(ne):
            b.add_entry(er[e], ec[e], ev[e])
        try:
            mine = b.build()
        except RuntimeError:
            continue
        h = Ref.lib().ref_problem_build(
            n, m, *[x.ctypes.data_as(C.c_void_p) for x in (lo, up, isint)], None,
            *[x.ctypes.data_as(C.c_void_p) for x in (cl, cu)], ne,
            *[x.ctypes.data_as(C.c_void_p) for x in (er, ec, ev)])
        ref = RefProblem(h).to_def()
        for f in ("row_start", "row_col", "col_start", "col_row", "is_integer"):
            assert np.array_equal(getattr(mine, f), getattr(ref, f)), f
        for f in ("row_val", "col_val", "var_lower", "var_upper", "cons_lower", "cons_upper"):
            assert np.array_equal(bits(getattr(mine, f)), bits(getattr(ref, f))), f


def test_work_plan_bins_like_reference():
    """test_propagation.cpp:13-58."""
    vars_ = [(0, 1, True)] * 70
    rows = [([(0, 1.0)], -INF, 100.0), ([(0, 1.0), (1, 1.0)], -INF, 100.0),
            ([(0, 1.0), (1, 1.0), (2, 1.0)], -INF, 100.0), ([(i, 1.0) for i in range(70)], -INF, 100.0)]
    plan = build_work_plan(make_problem(vars_, rows))
    assert [b.size_class for b in plan.row_bins] == [0, 1, 2, 7]
    assert [b.items for b in plan.row_bins] == [[0], [1], [2], [3]]
    assert size_class_of(1) == 0 and size_class_of(2) == 1 and size_class_of(3) == 2
    assert size_class_of(16384) == 14 and size_class_of(16385) == 15
    empty = build_work_plan(ProblemBuilder().build())
    assert empty.row_bins == [] and empty.var_bins == []


def test_c5_specs_and_lpt_partition():
    """C5 instance list is deterministic; LPT partitions every instance exactly once and balances."""
    from paper_2510_20499_b200 import synth
    a, b = synth.c5_specs(), synth.c5_specs()
    assert a == b and len(a) == 64
    sizes = [s[1] for s in a]
    assert 10_000 <= min(sizes) and max(sizes) <= 5_000_000
    for world in (1, 2, 4, 8):
        parts = synth.lpt_partition(sizes, world)
        assert sorted(i for p in parts for i in p) == list(range(64))
        loads = [sum(sizes[i] for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(sizes)
    p = synth.c5_instance(min(a, key=lambda s: s[1]))
    assert p.nnz() > 0
