"""Deterministic synthetic MILP generators for the benchmark configurations (BASELINE.json
``configs``; concrete shapes in SURVEY §8d).  All data is synthetic (no network, no MIPLIB).

C1  m=n=10k, row length 6+Binomial(4,1/2), mixed binary/integer/continuous     (configs[0])
C2  m=n=1M, Pareto row lengths (median 7, max 100k) + 8 rows of 100k, mildly
    Zipf-skewed columns                                                          (configs[1])
C3  m=n=500k set-covering: 200k binaries + 300k continuous, 400k cover rows,
    100k linking rows Σy − 20x_b <= 0                                            (configs[2])

Every row has a planted feasible point, so propagation never proves infeasibility on the
original bounds. Output is a built ProblemDef (sorted, duplicate-free CSR; integral integer
bounds exactly like ProblemBuilder::build).
"""
from __future__ import annotations

import math

import numpy as np

from .problem import ProblemDef, problem_from_csr


def _distinct_cols(rng, lengths, n, col_sampler):
    """Per-row columns (sorted, duplicates removed) for the given row lengths."""
    m = lengths.size
    rows = np.repeat(np.arange(m, dtype=np.int64), lengths)
    cols = col_sampler(rows.size).astype(np.int64)
    key = rows * n + cols
    key.sort()
    if key.size:
        keep = np.empty(key.size, dtype=bool)
        keep[0] = True
        np.not_equal(key[1:], key[:-1], out=keep[1:])
        key = key[keep]  # sorted by (row, col), distinct
    r = (key // n).astype(np.int64)
    c = (key % n).astype(np.int32)
    row_start = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=m), out=row_start[1:])
    return row_start, c


def mixed_instance(n, m, lengths, seed, col_sampler=None, frac=(0.5, 0.3, 0.2), name="mixed"):
    """Mixed binary/integer/continuous instance with a planted feasible point.

    vars: frac[0] binary [0,1], frac[1] integer [0,10], rest continuous [0, U(1,100)]
    coefficients: ±(1+floor(9U)) on integer vars, ±U(0.1,10) on continuous vars
    rows: 70% <=, 20% >=, 5% ranged, 5% equality; rhs = planted LHS ± U(0,3)
    """
    rng = np.random.default_rng(seed)
    if col_sampler is None:
        col_sampler = lambda size: rng.integers(0, n, size=size)
    kind = rng.random(n)
    is_bin = kind < frac[0]
    is_int = kind < frac[0] + frac[1]
    lo = np.zeros(n)
    up = np.where(is_bin, 1.0, np.where(is_int, 10.0, rng.uniform(1.0, 100.0, size=n)))
    isint = is_int.astype(np.uint8)
    x = np.where(is_int, np.floor(rng.random(n) * (up + 1.0)), rng.random(n) * up)
    x = np.minimum(x, up)

    row_start, cols = _distinct_cols(rng, lengths, n, col_sampler)
    nnz = cols.size
    sign = np.where(rng.random(nnz) < 0.5, -1.0, 1.0)
    ci = isint[cols].astype(bool)
    mag = np.where(ci, 1.0 + np.floor(9.0 * rng.random(nnz)), rng.uniform(0.1, 10.0, size=nnz))
    vals = sign * mag
    lhs = np.add.reduceat(vals * x[cols], row_start[:-1]) if nnz else np.zeros(m)
    empty = np.diff(row_start) == 0
    lhs[empty] = 0.0
    sense = rng.random(m)
    s1 = rng.uniform(0.0, 3.0, size=m)
    s2 = rng.uniform(0.0, 3.0, size=m)
    cl = np.full(m, -math.inf)
    cu = np.full(m, math.inf)
    le = sense < 0.70
    ge = (sense >= 0.70) & (sense < 0.90)
    rg = (sense >= 0.90) & (sense < 0.95)
    eq = sense >= 0.95
    cu[le] = lhs[le] + s1[le]
    cl[ge] = lhs[ge] - s1[ge]
    cl[rg] = lhs[rg] - s1[rg]
    cu[rg] = lhs[rg] + s2[rg]
    cl[eq] = lhs[eq]
    cu[eq] = lhs[eq]
    return problem_from_csr(n, m, row_start.astype(np.int32), cols, vals, lo, up, isint, cl, cu,
                            name=name)


def c1(seed=1, n=10_000, m=10_000) -> ProblemDef:
    """configs[0]: 10k x 10k, ~8 nnz/row, mixed types."""
    rng = np.random.default_rng(seed + 1000)
    lengths = 6 + rng.binomial(4, 0.5, size=m)
    return mixed_instance(n, m, lengths, seed, name=f"C1-{n}x{m}")


def pareto_lengths(rng, m, alpha=1.239, xmin=4.0, cap=100_000, n_heavy=8):
    L = np.floor(xmin * rng.random(m) ** (-1.0 / alpha)).astype(np.int64)
    L = np.clip(L, 1, cap)
    heavy = rng.choice(m, size=min(n_heavy, m), replace=False)
    L[heavy] = cap
    return L


def c2(seed=2, n=1_000_000, m=1_000_000, cap=100_000, n_heavy=8) -> ProblemDef:
    """configs[1]: 1M x 1M power-law rows (median 7, max 100k), skewed columns."""
    rng = np.random.default_rng(seed + 2000)
    lengths = pareto_lengths(rng, m, cap=min(cap, n), n_heavy=n_heavy)
    perm = rng.permutation(n)

    def cols(size):
        u = rng.random(size)
        skew = rng.random(size) < 0.5
        c = np.where(skew, np.floor(n * u * u), np.floor(n * u)).astype(np.int64)
        return perm[np.minimum(c, n - 1)]

    return mixed_instance(n, m, lengths, seed, col_sampler=cols, name=f"C2-{n}x{m}")


def c3(seed=3, n_bin=200_000, n_cont=300_000, n_cover=400_000, n_link=100_000) -> ProblemDef:
    """configs[2]: set covering + linking. Vars [0, n_bin) binary, then continuous."""
    rng = np.random.default_rng(seed + 3000)
    n = n_bin + n_cont
    m = n_cover + n_link
    lo = np.zeros(n)
    up = np.concatenate([np.ones(n_bin), rng.uniform(1.0, 20.0, size=n_cont)])
    isint = np.concatenate([np.ones(n_bin, np.uint8), np.zeros(n_cont, np.uint8)])
    # cover rows: sum of 4..12 distinct binaries >= 1
    lens = rng.integers(4, 13, size=n_cover)
    rs, cc = _distinct_cols(rng, lens, n_bin, lambda size: rng.integers(0, n_bin, size=size))
    cover_vals = np.ones(cc.size)
    # linking rows: sum_j y_j - 20 x_b <= 0, each continuous var in exactly one linking row
    ys = rng.permutation(n_cont) + n_bin
    split = np.sort(rng.choice(np.arange(1, n_cont), size=n_link - 1, replace=False))
    ygroups = np.split(ys, split)
    xb = rng.integers(0, n_bin, size=n_link)
    link_cols, link_vals, link_start = [], [], [0]
    for g, b in zip(ygroups, xb):
        cols_k = np.concatenate([[b], np.sort(g)]).astype(np.int32)
        vals_k = np.concatenate([[-20.0], np.ones(g.size)])
        link_cols.append(cols_k)
        link_vals.append(vals_k)
        link_start.append(link_start[-1] + cols_k.size)
    row_start = np.concatenate([rs, rs[-1] + np.array(link_start[1:], dtype=np.int64)])
    cols = np.concatenate([cc] + link_cols).astype(np.int32)
    vals = np.concatenate([cover_vals] + link_vals)
    cl = np.concatenate([np.ones(n_cover), np.full(n_link, -math.inf)])
    cu = np.concatenate([np.full(n_cover, math.inf), np.zeros(n_link)])
    return problem_from_csr(n, m, row_start.astype(np.int32), cols, vals, lo, up, isint, cl, cu,
                            name=f"C3-{n}x{m}")


CONFIGS = {"C1": c1, "C2": c2, "C3": c3}


def c4(seed=4, n=2_000_000, m=2_000_000, bin_frac=0.8, n_long=100, long_len=20_000):
    """configs[3]: knapsack/assignment mix. Binaries are partitioned into
    assignment blocks of 4..16 (sum = 1 equalities); the other rows are knapsacks
    sum w_j x_j <= C with integer weights 1..99 over random binaries / integers [0, 10] (a few
    long ones), capacities planted around a feasible point. Returns (problem, start point U(lb, ub))."""
    rng = np.random.default_rng(seed + 4000)
    nb = int(n * bin_frac)
    lo = np.zeros(n)
    up = np.concatenate([np.ones(nb), np.full(n - nb, 10.0)])
    isint = np.ones(n, np.uint8)
    # assignment blocks over the binaries
    sizes = []
    tot = 0
    while tot < nb:
        s = int(rng.integers(4, 17))
        s = min(s, nb - tot)
        sizes.append(s)
        tot += s
    sizes = np.array(sizes, dtype=np.int64)
    n_asg = sizes.size
    x = np.zeros(n)
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    pick = starts + np.floor(rng.random(n_asg) * sizes).astype(np.int64)
    x[pick] = 1.0
    x[nb:] = rng.integers(0, 11, size=n - nb)
    m_k = max(m - n_asg, 0)
    lens = 6 + rng.poisson(6, size=m_k)
    if n_long and m_k > n_long:
        lens[rng.choice(m_k, size=n_long, replace=False)] = min(long_len, n)
    rs_k, cols_k = _distinct_cols(rng, lens, n, lambda size: rng.integers(0, n, size=size))
    w = rng.integers(1, 100, size=cols_k.size).astype(np.float64)
    lhs = np.add.reduceat(w * x[cols_k], rs_k[:-1]) if cols_k.size else np.zeros(m_k)
    lhs[np.diff(rs_k) == 0] = 0.0
    cap_max = np.add.reduceat(w * up[cols_k], rs_k[:-1]) if cols_k.size else np.zeros(m_k)
    cap = np.floor(lhs + rng.uniform(0.0, 0.15, size=m_k) * (cap_max - lhs))
    # assemble: assignment rows first, then knapsacks
    a_cols = np.arange(nb, dtype=np.int32)
    row_start = np.concatenate([starts, [nb], nb + rs_k[1:]]).astype(np.int64)
    cols = np.concatenate([a_cols, cols_k]).astype(np.int32)
    vals = np.concatenate([np.ones(nb), w])
    cl = np.concatenate([np.ones(n_asg), np.full(m_k, -math.inf)])
    cu = np.concatenate([np.ones(n_asg), cap])
    p = problem_from_csr(n, n_asg + m_k, row_start.astype(np.int32), cols, vals, lo, up, isint, cl,
                         cu, name=f"C4-{n}x{n_asg + m_k}")
    start = lo + rng.random(n) * (up - lo)
    return p, start


def c5_specs(seed=100, count=64, lo_nnz=10_000, hi_nnz=5_000_000):
    """configs[4] instance list without building anything: (seed, target nnz, kind, row/col ratio)
    per instance; nnz log-uniform in [lo_nnz, hi_nnz], kind = which of the C1-C4 generators,
    ratio U(0.5, 2). Lets ranks LPT-partition by size and build only their own."""
    out = []
    for j in range(count):
        rng = np.random.default_rng(seed + j)
        nnz = float(np.exp(rng.uniform(np.log(lo_nnz), np.log(hi_nnz))))
        ratio = float(rng.uniform(0.5, 2.0))
        kind = int(rng.integers(0, 4))
        out.append((seed + j, nnz, kind, ratio))
    return out


def c5_instance(spec) -> ProblemDef:
    """Builds one C5 instance from its spec (see c5_specs)."""
    s, nnz, kind, ratio = spec
    rng = np.random.default_rng(s)
    rng.uniform(), rng.uniform(), rng.integers(0, 4)  # the draws c5_specs consumed
    j = s
    if kind == 0:  # C1-like: ~8 nnz per row
        m = max(int(nnz / 8), 10)
        n = max(int(m / ratio), 10)
        lengths = np.minimum(6 + rng.binomial(4, 0.5, size=m), n)
        return mixed_instance(n, m, lengths, s, name=f"C5-{j}-C1")
    if kind == 1:  # C2-like power law
        m = max(int(nnz / 19), 10)
        n = max(int(m / ratio), 10)
        lengths = pareto_lengths(rng, m, cap=min(100_000, n), n_heavy=min(8, max(m // 1000, 1)))
        return mixed_instance(n, m, lengths, s, name=f"C5-{j}-C2")
    if kind == 2:  # C3-like covering
        nb = max(int(nnz / 36), 100)
        return c3(s, n_bin=nb, n_cont=int(1.5 * nb), n_cover=max(int(2 * nb / ratio), 10),
                  n_link=max(nb // 2, 1))
    n = max(int(nnz / 12), 100)  # C4-like knapsack/assignment
    return c4(s, n=n, m=max(int(n * ratio), 50), n_long=0)[0]


def c5(seed=100, count=64, lo_nnz=10_000, hi_nnz=5_000_000):
    """configs[4]: `count` heterogeneous instances (c5_specs), yields (seed, problem)."""
    for spec in c5_specs(seed, count, lo_nnz, hi_nnz):
        yield spec[0], c5_instance(spec)


def lpt_partition(sizes, world):
    """Longest-processing-time assignment of items (by size) to `world` bins: list of index lists."""
    bins = [[] for _ in range(world)]
    load = [0.0] * world
    for i in sorted(range(len(sizes)), key=lambda i: -sizes[i]):
        b = min(range(world), key=lambda r: load[r])
        bins[b].append(i)
        load[b] += sizes[i]
    return bins


CONFIGS["C4"] = c4


def with_bounds(p, bounds) -> ProblemDef:
    """The same instance with its variable bounds replaced by ``bounds`` (interleaved 2n), e.g. a
    propagated fixpoint ("presolved" root: probing and rounding then start from a certified
    fixpoint, so every branch starts from its own frontier)."""
    b = np.asarray(bounds, dtype=np.float64)
    return problem_from_csr(p.n_vars, p.n_cons, p.row_start, p.row_col, p.row_val, b[0::2].copy(),
                            b[1::2].copy(), p.is_integer, p.cons_lower, p.cons_upper,
                            name=p.name + "-presolved", apply_integral=False, validate=False)
