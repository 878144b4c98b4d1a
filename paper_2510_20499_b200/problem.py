"""Host-side problem model: the Python mirror of ``pulse::ProblemDef`` / ``pulse::ProblemBuilder``.

Reference: /root/reference/proj/include/pulse/problem.hpp:25-84 (ProblemDef) and :102-243
(ProblemBuilder).  ``ProblemBuilder.build`` reproduces ``ProblemBuilder::build`` (problem.hpp:141-227):

* integral tightening of integer-variable bounds with ``ceil(lb - 1e-9)`` / ``floor(ub + 1e-9)``
  (so an integer lower bound of 0 becomes ``-0.0``, exactly like the reference);
* ``runtime_error`` on an empty variable domain or crossed row bounds, ``out_of_range`` on bad
  entry indices (raised here as ``RuntimeError`` / ``IndexError``);
* entries sorted by (row, col), duplicate (row, col) pairs coalesced by summation, explicit
  zeros dropped;
* CSC by a stable transpose of the CSR (columns list their rows ascending).

The reference sorts with ``std::sort`` (not stable), so the summation order of duplicate entries
is unspecified there; here duplicates are summed in insertion order.  Integer-valued duplicates
(the only kind the reference's tests use) sum identically in any order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

K_INF = math.inf
K_INF_THRESHOLD = 1e20  # common.hpp:17
K_SUM_SEGMENT = 16384  # problem.hpp:274


@dataclass
class ProblemDef:
    """Immutable sparse MILP (problem.hpp:25-84), CSR + CSC views as numpy arrays."""

    n_vars: int
    n_cons: int
    obj_coeffs: np.ndarray
    var_lower: np.ndarray
    var_upper: np.ndarray
    is_integer: np.ndarray  # uint8
    row_start: np.ndarray  # int32, n_cons + 1
    row_col: np.ndarray  # int32
    row_val: np.ndarray  # float64
    col_start: np.ndarray  # int32, n_vars + 1
    col_row: np.ndarray  # int32
    col_val: np.ndarray  # float64
    cons_lower: np.ndarray
    cons_upper: np.ndarray
    name: str = ""
    var_names: list = field(default_factory=list)
    cons_names: list = field(default_factory=list)

    def nnz(self) -> int:
        return int(self.row_col.shape[0])

    def row_nnz(self, k: int) -> int:
        return int(self.row_start[k + 1] - self.row_start[k])

    def col_nnz(self, i: int) -> int:
        return int(self.col_start[i + 1] - self.col_start[i])

    def row_cols(self, k: int) -> np.ndarray:
        return self.row_col[self.row_start[k] : self.row_start[k + 1]]

    def row_vals(self, k: int) -> np.ndarray:
        return self.row_val[self.row_start[k] : self.row_start[k + 1]]

    def col_rows(self, i: int) -> np.ndarray:
        return self.col_row[self.col_start[i] : self.col_start[i + 1]]

    def col_vals(self, i: int) -> np.ndarray:
        return self.col_val[self.col_start[i] : self.col_start[i + 1]]

    def var_fixed(self, i: int) -> bool:
        return bool(self.var_lower[i] == self.var_upper[i])

    def integer_vars(self) -> np.ndarray:
        return np.nonzero(self.is_integer)[0].astype(np.int32)

    def root_bounds(self) -> np.ndarray:
        """Interleaved original bounds, the layout of BoundsState(p) (propagation.hpp:22-29)."""
        b = np.empty(2 * self.n_vars, dtype=np.float64)
        b[0::2] = self.var_lower
        b[1::2] = self.var_upper
        return b


def csc_from_csr(n_vars: int, row_start, row_col, row_val):
    """Stable transpose (problem.hpp:211-225): entries of column i list their rows ascending."""
    n_cons = len(row_start) - 1
    rows = np.repeat(np.arange(n_cons, dtype=np.int64), np.diff(row_start))
    # (col, row) keys are unique, so any sort is the stable transpose
    order = np.argsort(np.asarray(row_col, dtype=np.int64) * max(n_cons, 1) + rows)
    counts = np.bincount(row_col, minlength=n_vars)
    col_start = np.zeros(n_vars + 1, dtype=np.int32)
    np.cumsum(counts, out=col_start[1:])
    return col_start, rows[order].astype(np.int32), np.asarray(row_val, dtype=np.float64)[order]


def round_integer_bounds(var_lower, var_upper, is_integer):
    """problem.hpp:157-163: ceil_eps(lb, 1e-9) / floor_eps(ub, 1e-9) on finite integer bounds."""
    lo = np.array(var_lower, dtype=np.float64, copy=True)
    up = np.array(var_upper, dtype=np.float64, copy=True)
    isint = np.asarray(is_integer).astype(bool)
    with np.errstate(invalid="ignore"):
        m = isint & np.isfinite(lo)
        lo[m] = np.ceil(lo[m] - 1e-9)
        m = isint & np.isfinite(up)
        up[m] = np.floor(up[m] + 1e-9)
    return lo, up


def problem_from_csr(n_vars, n_cons, row_start, row_col, row_val, var_lower, var_upper, is_integer,
                     cons_lower, cons_upper, obj=None, name="", apply_integral=True,
                     validate=True) -> ProblemDef:
    """ProblemDef from an already sorted/coalesced/zero-free CSR (the generators' output)."""
    row_start = np.ascontiguousarray(row_start, dtype=np.int32)
    row_col = np.ascontiguousarray(row_col, dtype=np.int32)
    row_val = np.ascontiguousarray(row_val, dtype=np.float64)
    is_integer = np.ascontiguousarray(is_integer, dtype=np.uint8)
    if apply_integral:
        var_lower, var_upper = round_integer_bounds(var_lower, var_upper, is_integer)
    var_lower = np.ascontiguousarray(var_lower, dtype=np.float64)
    var_upper = np.ascontiguousarray(var_upper, dtype=np.float64)
    cons_lower = np.ascontiguousarray(cons_lower, dtype=np.float64)
    cons_upper = np.ascontiguousarray(cons_upper, dtype=np.float64)
    if validate:
        bad = np.nonzero(var_lower > var_upper)[0]
        if bad.size:
            raise RuntimeError(f"variable 'x{bad[0]}' has empty domain after bound tightening")
        bad = np.nonzero(cons_lower > cons_upper)[0]
        if bad.size:
            raise RuntimeError(f"constraint 'c{bad[0]}' has crossed bounds")
    col_start, col_row, col_val = csc_from_csr(n_vars, row_start, row_col, row_val)
    return ProblemDef(
        n_vars=int(n_vars), n_cons=int(n_cons),
        obj_coeffs=np.zeros(n_vars) if obj is None else np.asarray(obj, dtype=np.float64),
        var_lower=var_lower, var_upper=var_upper, is_integer=is_integer,
        row_start=row_start, row_col=row_col, row_val=row_val,
        col_start=col_start, col_row=col_row, col_val=col_val,
        cons_lower=cons_lower, cons_upper=cons_upper, name=name)


class ProblemBuilder:
    """Mirror of pulse::ProblemBuilder (problem.hpp:102-243)."""

    def __init__(self):
        self._lo, self._up, self._int, self._obj, self._vn = [], [], [], [], []
        self._clo, self._cup, self._cn = [], [], []
        self._er, self._ec, self._ev = [], [], []
        self.name = ""

    def add_var(self, name, lower, upper, integer, obj=0.0) -> int:
        self._vn.append(name)
        self._lo.append(float(lower))
        self._up.append(float(upper))
        self._int.append(1 if integer else 0)
        self._obj.append(float(obj))
        return len(self._vn) - 1

    def add_row(self, name, lower, upper) -> int:
        self._cn.append(name)
        self._clo.append(float(lower))
        self._cup.append(float(upper))
        return len(self._cn) - 1

    def add_entry(self, row, col, val):
        self._er.append(int(row))
        self._ec.append(int(col))
        self._ev.append(float(val))

    def n_vars(self):
        return len(self._vn)

    def n_rows(self):
        return len(self._cn)

    def build(self) -> ProblemDef:
        n, m = self.n_vars(), self.n_rows()
        isint = np.array(self._int, dtype=np.uint8)
        lo, up = round_integer_bounds(np.array(self._lo), np.array(self._up), isint)
        bad = np.nonzero(lo > up)[0]
        if bad.size:
            raise RuntimeError(f"variable '{self._vn[bad[0]]}' has empty domain after bound tightening")
        clo, cup = np.array(self._clo, dtype=np.float64), np.array(self._cup, dtype=np.float64)
        bad = np.nonzero(clo > cup)[0]
        if bad.size:
            raise RuntimeError(f"constraint '{self._cn[bad[0]]}' has crossed bounds")
        er = np.array(self._er, dtype=np.int64)
        ec = np.array(self._ec, dtype=np.int64)
        ev = np.array(self._ev, dtype=np.float64)
        if er.size and (er.min() < 0 or er.max() >= m):
            raise IndexError("entry row out of range")
        if ec.size and (ec.min() < 0 or ec.max() >= n):
            raise IndexError("entry col out of range")
        order = np.lexsort((ec, er))  # stable
        er, ec, ev = er[order], ec[order], ev[order]
        if er.size:
            key = er * max(n, 1) + ec
            first = np.ones(er.size, dtype=bool)
            first[1:] = key[1:] != key[:-1]
            grp = np.cumsum(first) - 1
            vals = np.zeros(int(first.sum()), dtype=np.float64)
            for j in range(ev.size):  # sequential coalescing in sorted order
                vals[grp[j]] += ev[j]
            er, ec, ev = er[first], ec[first], vals
            keep = ev != 0.0
            er, ec, ev = er[keep], ec[keep], ev[keep]
        row_start = np.zeros(m + 1, dtype=np.int32)
        np.cumsum(np.bincount(er, minlength=m), out=row_start[1:])
        p = problem_from_csr(n, m, row_start, ec.astype(np.int32), ev, lo, up, isint, clo, cup,
                             obj=np.array(self._obj, dtype=np.float64), name=self.name,
                             apply_integral=False, validate=False)
        p.var_names = list(self._vn)
        p.cons_names = list(self._cn)
        return p


def build_on_device(b: ProblemBuilder, device: int | None = None) -> ProblemDef:
    """ProblemBuilder::build (problem.hpp:141-227) with every O(N log N) step on the GPU
    (bp_build_problem): the returned ProblemDef carries the device problem it was built into.
    Same results and error types as ``ProblemBuilder.build`` (duplicates summed in insertion
    order); messages name variables / rows by index."""
    import ctypes as C

    from . import _lib
    from .propagation import DeviceProblem, default_device
    device = default_device() if device is None else device
    n, m = b.n_vars(), b.n_rows()
    lo = np.ascontiguousarray(b._lo, dtype=np.float64)
    up = np.ascontiguousarray(b._up, dtype=np.float64)
    isint = np.ascontiguousarray(b._int, dtype=np.uint8)
    clo = np.ascontiguousarray(b._clo, dtype=np.float64)
    cup = np.ascontiguousarray(b._cup, dtype=np.float64)
    er = np.ascontiguousarray(b._er, dtype=np.int32)
    ec = np.ascontiguousarray(b._ec, dtype=np.int32)
    ev = np.ascontiguousarray(b._ev, dtype=np.float64)
    N = er.size
    P = _lib.ptr
    d = _lib.bp_builder_desc(n, m, N, P(er), P(ec), P(ev), P(lo), P(up), P(isint), P(clo), P(cup))
    rs = np.zeros(m + 1, np.int32)
    cs = np.zeros(n + 1, np.int32)
    rc_, rv = np.zeros(max(N, 1), np.int32), np.zeros(max(N, 1))
    cr, cv = np.zeros(max(N, 1), np.int32), np.zeros(max(N, 1))
    olo, oup = np.zeros(max(n, 1)), np.zeros(max(n, 1))
    out = _lib.bp_built(0, P(rs), P(rc_), P(rv), P(cs), P(cr), P(cv), P(olo), P(oup))
    h = C.c_void_p()
    # empty domain / crossed row: BPError (a RuntimeError); bad entry index: IndexError
    _lib.check(_lib.lib().bp_build_problem(C.byref(d), int(device), C.byref(out), C.byref(h)))
    nnz = int(out.nnz)
    p = ProblemDef(n_vars=n, n_cons=m, obj_coeffs=np.array(b._obj, dtype=np.float64),
                   var_lower=olo[:n].copy(), var_upper=oup[:n].copy(), is_integer=isint,
                   row_start=rs, row_col=rc_[:nnz].copy(), row_val=rv[:nnz].copy(),
                   col_start=cs, col_row=cr[:nnz].copy(), col_val=cv[:nnz].copy(),
                   cons_lower=clo, cons_upper=cup, name=b.name)
    p.var_names = list(b._vn)
    p.cons_names = list(b._cn)
    p._device_handle = DeviceProblem.adopt(p, h, device)
    return p


def make_problem(vars_spec, rows_spec) -> ProblemDef:
    """testkit::make_problem (tests/testkit.hpp:36-48): vars = [(lo, up, integer[, obj])],
    rows = [([(col, val), ...], lo, up)]."""
    b = ProblemBuilder()
    for i, v in enumerate(vars_spec):
        b.add_var(f"x{i}", v[0], v[1], bool(v[2]), v[3] if len(v) > 3 else 0.0)
    for k, (entries, lo, up) in enumerate(rows_spec):
        b.add_row(f"c{k}", lo, up)
        for col, val in entries:
            b.add_entry(k, col, val)
    return b.build()
