"""Python mirror of the reference propagation API (pulse/propagation.hpp), backed by the GPU engine.

Same names, argument meaning and error behaviour as the reference:

* ``BoundsState`` (propagation.hpp:19-69): interleaved ``b[2i] = lo, b[2i+1] = up`` + infeasible flag;
* ``ActivityState`` (:74-93); ``WorkPlan`` / ``size_class_of`` / ``build_work_plan`` (:97-141);
* ``compute_activities`` (:226), ``tighten_bounds`` (:378), ``propagate`` (:418);
* ``PropagationLimits`` / ``PropagationStatus`` / ``PropagationResult`` (:253-267).

Every compute call goes through libbp.so (C-ABI, include/bp.h) on the GPU; there is no CPU path.
The device copy of a ProblemDef is created on first use and cached on the object (one upload per
ProblemDef, SURVEY §3 "Problem upload, once per ProblemDef").
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .problem import ProblemDef

K_INF = math.inf


class PropagationStatus(enum.IntEnum):
    Tightened = 0
    Infeasible = 1
    Unchanged = 2


@dataclass
class PropagationLimits:
    max_rounds: int = 64
    time_limit: float = math.inf
    abs_threshold: float = 1e-7
    rel_threshold: float = 1e-4
    incremental: bool = True


@dataclass
class PropagationResult:
    status: PropagationStatus = PropagationStatus.Unchanged
    rounds: int = 0
    crossed_vars: int = 0


class BoundsState:
    """Interleaved variable bounds (propagation.hpp:19-69)."""

    def __init__(self, p: ProblemDef | None = None, raw: np.ndarray | None = None,
                 infeasible: bool = False):
        if raw is not None:
            self.b = np.ascontiguousarray(raw, dtype=np.float64).copy()
        elif p is not None:
            self.b = p.root_bounds()
        else:
            self.b = np.zeros(0, dtype=np.float64)
        self._infeasible = bool(infeasible)

    def n_vars(self):
        return self.b.size // 2

    def lower(self, i):
        return float(self.b[2 * i])

    def upper(self, i):
        return float(self.b[2 * i + 1])

    def set_lower(self, i, v):
        self.b[2 * i] = v

    def set_upper(self, i, v):
        self.b[2 * i + 1] = v

    def fix(self, i, v):
        self.b[2 * i] = v
        self.b[2 * i + 1] = v

    def fixed(self, i):
        return bool(self.b[2 * i] == self.b[2 * i + 1])

    def width(self, i):
        return float(self.b[2 * i + 1] - self.b[2 * i])

    def infeasible(self):
        return self._infeasible

    def mark_infeasible(self):
        self._infeasible = True

    def clear_infeasible(self):
        self._infeasible = False

    def meet(self, other: "BoundsState"):
        """propagation.hpp:49-56 (std::max/std::min keep the first operand on ties)."""
        lo, up = self.b[0::2], self.b[1::2]
        olo, oup = other.b[0::2], other.b[1::2]
        self.b[0::2] = np.where(lo < olo, olo, lo)
        self.b[1::2] = np.where(oup < up, oup, up)
        if np.any(self.b[0::2] > self.b[1::2]):
            self._infeasible = True

    def raw(self):
        return self.b

    def copy(self):
        return BoundsState(raw=self.b, infeasible=self._infeasible)

    def __eq__(self, o):
        return (isinstance(o, BoundsState) and self.b.size == o.b.size
                and bool(np.all(self.b == o.b)) and self._infeasible == o._infeasible)


@dataclass
class ActivityState:
    """propagation.hpp:74-93."""

    act: np.ndarray = field(default_factory=lambda: np.zeros(0))
    n_inf_min: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int32))
    n_inf_max: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int32))

    def resize(self, n_cons):
        self.act = np.zeros(2 * n_cons, dtype=np.float64)
        self.n_inf_min = np.zeros(n_cons, dtype=np.int32)
        self.n_inf_max = np.zeros(n_cons, dtype=np.int32)

    def min_unbounded(self, k):
        return self.n_inf_min[k] > 0

    def max_unbounded(self, k):
        return self.n_inf_max[k] > 0

    def min_activity(self, k):
        return -K_INF if self.min_unbounded(k) else float(self.act[2 * k])

    def max_activity(self, k):
        return K_INF if self.max_unbounded(k) else float(self.act[2 * k + 1])

    def min_finite_part(self, k):
        return float(self.act[2 * k])

    def max_finite_part(self, k):
        return float(self.act[2 * k + 1])


@dataclass
class WorkPlanBin:
    size_class: int
    items: list


@dataclass
class WorkPlan:
    """propagation.hpp:97-109. The GPU engine builds its own warp-oriented partition at upload;
    the plan is accepted for API compatibility and never changes results (the reference's own
    binning is also result-neutral, test_propagation.cpp:244-262)."""

    row_bins: list = field(default_factory=list)
    var_bins: list = field(default_factory=list)
    kHeavyNnz = 16384
    kSmallNnz = 32


def size_class_of(nnz: int) -> int:
    """propagation.hpp:111-121: ceil(log2(nnz)), 0 for nnz <= 1."""
    if nnz <= 1:
        return 0
    return int(nnz - 1).bit_length()


def build_work_plan(p: ProblemDef) -> WorkPlan:
    """propagation.hpp:123-141."""
    plan = WorkPlan()
    for bins, counts in ((plan.row_bins, np.diff(p.row_start)), (plan.var_bins, np.diff(p.col_start))):
        by = {}
        for k, c in enumerate(counts):
            by.setdefault(size_class_of(int(c)), []).append(k)
        for c in sorted(by):
            bins.append(WorkPlanBin(c, by[c]))
    return plan


class DeviceProblem:
    """Owning handle of the device-resident problem (bp_problem_create)."""

    def __init__(self, p: ProblemDef, device: int = 0):
        L = _lib.lib()
        self.p = p
        self._keep = [np.ascontiguousarray(a) for a in (
            p.row_start, p.row_col, p.row_val, p.col_start, p.col_row, p.col_val,
            p.var_lower, p.var_upper, p.is_integer, p.cons_lower, p.cons_upper)]
        a = self._keep
        d = _lib.bp_problem_desc(p.n_vars, p.n_cons, *[_lib.ptr(x) for x in a])
        h = C.c_void_p()
        _lib.check(L.bp_problem_create(C.byref(d), int(device), C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def adopt(cls, p: ProblemDef, handle: C.c_void_p, device: int = 0) -> "DeviceProblem":
        """Wraps a handle created elsewhere (bp_build_problem) for problem p."""
        dp = cls.__new__(cls)
        dp.p = p
        dp._keep = []
        dp.h = handle
        dp.device = device
        return dp

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib._lib is not None:
                _lib._lib.bp_problem_destroy(self.h)
                self.h = None
        except Exception:
            pass


_DEFAULT_DEVICE = 0


def set_device(device: int) -> None:
    """GPU for problems uploaded from now on (pulse_gpu.hpp's set_device): one process per GPU
    calls it with its local rank."""
    global _DEFAULT_DEVICE
    _DEFAULT_DEVICE = int(device)


def default_device() -> int:
    return _DEFAULT_DEVICE


def device_problem(p: ProblemDef, device: int | None = None) -> DeviceProblem:
    """The device copy of p: the one already attached when no device is named, else uploaded to
    `device` (default: set_device's)."""
    dp = getattr(p, "_device_handle", None)
    if device is None:
        if dp is not None:
            return dp
        device = _DEFAULT_DEVICE
    if dp is None or dp.device != device:
        dp = DeviceProblem(p, device)
        p._device_handle = dp
    return dp


def compute_activities(p: ProblemDef, b: BoundsState, rows, a: ActivityState, plan=None):
    """pulse::compute_activities (propagation.hpp:226). ``rows=None`` recomputes every row."""
    if a.n_inf_min.size != p.n_cons:
        a.resize(p.n_cons)
    dp = device_problem(p)
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    _lib.check(_lib.lib().bp_compute_activities(
        dp.h, _lib.ptr(b.b), _lib.ptr(r), -1 if r is None else int(r.size),
        _lib.ptr(a.act), _lib.ptr(a.n_inf_min), _lib.ptr(a.n_inf_max)))


def tighten_bounds(p: ProblemDef, b: BoundsState, a: ActivityState, vars_, lim: PropagationLimits,
                   crossed_out: list | None = None, plan=None) -> list:
    """pulse::tighten_bounds (propagation.hpp:378): returns the changed vars ascending."""
    dp = device_problem(p)
    v = None if vars_ is None else np.ascontiguousarray(vars_, dtype=np.int32)
    changed = np.zeros(max(p.n_vars, 1), dtype=np.int32)
    nch = C.c_int32(0)
    crossed = C.c_int32(0)
    inf = C.c_int32(1 if b.infeasible() else 0)
    ls = _lib.limits_struct(lim)
    _lib.check(_lib.lib().bp_tighten_bounds(
        dp.h, _lib.ptr(b.b), C.byref(inf), _lib.ptr(a.act), _lib.ptr(a.n_inf_min),
        _lib.ptr(a.n_inf_max), _lib.ptr(v), -1 if v is None else int(v.size), C.byref(ls),
        _lib.ptr(changed), C.byref(nch), C.byref(crossed)))
    if inf.value:
        b.mark_infeasible()
    if crossed_out is not None:
        crossed_out.clear()
        crossed_out.append(int(crossed.value))
    return [int(x) for x in changed[: nch.value]]


def propagate(p: ProblemDef, b: BoundsState, lim: PropagationLimits | None = None,
              plan=None) -> PropagationResult:
    """pulse::propagate (propagation.hpp:418), in place on ``b``."""
    dp = device_problem(p)
    inf = C.c_int32(1 if b.infeasible() else 0)
    res = _lib.bp_result()
    ls = _lib.limits_struct(lim)
    _lib.check(_lib.lib().bp_propagate(dp.h, _lib.ptr(b.b), C.byref(inf), C.byref(ls), C.byref(res)))
    if inf.value:
        b.mark_infeasible()
    return PropagationResult(PropagationStatus(res.status), int(res.rounds), int(res.crossed_vars))


FORCE_FRONTIER = 1


def propagate_device(p: ProblemDef, d_bounds_ptr: int, infeasible: bool = False,
                     lim: PropagationLimits | None = None, stream_ptr: int = 0, flags: int = 0,
                     d_stats_ptr: int = 0):
    """Device-resident variant: ``d_bounds_ptr`` is a device pointer to 2n doubles (e.g. a torch
    tensor's ``data_ptr()``). ``flags``/``d_stats_ptr`` as bp_propagate_ex.
    Returns (PropagationResult, infeasible)."""
    dp = device_problem(p)
    inf = C.c_int32(1 if infeasible else 0)
    res = _lib.bp_result()
    ls = _lib.limits_struct(lim)
    _lib.check(_lib.lib().bp_propagate_ex(dp.h, C.c_void_p(d_bounds_ptr), C.byref(inf),
                                          C.byref(ls), C.byref(res),
                                          C.c_void_p(stream_ptr) if stream_ptr else None,
                                          int(flags), C.c_void_p(d_stats_ptr) if d_stats_ptr else None))
    return PropagationResult(PropagationStatus(res.status), int(res.rounds),
                             int(res.crossed_vars)), bool(inf.value)
