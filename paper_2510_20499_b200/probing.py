"""Python mirror of the reference probing API (pulse/probing.hpp), backed by the GPU engine.

* ``BranchKind`` / ``BranchSpec`` / ``make_branch_spec`` (probing.hpp:21-60)
* ``BoundDelta`` / ``ProbeBranch`` / ``ProbeEntry`` / ``ProbingCache`` (:62-98)
* ``prioritize_probe_vars`` (:105), ``probe_variable`` (:225), ``build_cache`` (:243),
  ``assemble_bulk_warm_start`` (:292)
* ``probe_variables``: the batched entry point (all branches of many variables in one launch).

A ProbingCache wraps the engine's packed cache (C-ABI ``bp_cache``); entries are materialised
on access. ``pack`` / ``merge_packed`` serialise cache slices for the multi-GPU gather.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .problem import ProblemDef
from .propagation import BoundsState, WorkPlan, device_problem


class BranchKind(enum.IntEnum):
    BoxedSplit = 0
    AtLowerBound = 1
    AtUpperBound = 2


@dataclass
class BranchSpec:
    var: int = -1
    kind: BranchKind = BranchKind.BoxedSplit
    down_lower: float = 0.0
    down_upper: float = 0.0
    up_lower: float = 0.0
    up_upper: float = 0.0


def make_branch_spec(root: BoundsState, v: int):
    """probing.hpp:30-60 (follow the code, not SPEC.md:229: mid = ceil((l+u)/2))."""
    lo, up = root.lower(v), root.upper(v)
    if lo == up:
        return None
    if math.isfinite(lo) and math.isfinite(up):
        mid = math.ceil((lo + up) / 2.0)
        return BranchSpec(v, BranchKind.BoxedSplit, lo, mid - 1.0, float(mid), up)
    if math.isfinite(lo):
        return BranchSpec(v, BranchKind.AtLowerBound, lo, lo, lo + 1.0, up)
    if math.isfinite(up):
        return BranchSpec(v, BranchKind.AtUpperBound, lo, up - 1.0, up, up)
    return None


@dataclass
class BoundDelta:
    var: int
    new_lower: float
    new_upper: float


@dataclass
class ProbeBranch:
    feasible: bool = True
    branch_lower: float = 0.0
    branch_upper: float = 0.0
    deltas: list = field(default_factory=list)


@dataclass
class ProbeEntry:
    var: int = -1
    kind: BranchKind = BranchKind.BoxedSplit
    down: ProbeBranch = field(default_factory=ProbeBranch)
    up: ProbeBranch = field(default_factory=ProbeBranch)
    forces_down: bool = False
    forces_up: bool = False


class ProbingCache:
    """probing.hpp:87-98 over the engine's packed cache."""

    def __init__(self, handle: C.c_void_p):
        self.h = handle
        n = C.c_int32()
        npb = C.c_int32()
        ninf = C.c_int32()
        nd = C.c_int64()
        nfb = C.c_int32()
        cert = C.c_int32()
        ms = C.c_double()
        _lib.check(_lib.lib().bp_cache_info(self.h, C.byref(n), C.byref(npb), C.byref(ninf),
                                            C.byref(nd), C.byref(nfb), C.byref(cert), C.byref(ms)))
        self.n_vars = n.value
        self.n_probed = npb.value
        self.n_infeasible_branches = ninf.value
        self.n_deltas = nd.value
        self.n_fallback = nfb.value
        self.certified = bool(cert.value)
        self.probe_ms = ms.value
        nb = C.c_int32()
        _lib.check(_lib.lib().bp_cache_block_branches(self.h, C.byref(nb)))
        self.n_block = nb.value  # branches run by the block-per-branch kernel
        wk = np.zeros(5, np.int64)
        _lib.check(_lib.lib().bp_cache_work(self.h, _lib.ptr(wk)))
        # Σ over branches and rounds of |R|, row nnz of R, |V|, col nnz of V, |C|
        self.work = [int(x) for x in wk]
        self._root = None
        self._memo = {}

    @property
    def root(self) -> BoundsState:
        """probing.hpp:96 (materialised on first access: a 16n-byte copy)."""
        if self._root is None:
            r = np.zeros(2 * self.n_vars)
            _lib.check(_lib.lib().bp_cache_root(self.h, _lib.ptr(r)))
            self._root = BoundsState(raw=r)
        return self._root

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib._lib is not None:
                _lib._lib.bp_cache_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def refresh(self):
        self.__init__(self.h)

    def has(self, v: int) -> bool:
        if v < 0 or v >= self.n_vars:
            return False
        return self._entry_raw(v) is not None

    def _entry_raw(self, v):
        present = C.c_int32()
        hdr = np.zeros(7, np.int32)
        br = np.zeros(4)
        _lib.check(_lib.lib().bp_cache_entry(self.h, int(v), C.byref(present), _lib.ptr(hdr),
                                             _lib.ptr(br)))
        return (hdr, br) if present.value else None

    def deltas(self, v: int, side: int):
        """(vars, lo, up) arrays of one branch."""
        raw = self._entry_raw(v)
        if raw is None:
            raise IndexError(f"var {v} has no cache entry")
        cnt = int(raw[0][5 + side])
        vv = np.zeros(max(cnt, 1), np.int32)
        lo = np.zeros(max(cnt, 1))
        up = np.zeros(max(cnt, 1))
        _lib.check(_lib.lib().bp_cache_deltas(self.h, int(v), int(side), _lib.ptr(vv), _lib.ptr(lo),
                                              _lib.ptr(up)))
        return vv[:cnt], lo[:cnt], up[:cnt]

    def at(self, v: int) -> ProbeEntry:
        if v in self._memo:
            return self._memo[v]
        raw = self._entry_raw(v)
        if raw is None:
            raise IndexError(f"var {v} has no cache entry")
        hdr, br = raw
        branches = []
        for side in range(2):
            vv, lo, up = self.deltas(v, side)
            branches.append(ProbeBranch(bool(hdr[3 + side]), float(br[2 * side]), float(br[2 * side + 1]),
                                        [BoundDelta(int(a), float(b), float(c)) for a, b, c in zip(vv, lo, up)]))
        e = ProbeEntry(int(v), BranchKind(int(hdr[0])), branches[0], branches[1], bool(hdr[1]),
                       bool(hdr[2]))
        self._memo[v] = e
        return e

    # ---- multi-GPU gather support
    def pack(self) -> np.ndarray:
        nb = C.c_int64()
        _lib.check(_lib.lib().bp_cache_pack_size(self.h, C.byref(nb)))
        buf = np.zeros(nb.value, np.uint8)
        _lib.check(_lib.lib().bp_cache_pack(self.h, _lib.ptr(buf), nb.value))
        return buf

    def merge_packed(self, buf: np.ndarray):
        buf = np.ascontiguousarray(buf, dtype=np.uint8)
        _lib.check(_lib.lib().bp_cache_merge_packed(self.h, _lib.ptr(buf), buf.size))
        self._memo.clear()
        self.refresh()

    @classmethod
    def empty(cls, root: BoundsState) -> "ProbingCache":
        h = C.c_void_p()
        _lib.check(_lib.lib().bp_cache_create_empty(root.n_vars(), _lib.ptr(root.b), C.byref(h)))
        return cls(h)


def prioritize_probe_vars(p: ProblemDef) -> list:
    """probing.hpp:105-190."""
    dp = device_problem(p)
    order = np.zeros(max(p.n_vars, 1), np.int32)
    n = C.c_int32()
    _lib.check(_lib.lib().bp_prioritize_probe_vars(dp.h, _lib.ptr(order), C.byref(n)))
    return [int(x) for x in order[: n.value]]


def probe_variables(p: ProblemDef, root: BoundsState | None, vars_) -> ProbingCache:
    """Batched double probing of ``vars_`` from ``root`` (None = original bounds)."""
    dp = device_problem(p)
    v = np.ascontiguousarray(vars_, dtype=np.int32)
    h = C.c_void_p()
    _lib.check(_lib.lib().bp_probe_variables(dp.h, None if root is None else _lib.ptr(root.b),
                                             _lib.ptr(v), int(v.size), C.byref(h)))
    return ProbingCache(h)


def probe_variable(p: ProblemDef, root: BoundsState, v: int, plan: WorkPlan | None = None) -> ProbeEntry:
    """probing.hpp:225-238."""
    return probe_variables(p, root, [v]).at(v)


def build_cache(p: ProblemDef, budget_sec: float) -> ProbingCache:
    """probing.hpp:243-281."""
    dp = device_problem(p)
    h = C.c_void_p()
    _lib.check(_lib.lib().bp_build_cache(dp.h, float(budget_sec), C.byref(h)))
    return ProbingCache(h)


def build_cache_multi(p: ProblemDef, devices, vars_=None, budget_sec: float = 1e9):
    """pulse::build_cache (probing.hpp:243-281) over several GPUs of this process
    (bp_build_cache_multi): the problem is replicated on every device, device d probes positions
    d, d + G, ... of the candidate list (``vars_``, or build_cache's priority order under
    ``budget_sec``), and the packed slices are gathered to ``devices[0]`` with NCCL send/recv and
    merged there. Returns (ProbingCache, per-device probe-kernel ms)."""
    from .propagation import DeviceProblem
    devices = [int(d) for d in devices]
    reps = [device_problem(p, devices[0])] + [DeviceProblem(p, d) for d in devices[1:]]
    hs = (C.c_void_p * len(reps))(*[r.h for r in reps])
    v = None if vars_ is None else np.ascontiguousarray(vars_, dtype=np.int32)
    ms = np.zeros(len(reps))
    h = C.c_void_p()
    _lib.check(_lib.lib().bp_build_cache_multi(hs, len(reps), float(budget_sec), _lib.ptr(v),
                                               -1 if v is None else int(v.size), C.byref(h),
                                               _lib.ptr(ms)))
    return ProbingCache(h), ms.tolist()


@dataclass
class BulkWarmStart:
    bounds: BoundsState
    conflicts: list
    evicted: list


def assemble_bulk_warm_start(cache: ProbingCache, assignments) -> BulkWarmStart:
    """probing.hpp:292-352."""
    vars_ = np.ascontiguousarray([a[0] for a in assignments], dtype=np.int32)
    vals = np.ascontiguousarray([a[1] for a in assignments], dtype=np.float64)
    n = cache.n_vars
    b = np.zeros(2 * n)
    conf = np.zeros(2 * max(len(vars_), 1), np.int32)
    ev = np.zeros(max(len(vars_), 1), np.int32)
    nc = C.c_int32()
    ne = C.c_int32()
    _lib.check(_lib.lib().bp_assemble_bulk_warm_start(cache.h, _lib.ptr(vars_), _lib.ptr(vals),
                                                      int(vars_.size), _lib.ptr(b), _lib.ptr(conf),
                                                      C.byref(nc), _lib.ptr(ev), C.byref(ne)))
    conflicts = [(int(conf[2 * j]), int(conf[2 * j + 1])) for j in range(nc.value)]
    return BulkWarmStart(BoundsState(raw=b), conflicts, [int(x) for x in ev[: ne.value]])
