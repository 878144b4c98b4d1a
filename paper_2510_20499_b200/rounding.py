"""Python mirror of the reference fix-and-propagate API (pulse/rounding.hpp), on the GPU driver.

* ``RoundingConfig`` (rounding.hpp:18-31), ``RoundingOutcome`` (:347-355)
* ``initial_sort`` (:35-65) and ``get_bulk_size`` (:119-123) (host helpers)
* ``propagation_round`` (:393-558): the whole bulk loop runs in libbp's driver with device-resident
  bounds; the host RNG stream is the reference's (std::mt19937_64(seed)).
* ``repair`` (:234-311): device activity sweeps + most-violated-row scan, host shift choice

``lp_polish`` (PDHG) is out of scope: ``propagation_round`` returns the point the reference would
polish, and ``outcome.bounds_feasible`` tells whether it would.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .problem import ProblemDef
from .probing import ProbingCache
from .propagation import device_problem


@dataclass
class RoundingConfig:
    random_band: float = 0.25
    single_var_tail: int = 36
    repair_enabled: bool = False
    repair_attempt_cap: int = 16
    repair_shift_cap: int = 64


@dataclass
class RoundingOutcome:
    values: np.ndarray
    rounding_infeasible: bool
    timed_out: bool
    completed: bool
    repair_attempts: int
    bulks_committed: int
    set_count: int
    bounds_feasible: bool
    bp_calls: int
    device_ms: float


def initial_sort(p: ProblemDef, values) -> list:
    """rounding.hpp:35-65 (stable: width class, then distance to the nearest integer)."""
    items = []
    for i in range(p.n_vars):
        if not p.is_integer[i]:
            continue
        w = p.var_upper[i] - p.var_lower[i]
        cls = 0 if w == 1.0 else (1 if w == 2.0 else 2)
        v = float(values[i])
        items.append((cls, abs(v - _round_half_away(v)), i))
    items.sort(key=lambda t: (t[0], t[1]))  # Python's sort is stable
    return [t[2] for t in items]


def _round_half_away(v: float) -> float:
    """std::round (half away from zero)."""
    return math.copysign(math.floor(abs(v) + 0.5), v)


def get_bulk_size(remaining: int, recovery: bool, single_var_tail: int = 36) -> int:
    """rounding.hpp:119-123 (std::lround: half away from zero)."""
    if recovery or remaining <= single_var_tail:
        return 1
    return int(_round_half_away(math.sqrt(float(remaining))))


def _config(cfg: RoundingConfig | None):
    cfg = cfg or RoundingConfig()
    c = _lib.bp_rounding_config()
    _lib.lib().bp_rounding_config_default(C.byref(c))
    c.random_band = cfg.random_band
    c.single_var_tail = cfg.single_var_tail
    c.repair_enabled = 1 if cfg.repair_enabled else 0
    c.repair_attempt_cap = cfg.repair_attempt_cap
    c.repair_shift_cap = cfg.repair_shift_cap
    return c


@dataclass
class RepairResult:
    """rounding.hpp:225-228."""
    values: list              # [(var, value)] in the input order
    bounds: "object"          # BoundsState


def repair(p: ProblemDef, fixed, deadline_sec: float = math.inf,
           cfg: RoundingConfig | None = None, plan=None) -> RepairResult | None:
    """rounding.hpp:234-311 on the engine: None where the reference returns std::nullopt. The
    plan argument is accepted for signature parity only."""
    from .propagation import BoundsState
    dp = device_problem(p)
    c = _config(cfg)
    fv = np.ascontiguousarray([v for v, _ in fixed], dtype=np.int32)
    fx = np.ascontiguousarray([x for _, x in fixed], dtype=np.float64)
    out = np.zeros(max(len(fixed), 1))
    b = np.zeros(max(2 * p.n_vars, 1))
    ok = C.c_int32(0)
    dl = 0.0 if not math.isfinite(deadline_sec) else float(deadline_sec)
    _lib.check(_lib.lib().bp_repair(dp.h, _lib.ptr(fv), _lib.ptr(fx), len(fixed), dl, C.byref(c),
                                    C.byref(ok), _lib.ptr(out), _lib.ptr(b)))
    if not ok.value:
        return None
    return RepairResult([(int(v), float(out[j])) for j, (v, _) in enumerate(fixed)],
                        BoundsState(raw=b[: 2 * p.n_vars]))


def propagation_round(p: ProblemDef, start_values, cache: ProbingCache | None, seed: int,
                      deadline_sec: float = math.inf, cfg: RoundingConfig | None = None) -> RoundingOutcome:
    """rounding.hpp:393 with Rng(seed) and Deadline(deadline_sec) (inf = never)."""
    dp = device_problem(p)
    L = _lib.lib()
    c = _config(cfg)
    sv = np.ascontiguousarray(start_values, dtype=np.float64)
    out = np.zeros(max(p.n_vars, 1))
    o = _lib.bp_rounding_outcome()
    dl = 0.0 if not math.isfinite(deadline_sec) else float(deadline_sec)
    _lib.check(L.bp_propagation_round(dp.h, _lib.ptr(sv), cache.h if cache is not None else None,
                                      C.c_uint64(seed), dl, C.byref(c), _lib.ptr(out), C.byref(o)))
    return RoundingOutcome(out[: p.n_vars], bool(o.rounding_infeasible), bool(o.timed_out),
                           bool(o.completed), int(o.repair_attempts), int(o.bulks_committed),
                           int(o.set_count), bool(o.bounds_feasible), int(o.bp_calls),
                           float(o.device_ms))


@dataclass
class ProbeResult:
    """rounding.hpp:154-159."""
    bounds: "object"          # BoundsState
    infeas_count: int
    evicted: list
    fixed: list               # [(var, value)]


def parallel_propagate(p: ProblemDef, base, vars_, probe_vec_0, probe_vec_1,
                       cache: ProbingCache | None = None, plan=None):
    """rounding.hpp:213-224 (both probes of detail::run_probe, :167-207, on the engine). Returns
    the pair of ProbeResult; the plan argument is accepted for signature parity only."""
    from .propagation import BoundsState
    dp = device_problem(p)
    L = _lib.lib()
    n, k = p.n_vars, len(vars_)
    if len(probe_vec_0) != k or len(probe_vec_1) != k:
        raise ValueError("candidate vector size mismatch")
    vv = np.ascontiguousarray(vars_, dtype=np.int32)
    a = np.ascontiguousarray(probe_vec_0, dtype=np.float64)
    b = np.ascontiguousarray(probe_vec_1, dtype=np.float64)
    out = np.zeros(max(4 * n, 1))
    inf, cnt, nev, nfx = (np.zeros(2, dtype=np.int32) for _ in range(4))
    ev = np.zeros(max(2 * k, 1), dtype=np.int32)
    fv = np.zeros(max(2 * k, 1), dtype=np.int32)
    fx = np.zeros(max(2 * k, 1))
    base_raw = np.ascontiguousarray(base.raw(), dtype=np.float64)
    _lib.check(L.bp_parallel_propagate(dp.h, _lib.ptr(base_raw), 1 if base.infeasible() else 0,
                                       _lib.ptr(vv), k, _lib.ptr(a), _lib.ptr(b),
                                       cache.h if cache is not None else None, _lib.ptr(out),
                                       _lib.ptr(inf), _lib.ptr(cnt), _lib.ptr(ev), _lib.ptr(nev),
                                       _lib.ptr(fv), _lib.ptr(fx), _lib.ptr(nfx)))
    res = []
    for q in range(2):
        bs = BoundsState(raw=out[2 * n * q: 2 * n * (q + 1)], infeasible=bool(inf[q]))
        res.append(ProbeResult(bs, int(cnt[q]), ev[k * q: k * q + nev[q]].tolist(),
                               [(int(fv[k * q + j]), float(fx[k * q + j])) for j in range(nfx[q])]))
    return res
