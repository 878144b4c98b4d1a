"""PDHG products on the device: the Python mirror of ``pulse::LpInstance`` (lp.hpp:17-47) and of
``lpdetail::spmv_rows`` / ``spmv_cols`` (lp.hpp:74-102), plus the solver's inner iteration
(lp.hpp:315-340) with fixed step sizes, all through the C-ABI (``bp_lp_*``, ``bp_lp.cu``).
Results are bit-identical to the reference's (16384-entry segment sums, no FMA)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .problem import ProblemDef


@dataclass
class LpInstance:
    n_vars: int
    n_rows: int
    obj: np.ndarray
    row_start: np.ndarray
    row_col: np.ndarray
    row_val: np.ndarray
    col_start: np.ndarray
    col_row: np.ndarray
    col_val: np.ndarray
    row_lower: np.ndarray
    row_upper: np.ndarray
    var_lower: np.ndarray
    var_upper: np.ndarray

    @classmethod
    def relax(cls, p: ProblemDef) -> "LpInstance":
        """lp.hpp:28-46."""
        return cls(p.n_vars, p.n_cons, p.obj_coeffs, p.row_start, p.row_col, p.row_val, p.col_start,
                   p.col_row, p.col_val, p.cons_lower, p.cons_upper, p.var_lower, p.var_upper)


class DeviceLp:
    """Owning handle of a device LP instance (bp_lp_create)."""

    def __init__(self, s: LpInstance, device: int | None = None):
        from .propagation import default_device
        device = default_device() if device is None else device
        f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
        self._keep = [i32(s.row_start), i32(s.row_col), f64(s.row_val), i32(s.col_start),
                      i32(s.col_row), f64(s.col_val), f64(s.obj), f64(s.row_lower), f64(s.row_upper),
                      f64(s.var_lower), f64(s.var_upper)]
        P = _lib.ptr
        d = _lib.bp_lp_desc(s.n_vars, s.n_rows, *[P(a) for a in self._keep])
        h = C.c_void_p()
        _lib.check(_lib.lib().bp_lp_create(C.byref(d), int(device), C.byref(h)))
        self.h = h
        self.n, self.m = s.n_vars, s.n_rows

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib._lib is not None:
                _lib._lib.bp_lp_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def spmv_rows(self, x) -> np.ndarray:
        """lp.hpp:74-87."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(max(self.m, 1))
        _lib.check(_lib.lib().bp_lp_spmv_rows(self.h, _lib.ptr(x), _lib.ptr(out)))
        return out[: self.m]

    def spmv_cols(self, y) -> np.ndarray:
        """lp.hpp:89-102."""
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros(max(self.n, 1))
        _lib.check(_lib.lib().bp_lp_spmv_cols(self.h, _lib.ptr(y), _lib.ptr(out)))
        return out[: self.n]

    def pdhg_iterate(self, x, y, x_bar, x_sum, y_sum, tau: float, sigma: float, iters: int):
        """lp.hpp:315-340, `iters` times; returns the updated (x, y, x_bar, x_sum, y_sum)."""
        v = [np.array(a, dtype=np.float64, copy=True) for a in (x, y, x_bar, x_sum, y_sum)]
        _lib.check(_lib.lib().bp_lp_pdhg_iterate(self.h, *[_lib.ptr(a) for a in v], float(tau),
                                                 float(sigma), int(iters)))
        return tuple(v)

    def evaluate_kkt(self, x, y) -> dict:
        """lp.hpp:134-206: residual maxima exact, objectives compensated (a few ulps from the
        reference's Neumaier sums)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros(7)
        _lib.check(_lib.lib().bp_lp_evaluate_kkt(self.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(out)))
        keys = ("primal_res", "dual_res", "gap", "primal_obj", "dual_obj", "x_norm", "score")
        return dict(zip(keys, (float(v) for v in out)))

    def last_ms(self) -> float:
        ms = C.c_double()
        _lib.check(_lib.lib().bp_lp_last_ms(self.h, C.byref(ms)))
        return ms.value
