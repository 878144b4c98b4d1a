"""ctypes binding of the engine's C-ABI (include/bp.h) — the only way Python reaches the GPU.

The shared library is built in-tree (``paper_2510_20499_b200/libbp.so``) by ``__graft_entry__.build``
or ``make -C paper_2510_20499_b200/csrc``.  There is no CPU fallback: importing works without a
GPU, but every compute call fails loudly (``BPError``) when the library or a device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
# BP_LIB selects an alternative in-tree build of the same library (A/B experiments of build
# variants, e.g. a different occupancy target); default: the production build.
LIB_PATH = Path(os.environ["BP_LIB"]).resolve() if os.environ.get("BP_LIB") else _HERE / "libbp.so"

BP_OK, BP_ERR_INVALID_ARGUMENT, BP_ERR_OUT_OF_RANGE, BP_ERR_RUNTIME, BP_ERR_CUDA = 0, 1, 2, 3, 4
TIGHTENED, INFEASIBLE, UNCHANGED = 0, 1, 2


class BPError(RuntimeError):
    """Engine failure; ``code`` is the C-ABI error code."""

    def __init__(self, code, msg):
        super().__init__(f"[bp error {code}] {msg}")
        self.code = code


class bp_problem_desc(C.Structure):
    _fields_ = [
        ("n_vars", C.c_int32), ("n_cons", C.c_int32),
        ("row_start", C.c_void_p), ("row_col", C.c_void_p), ("row_val", C.c_void_p),
        ("col_start", C.c_void_p), ("col_row", C.c_void_p), ("col_val", C.c_void_p),
        ("var_lower", C.c_void_p), ("var_upper", C.c_void_p), ("is_integer", C.c_void_p),
        ("cons_lower", C.c_void_p), ("cons_upper", C.c_void_p),
    ]


class bp_builder_desc(C.Structure):
    _fields_ = [
        ("n_vars", C.c_int32), ("n_cons", C.c_int32), ("n_entries", C.c_int64),
        ("entry_row", C.c_void_p), ("entry_col", C.c_void_p), ("entry_val", C.c_void_p),
        ("var_lower", C.c_void_p), ("var_upper", C.c_void_p), ("is_integer", C.c_void_p),
        ("cons_lower", C.c_void_p), ("cons_upper", C.c_void_p),
    ]


class bp_built(C.Structure):
    _fields_ = [
        ("nnz", C.c_int64),
        ("row_start", C.c_void_p), ("row_col", C.c_void_p), ("row_val", C.c_void_p),
        ("col_start", C.c_void_p), ("col_row", C.c_void_p), ("col_val", C.c_void_p),
        ("var_lower", C.c_void_p), ("var_upper", C.c_void_p),
    ]


class bp_lp_desc(C.Structure):
    _fields_ = [
        ("n_vars", C.c_int32), ("n_rows", C.c_int32),
        ("row_start", C.c_void_p), ("row_col", C.c_void_p), ("row_val", C.c_void_p),
        ("col_start", C.c_void_p), ("col_row", C.c_void_p), ("col_val", C.c_void_p),
        ("obj", C.c_void_p), ("row_lower", C.c_void_p), ("row_upper", C.c_void_p),
        ("var_lower", C.c_void_p), ("var_upper", C.c_void_p),
    ]


class bp_limits(C.Structure):
    _fields_ = [("max_rounds", C.c_int32), ("time_limit", C.c_double),
                ("abs_threshold", C.c_double), ("rel_threshold", C.c_double),
                ("incremental", C.c_int32)]


class bp_rounding_config(C.Structure):
    _fields_ = [("random_band", C.c_double), ("single_var_tail", C.c_int32),
                ("repair_enabled", C.c_int32), ("repair_attempt_cap", C.c_int32),
                ("repair_shift_cap", C.c_int32)]


class bp_rounding_outcome(C.Structure):
    _fields_ = [("rounding_infeasible", C.c_int32), ("timed_out", C.c_int32),
                ("completed", C.c_int32), ("repair_attempts", C.c_int32),
                ("bulks_committed", C.c_int32), ("set_count", C.c_int32),
                ("bounds_feasible", C.c_int32), ("bp_calls", C.c_int32),
                ("device_ms", C.c_double)]


class bp_result(C.Structure):
    _fields_ = [("status", C.c_int32), ("rounds", C.c_int32), ("crossed_vars", C.c_int32)]


_lib = None

# (name, restype, argtypes) — every symbol include/bp.h declares.
_SIGS = [
    ("bp_last_error", C.c_char_p, []),
    ("bp_limits_default", None, [C.POINTER(bp_limits)]),
    ("bp_device_count", C.c_int, [C.POINTER(C.c_int32)]),
    ("bp_problem_create", C.c_int, [C.POINTER(bp_problem_desc), C.c_int32, C.POINTER(C.c_void_p)]),
    ("bp_problem_destroy", C.c_int, [C.c_void_p]),
    ("bp_problem_info", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int64)]),
    ("bp_compute_activities", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                        C.c_void_p, C.c_void_p]),
    ("bp_tighten_bounds", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                    C.POINTER(bp_limits), C.c_void_p, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32)]),
    ("bp_propagate", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.POINTER(bp_limits),
                               C.POINTER(bp_result)]),
    ("bp_propagate_device", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32),
                                      C.POINTER(bp_limits), C.POINTER(bp_result), C.c_void_p]),
    ("bp_propagate_ex", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32),
                                  C.POINTER(bp_limits), C.POINTER(bp_result), C.c_void_p, C.c_int32,
                                  C.c_void_p]),
    ("bp_probe_variables", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                     C.POINTER(C.c_void_p)]),
    ("bp_prioritize_probe_vars", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]),
    ("bp_build_cache", C.c_int, [C.c_void_p, C.c_double, C.POINTER(C.c_void_p)]),
    ("bp_cache_block_branches", C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    ("bp_cache_work", C.c_int, [C.c_void_p, C.c_void_p]),
    ("bp_build_cache_multi", C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_void_p, C.c_int32,
                                       C.POINTER(C.c_void_p), C.c_void_p]),
    ("bp_cache_destroy", C.c_int, [C.c_void_p]),
    ("bp_cache_info", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    ("bp_cache_entry", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_void_p,
                                 C.c_void_p]),
    ("bp_cache_deltas", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_void_p]),
    ("bp_cache_root", C.c_int, [C.c_void_p, C.c_void_p]),
    ("bp_cache_create_empty", C.c_int, [C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("bp_cache_set_entry", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                     C.c_void_p, C.c_void_p]),
    ("bp_cache_pack_size", C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    ("bp_cache_pack", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    ("bp_cache_merge_packed", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    ("bp_assemble_bulk_warm_start", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                              C.c_void_p, C.c_void_p, C.POINTER(C.c_int32),
                                              C.c_void_p, C.POINTER(C.c_int32)]),
    ("bp_rounding_config_default", None, [C.POINTER(bp_rounding_config)]),
    ("bp_propagation_round", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_double,
                                       C.POINTER(bp_rounding_config), C.c_void_p,
                                       C.POINTER(bp_rounding_outcome)]),
    ("bp_propagation_round_rng", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p,
                                           C.c_int64, C.c_double, C.POINTER(bp_rounding_config),
                                           C.c_void_p, C.POINTER(bp_rounding_outcome)]),
    ("bp_repair", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_double,
                            C.POINTER(bp_rounding_config), C.POINTER(C.c_int32), C.c_void_p,
                            C.c_void_p]),
    ("bp_parallel_propagate", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]),
    ("bp_build_problem", C.c_int, [C.POINTER(bp_builder_desc), C.c_int32, C.POINTER(bp_built),
                                   C.POINTER(C.c_void_p)]),
    ("bp_lp_create", C.c_int, [C.POINTER(bp_lp_desc), C.c_int32, C.POINTER(C.c_void_p)]),
    ("bp_lp_destroy", C.c_int, [C.c_void_p]),
    ("bp_lp_spmv_rows", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("bp_lp_spmv_cols", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("bp_lp_pdhg_iterate", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_double, C.c_double, C.c_int32]),
    ("bp_lp_evaluate_kkt", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("bp_lp_last_ms", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("bp_kernel_launches", C.c_int64, []),
    ("bp_kernel_time", C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_int64)]),
]


def exported_symbols():
    return [s[0] for s in _SIGS]


def lib():
    """Load libbp.so (raises BPError if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise BPError(BP_ERR_RUNTIME, f"engine library not built: {LIB_PATH} "
                                          "(run __graft_entry__.build())")
        L = C.CDLL(str(LIB_PATH))
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc != BP_OK:
        msg = lib().bp_last_error().decode(errors="replace")
        if rc == BP_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        if rc == BP_ERR_OUT_OF_RANGE:
            raise IndexError(msg)
        raise BPError(rc, msg)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def limits_struct(lim=None) -> bp_limits:
    s = bp_limits()
    lib().bp_limits_default(C.byref(s))
    if lim is not None:
        s.max_rounds = int(lim.max_rounds)
        s.time_limit = float(lim.time_limit)
        s.abs_threshold = float(lim.abs_threshold)
        s.rel_threshold = float(lim.rel_threshold)
        s.incremental = 1 if lim.incremental else 0
    return s


def kernel_launches() -> int:
    return int(lib().bp_kernel_launches())


def device_count() -> int:
    c = C.c_int32(0)
    if os.environ.get("CUDA_VISIBLE_DEVICES", None) == "":
        return 0
    rc = lib().bp_device_count(C.byref(c))
    return int(c.value) if rc == BP_OK else 0
