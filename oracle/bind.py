"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU oracles (never used by the product path).

* ``Ref``  — the unmodified reference headers compiled by oracle/Makefile (oracle/_ref/libpulse_ref.so)
* ``Port`` — our plain-C restatement (oracle/_ref/libbp_oracle.so)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import this.
"""
from __future__ import annotations

import ctypes as C
import math
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libpulse_ref.so"
PORT_SO = HERE / "_ref" / "libbp_oracle.so"

V = C.c_void_p
I = C.c_int
D = C.c_double


def _p(a):
    return None if a is None else a.ctypes.data_as(V)


def build(ref=True):
    """Builds the port (always) and the reference shim (when /root/reference exists)."""
    targets = ["port"] + (["ref"] if ref and Path("/root/reference/proj/include/pulse").is_dir() else [])
    subprocess.run(["make", "-C", str(HERE)] + targets, check=True, capture_output=True)


def limits_array(lim=None):
    if lim is None:
        return np.array([64, math.inf, 1e-7, 1e-4, 1.0])
    return np.array([lim.max_rounds, lim.time_limit, lim.abs_threshold, lim.rel_threshold,
                     1.0 if lim.incremental else 0.0])


class Ref:
    """The reference implementation (compiled in place from /root/reference)."""

    _L = None

    @classmethod
    def available(cls):
        return REF_SO.exists()

    @classmethod
    def lib(cls):
        if cls._L is None:
            L = C.CDLL(str(REF_SO))
            sig = {
                "ref_problem_build": (V, [I, I, V, V, V, V, V, V, C.c_longlong, V, V, V]),
                "ref_problem_from_csr": (V, [I, I, V, V, V, V, V, V, V, V]),
                "ref_problem_free": (None, [V]),
                "ref_problem_dims": (None, [V, V, V, V]),
                "ref_problem_export": (None, [V] + [V] * 12),
                "ref_rng_new": (V, [C.c_ulonglong]),
                "ref_rng_free": (None, [V]),
                "ref_random_instance": (V, [V, I, I, I, D, I, I, I]),
                "ref_rng_uniform_int": (I, [V, I, I]),
                "ref_rng_uniform_real": (D, [V, D, D]),
                "ref_max_threads": (I, []),
                "ref_compute_activities": (None, [V, V, V, I, I, V, V, V]),
                "ref_tighten_bounds": (I, [V, V, V, V, V, V, V, I, V, V, V]),
                "ref_propagate": (None, [V, V, V, V, I, V]),
                "ref_make_branch_spec": (I, [D, D, V]),
                "ref_prioritize_probe_vars": (I, [V, V]),
                "ref_cache_new_empty": (V, [V]),
                "ref_build_cache": (V, [V, D]),
                "ref_cache_probe_into": (None, [V, V, V, I, I]),
                "ref_cache_free": (None, [V]),
                "ref_cache_stats": (None, [V, V, V]),
                "ref_cache_entry": (I, [V, I, V, V]),
                "ref_cache_deltas": (None, [V, I, I, V, V, V]),
                "ref_cache_set_entry": (None, [V, I, V, V, V, V, V]),
                "ref_cache_from_packed": (V, [V, V, C.c_longlong]),
                "ref_assemble_bulk_warm_start": (I, [V, V, V, I, V, V, V, V]),
                "ref_initial_sort": (I, [V, V, V]),
                "ref_implied_slack_sort": (None, [V, V, V, V, V, I]),
                "ref_get_bulk_size": (I, [I, I, I]),
                "ref_generate_candidate_values": (None, [V, V, I, V, I, V, D, V, V]),
                "ref_repair": (I, [V, V, V, I, I, V, V]),
                "ref_problem_set_obj": (None, [V, V]),
                "ref_lp_spmv_rows": (None, [V, V, V]),
                "ref_lp_evaluate_kkt": (None, [V, V, V, V]),
                "ref_lp_spmv_cols": (None, [V, V, V]),
                "ref_lp_pdhg_iterate": (None, [V, V, V, V, V, V, D, D, I]),
                "ref_parallel_propagate": (None, [V, V, I, V, I, V, V, V, V, V, V, V, V, V, V, V, V]),
                "ref_propagation_round": (None, [V, V, V, C.c_ulonglong, D, D, I, V, V]),
            }
            for n, (r, a) in sig.items():
                f = getattr(L, n)
                f.restype = r
                f.argtypes = a
            cls._L = L
        return cls._L


class RefProblem:
    """A pulse::ProblemDef living in the reference library."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        try:
            if self.h:
                Ref.lib().ref_problem_free(self.h)
        except Exception:
            pass

    @classmethod
    def from_def(cls, p):
        keep = [np.ascontiguousarray(x) for x in (p.row_start, p.row_col, p.row_val, p.var_lower,
                                                  p.var_upper, p.is_integer, p.cons_lower,
                                                  p.cons_upper)]
        h = Ref.lib().ref_problem_from_csr(p.n_vars, p.n_cons, *[_p(x) for x in keep])
        return cls(h)

    def to_def(self):
        from paper_2510_20499_b200.problem import ProblemDef
        L = Ref.lib()
        n, m, nnz = C.c_int(), C.c_int(), C.c_int()
        L.ref_problem_dims(self.h, C.byref(n), C.byref(m), C.byref(nnz))
        n, m, nnz = n.value, m.value, nnz.value
        a = dict(row_start=np.zeros(m + 1, np.int32), row_col=np.zeros(nnz, np.int32),
                 row_val=np.zeros(nnz), col_start=np.zeros(n + 1, np.int32),
                 col_row=np.zeros(nnz, np.int32), col_val=np.zeros(nnz), var_lower=np.zeros(n),
                 var_upper=np.zeros(n), is_integer=np.zeros(n, np.uint8), cons_lower=np.zeros(m),
                 cons_upper=np.zeros(m), obj_coeffs=np.zeros(n))
        order = ["row_start", "row_col", "row_val", "col_start", "col_row", "col_val", "var_lower",
                 "var_upper", "is_integer", "cons_lower", "cons_upper", "obj_coeffs"]
        L.ref_problem_export(self.h, *[_p(a[k]) for k in order])
        return ProblemDef(n_vars=n, n_cons=m, **a)


class RefRng:
    def __init__(self, seed):
        self.h = Ref.lib().ref_rng_new(seed)

    def __del__(self):
        try:
            Ref.lib().ref_rng_free(self.h)
        except Exception:
            pass

    def random_instance(self, max_vars=8, max_rows=8, max_bound_span=4, density=0.6,
                        force_feasible=False, allow_continuous=False, allow_one_sided=True):
        """testkit::random_instance (tests/testkit.hpp:69-143) on this generator's stream."""
        h = Ref.lib().ref_random_instance(self.h, max_vars, max_rows, max_bound_span, density,
                                          int(force_feasible), int(allow_continuous),
                                          int(allow_one_sided))
        return RefProblem(h)

    def uniform_int(self, lo, hi):
        return Ref.lib().ref_rng_uniform_int(self.h, lo, hi)

    def uniform_real(self, lo, hi):
        return Ref.lib().ref_rng_uniform_real(self.h, lo, hi)


def ref_propagate(rp, bounds, infeasible=False, lim=None, use_plan=True):
    """Reference propagate on a copy of ``bounds``. Returns (bounds, infeasible, status, rounds, crossed)."""
    b = np.array(bounds, dtype=np.float64, copy=True)
    inf = C.c_int(int(infeasible))
    out = np.zeros(3, np.int32)
    la = limits_array(lim)
    Ref.lib().ref_propagate(rp.h, _p(b), C.byref(inf), _p(la), int(use_plan), _p(out))
    return b, bool(inf.value), int(out[0]), int(out[1]), int(out[2])


def ref_compute_activities(rp, m, bounds, rows=None, act=None, nmin=None, nmax=None, use_plan=False):
    act = np.zeros(2 * m) if act is None else np.array(act, dtype=np.float64, copy=True)
    nmin = np.zeros(m, np.int32) if nmin is None else np.array(nmin, dtype=np.int32, copy=True)
    nmax = np.zeros(m, np.int32) if nmax is None else np.array(nmax, dtype=np.int32, copy=True)
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    Ref.lib().ref_compute_activities(rp.h, _p(np.ascontiguousarray(bounds, dtype=np.float64)), _p(r),
                                     -1 if r is None else r.size, int(use_plan), _p(act), _p(nmin),
                                     _p(nmax))
    return act, nmin, nmax


def ref_tighten_bounds(rp, n, bounds, infeasible, act, nmin, nmax, vars_=None, lim=None):
    b = np.array(bounds, dtype=np.float64, copy=True)
    inf = C.c_int(int(infeasible))
    ch = np.zeros(max(n, 1), np.int32)
    cr = C.c_int(0)
    v = None if vars_ is None else np.ascontiguousarray(vars_, dtype=np.int32)
    la = limits_array(lim)
    nch = Ref.lib().ref_tighten_bounds(rp.h, _p(b), C.byref(inf), _p(np.asarray(act, np.float64)),
                                       _p(np.asarray(nmin, np.int32)), _p(np.asarray(nmax, np.int32)),
                                       _p(v), -1 if v is None else v.size, _p(la), _p(ch), C.byref(cr))
    return b, bool(inf.value), list(ch[:nch]), int(cr.value)


# ------------------------------------------------------------------ port (plain C restatement)


class orc_problem(C.Structure):
    _fields_ = [("n_vars", C.c_int), ("n_cons", C.c_int)] + [
        (n, V) for n in ("row_start", "row_col", "row_val", "col_start", "col_row", "col_val",
                         "var_lower", "var_upper", "is_integer", "cons_lower", "cons_upper")]


class orc_limits(C.Structure):
    _fields_ = [("max_rounds", C.c_int), ("abs_threshold", D), ("rel_threshold", D),
                ("incremental", C.c_int)]


class Port:
    _L = None

    @classmethod
    def lib(cls):
        if cls._L is None:
            L = C.CDLL(str(PORT_SO))
            P = C.POINTER(orc_problem)
            LP = C.POINTER(orc_limits)
            sig = {
                "orc_default_limits": (None, [LP]),
                "orc_compute_activities": (None, [P, V, V, I, V, V, V]),
                "orc_tighten_bounds": (I, [P, V, V, V, V, V, V, I, LP, V, V]),
                "orc_propagate": (None, [P, V, V, LP, V]),
                "orc_make_branch_spec": (I, [D, D, V]),
                "orc_probe_variable": (I, [P, V, I, V, V, V, V, V]),
                "orc_implied_slack_sort": (None, [P, V, V, V, V, I]),
            }
            for n, (r, a) in sig.items():
                f = getattr(L, n)
                f.restype = r
                f.argtypes = a
            cls._L = L
        return cls._L


class PortProblem:
    def __init__(self, p):
        self.p = p
        self._keep = [np.ascontiguousarray(x) for x in (
            p.row_start, p.row_col, p.row_val, p.col_start, p.col_row, p.col_val, p.var_lower,
            p.var_upper, p.is_integer, p.cons_lower, p.cons_upper)]
        self.s = orc_problem(p.n_vars, p.n_cons, *[_p(x) for x in self._keep])

    def limits(self, lim=None):
        l = orc_limits()
        Port.lib().orc_default_limits(C.byref(l))
        if lim is not None:
            l.max_rounds = lim.max_rounds
            l.abs_threshold = lim.abs_threshold
            l.rel_threshold = lim.rel_threshold
            l.incremental = 1 if lim.incremental else 0
        return l

    def propagate(self, bounds, infeasible=False, lim=None):
        b = np.array(bounds, dtype=np.float64, copy=True)
        inf = C.c_int(int(infeasible))
        out = np.zeros(3, np.int32)
        l = self.limits(lim)
        Port.lib().orc_propagate(C.byref(self.s), _p(b), C.byref(inf), C.byref(l), _p(out))
        return b, bool(inf.value), int(out[0]), int(out[1]), int(out[2])

    def compute_activities(self, bounds, rows=None, act=None, nmin=None, nmax=None):
        m = self.p.n_cons
        act = np.zeros(2 * m) if act is None else np.array(act, dtype=np.float64, copy=True)
        nmin = np.zeros(m, np.int32) if nmin is None else np.array(nmin, dtype=np.int32, copy=True)
        nmax = np.zeros(m, np.int32) if nmax is None else np.array(nmax, dtype=np.int32, copy=True)
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
        Port.lib().orc_compute_activities(C.byref(self.s), _p(np.ascontiguousarray(bounds)), _p(r),
                                          -1 if r is None else r.size, _p(act), _p(nmin), _p(nmax))
        return act, nmin, nmax

    def tighten_bounds(self, bounds, infeasible, act, nmin, nmax, vars_=None, lim=None):
        b = np.array(bounds, dtype=np.float64, copy=True)
        inf = C.c_int(int(infeasible))
        ch = np.zeros(max(self.p.n_vars, 1), np.int32)
        cr = C.c_int(0)
        v = None if vars_ is None else np.ascontiguousarray(vars_, dtype=np.int32)
        l = self.limits(lim)
        nch = Port.lib().orc_tighten_bounds(C.byref(self.s), _p(b), C.byref(inf),
                                            _p(np.asarray(act, np.float64)),
                                            _p(np.asarray(nmin, np.int32)),
                                            _p(np.asarray(nmax, np.int32)), _p(v),
                                            -1 if v is None else v.size, C.byref(l), _p(ch),
                                            C.byref(cr))
        return b, bool(inf.value), list(ch[:nch]), int(cr.value)

    def probe_variable(self, root, v):
        n = self.p.n_vars
        feas = np.zeros(2, np.int32)
        nd = np.zeros(2, np.int32)
        dv = np.zeros(2 * n, np.int32)
        dl = np.zeros(2 * n)
        du = np.zeros(2 * n)
        kind = Port.lib().orc_probe_variable(C.byref(self.s), _p(np.ascontiguousarray(root)), v,
                                             _p(feas), _p(nd), _p(dv), _p(dl), _p(du))
        out = []
        for s in range(2):
            o = s * n
            out.append((bool(feas[s]), dv[o:o + nd[s]].copy(), dl[o:o + nd[s]].copy(),
                        du[o:o + nd[s]].copy()))
        return kind, out


# ------------------------------------------------------------------ reference rounding / cache


class RefCache:
    """A pulse::ProbingCache inside the reference library."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            Ref.lib().ref_cache_free(self.h)
        except Exception:
            pass

    @classmethod
    def build(cls, rp, budget=1e9):
        return cls(Ref.lib().ref_build_cache(rp.h, budget))

    @classmethod
    def from_packed(cls, rp, gpu_cache):
        """Every entry of an engine-built cache in a reference ProbingCache, in one call (the
        engine's packed slice format; for caches of millions of entries)."""
        buf = gpu_cache.pack()
        h = Ref.lib().ref_cache_from_packed(rp.h, _p(buf), int(buf.size))
        if not h:
            raise ValueError("packed cache does not match its size")
        return cls(h)

    @classmethod
    def from_gpu(cls, rp, gpu_cache):
        """Installs every entry of an engine-built cache into a reference ProbingCache."""
        L = Ref.lib()
        c = cls(L.ref_cache_new_empty(rp.h))
        for v in range(gpu_cache.n_vars):
            raw = gpu_cache._entry_raw(v)
            if raw is None:
                continue
            hdr, br = raw
            d0 = gpu_cache.deltas(v, 0)
            d1 = gpu_cache.deltas(v, 1)
            dv = np.ascontiguousarray(np.concatenate([d0[0], d1[0]]), dtype=np.int32)
            dl = np.ascontiguousarray(np.concatenate([d0[1], d1[1]]))
            du = np.ascontiguousarray(np.concatenate([d0[2], d1[2]]))
            L.ref_cache_set_entry(c.h, v, _p(np.ascontiguousarray(hdr, dtype=np.int32)),
                                  _p(np.ascontiguousarray(br)), _p(dv), _p(dl), _p(du))
        return c


    def entry(self, v):
        """(hdr7, br4, [(vars, lo, up) down, up]) of the reference entry of v, or None."""
        L = Ref.lib()
        hdr = np.zeros(7, np.int32)
        br = np.zeros(4)
        if not L.ref_cache_entry(self.h, int(v), _p(hdr), _p(br)):
            return None
        sides = []
        for side in range(2):
            cnt = int(hdr[5 + side])
            vv = np.zeros(max(cnt, 1), np.int32)
            lo = np.zeros(max(cnt, 1))
            up = np.zeros(max(cnt, 1))
            L.ref_cache_deltas(self.h, int(v), side, _p(vv), _p(lo), _p(up))
            sides.append((vv[:cnt], lo[:cnt], up[:cnt]))
        return hdr, br, sides

    @classmethod
    def probe_into(cls, rp, n_vars, root, vars_):
        """The reference's probe_variable (probing.hpp:225) of each var in ``vars_`` from ``root``,
        stored in a fresh cache handle. One call at a time: each probe already runs on the
        reference's pool, and concurrent external callers widen a use-after-scope race in its
        parallel_for (parallel.hpp:117-129: the waiter can return and destroy its mutex /
        condition variable while the last worker is about to lock them)."""
        c = cls(Ref.lib().ref_cache_new_empty(rp.h))
        r = np.ascontiguousarray(root, dtype=np.float64)
        for v in vars_:
            Ref.lib().ref_cache_probe_into(c.h, rp.h, _p(r), int(v), 0)
        return c


def cache_mismatches(gpu_cache, ref_cache, vars_):
    """Entries of ``vars_`` present in the reference cache that differ from the GPU cache in any
    bit (kind, forcing flags, feasibility, branch bounds, delta vars and values). Returns
    (checked, [mismatching vars])."""
    bad, checked = [], 0
    for v in vars_:
        r = ref_cache.entry(v)
        if r is None:
            continue
        checked += 1
        g = gpu_cache._entry_raw(v)
        if g is None:
            bad.append(int(v))
            continue
        rh, rb, rs = r
        gh, gb = g
        same = np.array_equal(np.asarray(gh[:7]), rh) and np.array_equal(np.asarray(gb).view(np.uint64), rb.view(np.uint64))
        if same:
            for side in range(2):
                gv, gl, gu = gpu_cache.deltas(v, side)
                rv, rl, ru = rs[side]
                same = same and np.array_equal(gv, rv) and np.array_equal(gl.view(np.uint64), rl.view(np.uint64)) \
                    and np.array_equal(gu.view(np.uint64), ru.view(np.uint64))
        if not same:
            bad.append(int(v))
    return checked, bad


def ref_propagation_round(rp, n_vars, start, cache=None, seed=0, deadline=0.0, band=0.25,
                          repair=False):
    """rounding.hpp:393 with Rng(seed); returns (values, flags dict). lp_polish runs inside."""
    vals = np.zeros(max(n_vars, 1))
    fl = np.zeros(6, np.int32)
    Ref.lib().ref_propagation_round(rp.h, _p(np.ascontiguousarray(start, dtype=np.float64)),
                                    None if cache is None else cache.h, seed, deadline, band,
                                    int(repair), _p(vals), _p(fl))
    keys = ["rounding_infeasible", "timed_out", "completed", "repair_attempts", "bulks_committed",
            "set_count"]
    return vals[:n_vars], dict(zip(keys, (int(x) for x in fl)))


def ref_repair(rp, n_vars, fixed, shift_cap=64):
    """rounding.hpp:234 repair through oracle/_ref: None (std::nullopt) or (values, bounds2n)."""
    k = len(fixed)
    fv = np.ascontiguousarray([v for v, _ in fixed] or [0], dtype=np.int32)
    fx = np.ascontiguousarray([x for _, x in fixed] or [0.0], dtype=np.float64)
    out = np.zeros(max(k, 1))
    b = np.zeros(max(2 * n_vars, 1))
    ok = Ref.lib().ref_repair(rp.h, _p(fv), _p(fx), k, int(shift_cap), _p(out), _p(b))
    if not ok:
        return None
    return [(int(v), float(out[j])) for j, (v, _) in enumerate(fixed)], b[: 2 * n_vars]
