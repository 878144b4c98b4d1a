"""Benchmark: BP nnz/s and HBM GB/s vs peak on BASELINE.json configs[1] (C2: synthetic 1M x 1M MILP,
power-law rows median 7 / max ~100k) — one full `propagate` to fixpoint from the original bounds per
step, on the persistent sm_100a engine.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C2|C1]

One JSON line on rank 0. `value` = BP nnz visits/s (the reference trajectory's work, counted by
the engine's exact-frontier stats pass) over all ranks, device-timed with CUDA events, max over
ranks; inputs resident in HBM. `e2e` = the same metric through the C-ABI with host (pinned)
bounds copied in and out every step. `roofline` = algorithmic bytes of the engine kernel per
launch / its CUDA-event duration vs MEASURED_PEAKS.json hbm_gbs. `cpu_baseline` = the reference
(oracle/_ref, compiled from /root/reference) propagate on the host cores. N > 1: independent
replicas (a single propagation does not shard), weak scaling.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json


_T0 = time.perf_counter()


def log(msg):
    """Progress on stderr (the JSON line is the only stdout output)."""
    print(f"[bench {time.perf_counter() - _T0:8.1f}s] {msg}", file=sys.stderr, flush=True)


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK, "fallback"


def make_workload(name):
    from paper_2510_20499_b200 import synth
    if name == "C2":
        return synth.c2(), "C2: synthetic MILP 1M x 1M, Pareto rows (median 7, max ~100k), skewed cols"
    if name == "C1":
        return synth.c1(), "C1: synthetic MILP 10k x 10k, ~8 nnz/row, mixed types"
    raise SystemExit(f"unknown workload {name}")


class ClockSampler:
    """nvidia-smi clock/throttle sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0, t1):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        self.t.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, smax, reasons, n_in = [], [], set(), 0
        for ts, line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            inside = t0 - 0.06 <= ts <= t1 + 0.06
            try:
                smax.append(float(f[2]))
                if inside:
                    sm.append(float(f[1]))
                    n_in += 1
                    for nm, v in zip(names, f[5:9]):
                        if v.lower().startswith("active"):
                            reasons.add(nm)
            except ValueError:
                continue
        if not sm:  # region shorter than one sample: nearest samples
            near = sorted(self.lines, key=lambda x: min(abs(x[0] - t0), abs(x[0] - t1)))[:2]
            for ts, line in near:
                f = [x.strip() for x in line.split(",")]
                try:
                    sm.append(float(f[1]))
                except (ValueError, IndexError):
                    pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples_in_region": n_in}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_reference_propagate(p, reps=1):
    """The reference's own propagate (oracle/_ref/libpulse_ref.so) on all host threads."""
    from oracle.bind import Ref, RefProblem, ref_propagate
    if not Ref.available():
        return None
    rp = RefProblem.from_def(p)
    root = p.root_bounds()
    times = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = ref_propagate(rp, root)
        times.append(time.perf_counter() - t0)
    return times, out, int(Ref.lib().ref_max_threads())


def cpu_reference_single_thread(workload):
    """Seconds of one reference propagate of `workload` with PULSE_THREADS=1 (the reference's pool
    size is fixed at first use, so this runs in a child process)."""
    code = ("import sys, time; sys.path.insert(0, %r); import bench; "
            "from oracle.bind import RefProblem, ref_propagate; p, _ = bench.make_workload(%r); "
            "rp = RefProblem.from_def(p); r = p.root_bounds(); t = time.perf_counter(); "
            "ref_propagate(rp, r); print(time.perf_counter() - t)") % (str(ROOT), workload)
    try:
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PULSE_THREADS="1"),
                             capture_output=True, text=True, timeout=600)
        return float(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None


def run_reference_arm(args, rank, world):
    """--impl reference: the reference CPU implementation on this box's host cores."""
    if rank != 0:
        return
    p, desc = make_workload(args.workload)
    visits = None
    res = cpu_reference_propagate(p, reps=1)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpulse_ref.so not built"}))
        return
    # the visit count of the reference trajectory (identical to ours; from the port's replay)
    visits = reference_visits(p)
    for _ in range(args.warmup):
        cpu_reference_propagate(p, reps=1)
    t0 = time.perf_counter()
    times, out, cores = cpu_reference_propagate(p, reps=args.steps)
    el = time.perf_counter() - t0
    v = visits * args.steps / el
    line = {"metric": "BP nnz/s", "value": v, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": desc, "rounds": out[3], "nnz_visits_per_step": visits},
            "cpu_baseline": {"value": v, "unit": "nnz/s", "cores": cores, "kind": "reference",
                             "sample": f"{args.steps} full propagate calls of {args.workload}"},
            "e2e": {"value": v, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def reference_visits(p):
    """Σ_r (row nnz of R_r + col nnz of V_r) of the reference trajectory, replayed round by round
    with the C port (CPU-side accounting for the reference arm; identical to the engine stats)."""
    from oracle.bind import PortProblem
    pp = PortProblem(p)
    b = p.root_bounds()
    n, m = p.n_vars, p.n_cons
    rnnz = np.diff(p.row_start).astype(np.int64)
    cnnz = np.diff(p.col_start).astype(np.int64)
    visits = int(rnnz.sum() + cnnz.sum())
    act, nmin, nmax = pp.compute_activities(b)
    b, inf, changed, _ = pp.tighten_bounds(b, False, act, nmin, nmax)
    rounds = 1
    while changed and not inf and rounds < 64:
        ch = np.array(changed, dtype=np.int64)
        rows = np.unique(np.concatenate([p.col_row[p.col_start[i]:p.col_start[i + 1]] for i in ch]))
        if rows.size == 0:
            break
        vars_ = np.unique(np.concatenate([p.row_col[p.row_start[k]:p.row_start[k + 1]] for k in rows]))
        visits += int(rnnz[rows].sum() + cnnz[vars_].sum())
        act, nmin, nmax = pp.compute_activities(b, rows=rows, act=act, nmin=nmin, nmax=nmax)
        b, inf, changed, _ = pp.tighten_bounds(b, False, act, nmin, nmax, vars_=vars_)
        rounds += 1
    return visits


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_probing(args, rank, world, local):
    """configs[2]: batched double probing of all 200k binaries of C3 (500k x 500k set covering),
    candidates sharded over the ranks, packed slices gathered to rank 0 (NCCL), merged there.
    probes/s = variables probed (both branches) / wall time of probe + gather + merge."""
    import torch
    import torch.distributed as dist

    from paper_2510_20499_b200 import synth
    from paper_2510_20499_b200.distributed import build_cache_sharded
    from paper_2510_20499_b200.probing import probe_variables

    log("probing: generating C3")
    p = synth.c3()
    vars_ = np.arange(200_000, dtype=np.int32)  # the binaries (every one is probed: order is immaterial)
    for _ in range(2):  # warm-up: kernels loaded, problem uploaded, probing scratch sized
        probe_variables(p, None, vars_)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    if world > 1:
        cache, dev_ms = build_cache_sharded(p, vars_, device=torch.device("cuda", local))
    else:
        cache = probe_variables(p, None, vars_)
        dev_ms = cache.probe_ms
    if world > 1:
        dist.barrier()
    el = _max_over_ranks(time.perf_counter() - t0, world)
    dev_ms = _max_over_ranks(dev_ms, world)
    if rank != 0:
        return None
    out = {"workload": "C3: set covering 500k x 500k (200k binaries + 300k continuous), N=%d" % p.nnz(),
           "probes_per_s": len(vars_) / el, "variables_probed": cache.n_probed,
           "branches": 2 * cache.n_probed, "infeasible_branches": cache.n_infeasible_branches,
           "deltas": cache.n_deltas, "fallback_branches": cache.n_fallback,
           "block_kernel_branches": cache.n_block,
           "root_certified_fixpoint": cache.certified, "wall_ms": el * 1e3,
           "probe_kernel_ms_max_rank": dev_ms, "n_gpus": world,
           "parallelism": f"candidates sharded x{world}, NCCL send/recv gather to rank 0"}
    if world == 1:
        # the BP byte formula summed over branches and rounds (the engine counts each
        # branch's dirty sets: R, row nnz A, V, col nnz B, changed C). C3's matrix (~90 MB) sits
        # largely in L2, so this is an EFFECTIVE bandwidth that can exceed the HBM figure.
        R, A, V, B, Cc = cache.work
        pb = 28 * A + 28 * R + 52 * B + 21 * V + 16 * Cc
        peak, peak_kind = peaks()
        ach = pb / (dev_ms * 1e-3) / 1e9
        out["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                           "frac": ach / peak, "peak_kind": peak_kind, "effective_l2": True,
                           "algorithmic_bytes": pb, "branch_work": {"rows": R, "row_nnz": A, "vars": V,
                                                                    "col_nnz": B, "changed": Cc},
                           "kernel": "k_probe (warp per branch) + k_probe_block, CUDA-event time"}
    if world == 1 and not args.no_cpu_baseline:
        from oracle.bind import Ref, RefCache, RefProblem, cache_mismatches
        if Ref.available():
            rp = RefProblem.from_def(p)
            L = Ref.lib()
            t0 = time.perf_counter()
            rc = RefCache(L.ref_build_cache(rp.h, args.cpu_sample_sec))
            el_cpu = time.perf_counter() - t0
            import ctypes as C
            npb, ninf = C.c_int(), C.c_int()
            L.ref_cache_stats(rc.h, C.byref(npb), C.byref(ninf))
            out["cpu_baseline"] = {"value": npb.value / args.cpu_sample_sec, "unit": "probes/s",
                                   "cores": int(L.ref_max_threads()), "kind": "reference",
                                   "sample": f"build_cache(p, {args.cpu_sample_sec:g} s): "
                                             f"{npb.value} vars probed ({el_cpu:.1f} s incl. "
                                             "prioritization)"}
            # parity: every entry the reference's build_cache produced equals the GPU cache's, bitwise
            checked, bad = cache_mismatches(cache, rc, range(p.n_vars))
            out["parity"] = {"reference_entries_checked": checked, "mismatches": len(bad),
                             "against": "pulse::build_cache (oracle/_ref) entries, bitwise"}
            assert checked == npb.value and not bad, f"C3 cache differs from the reference at {bad[:5]}"

    return out


def run_rounding(args, rank, world, local):
    """configs[3]: fix-and-propagate bulk rounding with a FULL-coverage probing cache on the 2M x 2M
    knapsack/assignment mix (presolved to its propagation fixpoint), propagation_round with
    Deadline::never() and Rng(4), one replica per rank. The CPU baseline runs the reference's
    propagation_round with the SAME cache (RefCache.from_packed) for a bounded time; the GPU is then
    timed on exactly the same number of committed bulks (identical trajectory), like for like."""
    from paper_2510_20499_b200 import BoundsState, propagate, synth
    from paper_2510_20499_b200.probing import build_cache
    from paper_2510_20499_b200.rounding import propagation_round

    p0, start = synth.c4()
    b = BoundsState(p0)
    r0 = propagate(p0, b)
    p = synth.with_bounds(p0, b.raw())
    log(f"rounding: C4 presolved in {r0.rounds} rounds; building the full-coverage cache")
    t0 = time.perf_counter()
    cache = build_cache(p, 1e9)  # fp.hpp:263 with an unbounded budget: every candidate probed
    cache_s = _max_over_ranks(time.perf_counter() - t0, world)
    log(f"rounding: cache {cache.n_probed} vars in {cache_s:.1f} s ({cache.n_block} block-kernel branches)")
    t0 = time.perf_counter()
    out = propagation_round(p, start, cache, seed=4 + rank, deadline_sec=args.round_deadline)
    el = _max_over_ranks(time.perf_counter() - t0, world)
    log(f"rounding: {out.bulks_committed} bulks, {out.bp_calls} BP calls in {el:.1f} s, completed={out.completed}")
    if rank != 0:
        return None
    free_int = int(sum(1 for v in range(p.n_vars) if p.is_integer[v] and p.var_lower[v] != p.var_upper[v]))
    res = {"workload": "C4: knapsack/assignment 2M x 2M (N=%d), presolved root (%d BP rounds)"
                       % (p.nnz(), r0.rounds),
           "cache_build_s": cache_s, "cache_budget_s": "unbounded (full coverage)",
           "cache_vars": cache.n_probed, "cache_free_integer_vars": free_int,
           "cache_probes_per_s": cache.n_probed / cache_s, "cache_fallback_branches": cache.n_fallback,
           "cache_block_kernel_branches": cache.n_block, "round_s": el,
           "bulks_committed": out.bulks_committed, "bp_calls": out.bp_calls,
           "bulks_committed_per_s": out.bulks_committed / el,
           "bp_calls_per_s": world * out.bp_calls / el, "completed": out.completed,
           "timed_out": out.timed_out, "deadline_s": args.round_deadline or None,
           "rounding_infeasible": out.rounding_infeasible, "set_count": out.set_count,
           "engine_device_ms": out.device_ms, "n_gpus": world, "parallelism": f"replicas x{world}"}
    if world == 1 and not args.no_cpu_baseline:
        from oracle.bind import Ref, RefCache, RefProblem, ref_propagation_round
        if Ref.available():
            rp = RefProblem.from_def(p)
            rcache = RefCache.from_packed(rp, cache)
            t0 = time.perf_counter()
            _, fl = ref_propagation_round(rp, p.n_vars, start, rcache, 4, deadline=args.cpu_sample_sec)
            el_cpu = time.perf_counter() - t0
            k = int(fl["bulks_committed"])
            res["cpu_baseline"] = {"value": k / el_cpu, "unit": "bulks committed/s",
                                   "cores": int(Ref.lib().ref_max_threads()), "kind": "reference",
                                   "sample": f"propagation_round with the same full cache, deadline "
                                             f"{args.cpu_sample_sec:g} s: the first {k} bulks"}
            if k > 0:  # the GPU on exactly those first k bulks (same trajectory)
                os.environ["BP_ROUND_MAX_BULKS"] = str(k)
                try:
                    t0 = time.perf_counter()
                    gk = propagation_round(p, start, cache, seed=4, deadline_sec=0.0)
                    el_k = time.perf_counter() - t0
                finally:
                    del os.environ["BP_ROUND_MAX_BULKS"]
                assert gk.bulks_committed == k
                res["like_for_like"] = {"bulks": k, "gpu_s": el_k, "cpu_s": el_cpu,
                                        "gpu_bulks_per_s": k / el_k, "cpu_bulks_per_s": k / el_cpu}
    return res


def run_lp(args, rank, world, local, p):
    """the PDHG inner iteration (lp.hpp:315-340: spmv_rows + dual prox +
    spmv_cols + primal step + running sums) on the C2 matrix, device-resident; CUDA-event time of
    `iters` iterations per call. Algorithmic (compulsory) bytes per iteration: both matrix views
    streamed once (24 B per nnz) and the elementwise vectors (dual step 40 B / row, primal step
    72 B / var + 16 B / row for the running sums)."""
    from paper_2510_20499_b200.lp import DeviceLp, LpInstance
    if rank != 0:
        return None
    n, m, N = p.n_vars, p.n_cons, p.nnz()
    s = LpInstance.relax(p)
    s.obj = np.random.default_rng(7).normal(size=n)
    lp = DeviceLp(s)
    x = np.clip(np.zeros(n), p.var_lower, p.var_upper)
    st = [x, np.zeros(m), x.copy(), np.zeros(n), np.zeros(m)]
    iters = 20
    lp.pdhg_iterate(*st, 1e-3, 1e-3, 3)  # warm-up
    ms = []
    for _ in range(3):
        st = list(lp.pdhg_iterate(*st, 1e-3, 1e-3, iters))
        ms.append(lp.last_ms() / iters)
    it_ms = float(np.median(ms))
    # compulsory unique traffic: both matrix views streamed once (24 B per nnz) + the elementwise
    # vectors; the x / y gathers of the products are L2 hits (16 MB vectors), not compulsory
    alg = 24 * N + 40 * m + 72 * n + 16 * m
    peak, peak_kind = peaks()
    out = {"workload": "PDHG inner iteration on the C2 matrix (1M x 1M, %d nnz)" % N,
           "ms_per_iteration": it_ms, "iterations_per_s": 1e3 / it_ms,
           "roofline": {"bound": "hbm", "achieved": alg / (it_ms * 1e-3) / 1e9, "peak": peak,
                        "unit": "GB/s", "frac": alg / (it_ms * 1e-3) / 1e9 / peak,
                        "algorithmic_bytes_per_iteration": alg, "peak_kind": peak_kind},
           "parity": "bitwise vs lpdetail::spmv_rows / spmv_cols (tests/test_gpu_lp.py)"}
    if world == 1 and not args.no_cpu_baseline:
        import ctypes as C

        from oracle.bind import Ref, RefProblem
        if Ref.available():
            rp = RefProblem.from_def(p)
            o = np.ascontiguousarray(s.obj)
            Ref.lib().ref_problem_set_obj(rp.h, o.ctypes.data_as(C.c_void_p))
            r = [np.ascontiguousarray(a, dtype=np.float64).copy() for a in st]
            P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
            k = 5
            t0 = time.perf_counter()
            Ref.lib().ref_lp_pdhg_iterate(rp.h, *[P(a) for a in r], 1e-3, 1e-3, k)
            el = time.perf_counter() - t0
            out["cpu_baseline"] = {"value": k / el, "unit": "iterations/s",
                                   "cores": int(Ref.lib().ref_max_threads()), "kind": "reference",
                                   "sample": f"{k} iterations of the reference's products (parallel_for) + "
                                             f"the restated elementwise steps ({el:.2f} s)"}
    return out


def run_build(args, rank, world, local, p):
    """ProblemBuilder::build (problem.hpp:141-227) of the C2 problem from its
    entries in shuffled insertion order, on the device (bp_build_problem: bounds, checks, sort,
    coalesce, CSR + CSC) from host arrays to host arrays, against the reference's own builder on the
    host (oracle/_ref). Wall time of the C-ABI call (host -> device -> host copies included)."""
    import ctypes as C

    from paper_2510_20499_b200 import _lib
    if rank != 0:
        return None
    n, m, N = p.n_vars, p.n_cons, p.nnz()
    rows = np.repeat(np.arange(m, dtype=np.int32), np.diff(p.row_start))
    perm = np.random.default_rng(11).permutation(N)
    er, ec, ev = (np.ascontiguousarray(a[perm]) for a in (rows, p.row_col, p.row_val))
    P = _lib.ptr
    ins = [np.ascontiguousarray(a) for a in (p.var_lower, p.var_upper, p.is_integer, p.cons_lower, p.cons_upper)]
    d = _lib.bp_builder_desc(n, m, N, P(er), P(ec), P(ev), *[P(a) for a in ins])
    outs = [np.zeros(m + 1, np.int32), np.zeros(N, np.int32), np.zeros(N), np.zeros(n + 1, np.int32),
            np.zeros(N, np.int32), np.zeros(N), np.zeros(n), np.zeros(n)]
    o = _lib.bp_built(0, *[P(a) for a in outs])
    L = _lib.lib()
    times = []
    for _ in range(4):  # first call warms up (allocations, module load)
        t0 = time.perf_counter()
        _lib.check(L.bp_build_problem(C.byref(d), int(local), C.byref(o), None))
        times.append(time.perf_counter() - t0)
    assert int(o.nnz) == N and np.array_equal(outs[1], p.row_col) and np.array_equal(outs[4], p.col_row)
    el = float(np.median(times[1:]))
    out = {"workload": "ProblemBuilder::build of C2 (1M x 1M, %d entries, shuffled)" % N,
           "build_ms": el * 1e3, "entries_per_s": N / el,
           "api": "bp_build_problem (C-ABI, host arrays in and out)",
           "parity": "bitwise vs the reference builder (tests/test_gpu_build.py, drop-in criterion)"}
    if world == 1 and not args.no_cpu_baseline:
        from oracle.bind import Ref
        if Ref.available():
            Q = lambda a: np.ascontiguousarray(a).ctypes.data_as(C.c_void_p)  # noqa: E731
            t0 = time.perf_counter()
            h = Ref.lib().ref_problem_build(n, m, Q(p.var_lower), Q(p.var_upper), Q(p.is_integer), None,
                                            Q(p.cons_lower), Q(p.cons_upper), N, Q(er), Q(ec), Q(ev))
            el_cpu = time.perf_counter() - t0
            Ref.lib().ref_problem_free(h)
            out["cpu_baseline"] = {"value": N / el_cpu, "unit": "entries/s", "cores": 1,
                                   "kind": "reference",
                                   "sample": f"pulse::ProblemBuilder::build of the same entries ({el_cpu:.2f} s)"}
    return out


def run_batch(args, rank, world, local):
    """configs[4]: 64 heterogeneous MIPLIB-shaped instances (10k-5M nnz), LPT-partitioned by size
    over the ranks; each rank uploads its instances and propagates them one after another on its
    GPU (device-resident bounds), one full `propagate` each. value = Σ reference-trajectory nnz
    visits of all instances / max-over-ranks device time."""
    import torch

    from paper_2510_20499_b200 import metrics, synth
    from paper_2510_20499_b200.propagation import FORCE_FRONTIER, device_problem, propagate_device

    specs = synth.c5_specs(count=args.c5_count)
    mine = synth.lpt_partition([sp[1] for sp in specs], world)[rank]
    log(f"batch: building {len(mine)} of {len(specs)} C5 instances")
    insts = []
    for j in mine:
        p = synth.c5_instance(specs[j])
        device_problem(p, device=local)
        insts.append(p)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    work = []
    visits = 0
    for p in insts:
        root = torch.from_numpy(p.root_bounds()).cuda()
        w = torch.empty_like(root)
        st = torch.zeros(64 * metrics.STAT_COLS, dtype=torch.int64, device="cuda")
        w.copy_(root)
        r, _ = propagate_device(p, w.data_ptr(), False, None, sptr, FORCE_FRONTIER, st.data_ptr())
        v = metrics.nnz_visits(metrics.trim(st.cpu().numpy(), r.rounds))
        visits += v
        work.append((p, root, w, v))
    log(f"batch: stats pass done, {visits} nnz visits")

    # instances are independent: `c5_streams` host threads each drive a share of them (largest
    # first) on their own CUDA stream, so small instances' grids run side by side
    from concurrent.futures import ThreadPoolExecutor
    nthr = max(1, min(args.c5_streams, len(work)))
    streams = [torch.cuda.Stream() for _ in range(nthr)]
    shares = [[] for _ in range(nthr)]
    loads = [0] * nthr
    for item in sorted(work, key=lambda x: -x[0].nnz()):
        j = loads.index(min(loads))
        shares[j].append(item)
        loads[j] += item[0].nnz()

    def run_share(j):
        st = streams[j]
        with torch.cuda.stream(st):
            for p, root, w, _ in shares[j]:
                w.copy_(root)
                propagate_device(p, w.data_ptr(), False, None, st.cuda_stream)

    pool = ThreadPoolExecutor(nthr)

    def sweep():  # noqa: E306
        ev = torch.cuda.Event()
        ev.record(stream)
        for st in streams:
            st.wait_event(ev)
        list(pool.map(run_share, range(nthr)))
        for st in streams:
            done = torch.cuda.Event()
            done.record(st)
            stream.wait_event(done)

    sweep()  # warm-up
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.c5_reps):
        sweep()
    e1.record(stream)
    torch.cuda.synchronize()
    pool.shutdown()
    ms = _max_over_ranks(e0.elapsed_time(e1) / args.c5_reps, world)
    tot_visits = _sum_over_ranks(visits, world)
    tot_nnz = int(_sum_over_ranks(sum(p.nnz() for p in insts), world))
    if rank != 0:
        return None
    out = {"workload": f"C5: {len(specs)} heterogeneous instances (C1-C4 generators, nnz log-uniform "
                       f"10k-5M), total nnz {tot_nnz}", "nnz_visits_per_s": tot_visits / (ms * 1e-3),
           "ms_per_sweep": ms, "nnz_visits_per_sweep": tot_visits, "n_gpus": world,
           "parallelism": f"LPT instance partition x{world}, no collective; {nthr} streams per GPU"}
    if world == 1 and not args.no_cpu_baseline:
        from oracle.bind import Ref, RefProblem, ref_propagate
        if Ref.available():
            done, v_cpu, el, bad = 0, 0, 0.0, []
            for p, _, w, v in sorted(work, key=lambda x: x[0].nnz()):
                rp = RefProblem.from_def(p)
                root = p.root_bounds()
                t1 = time.perf_counter()
                ob, oinf, ost, orr, ocr = ref_propagate(rp, root)
                el += time.perf_counter() - t1
                v_cpu += v
                done += 1
                del rp
                # parity: the device result of the timed sweeps (w) == the reference, bitwise
                if not np.array_equal(w.cpu().numpy().view(np.uint64), ob.view(np.uint64)):
                    bad.append(p.name)
            out["cpu_baseline"] = {"value": v_cpu / el, "unit": "nnz/s", "cores": int(Ref.lib().ref_max_threads()),
                                   "kind": "reference", "sample": f"reference propagate on {done} of "
                                                                  f"{len(work)} instances ({el:.1f} s)"}
            out["parity"] = {"instances_checked": done, "bound_mismatches": len(bad),
                             "against": "pulse::propagate (oracle/_ref), bounds bitwise"}
            assert not bad, f"C5 instances differ from the reference: {bad[:5]}"
    return out


def _sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2", choices=["C2", "C1"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-probing", action="store_true")
    ap.add_argument("--no-rounding", action="store_true")
    ap.add_argument("--cpu-sample-sec", type=float, default=20.0)
    ap.add_argument("--no-batch", action="store_true")
    ap.add_argument("--no-lp", action="store_true")
    ap.add_argument("--no-build", action="store_true")
    ap.add_argument("--round-deadline", type=float, default=0.0,
                    help="C4 propagation_round deadline (s), as the reference's Deadline; 0 = never")
    ap.add_argument("--c5-count", type=int, default=64)
    ap.add_argument("--c5-reps", type=int, default=3)
    ap.add_argument("--c5-streams", type=int, default=8)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = dist_env()
    if args.gpus != world:
        # one process per GPU: `python bench.py --gpus N` re-executes itself under torchrun; a
        # launcher whose WORLD_SIZE disagrees with --gpus, or too few GPUs, is an error (no
        # silent single-rank run)
        if "WORLD_SIZE" in os.environ:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        import torch
        ndev = torch.cuda.device_count() if args.impl == "ours" else args.gpus
        if ndev < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} requested, {ndev} GPU(s) visible")
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                   "--master-port", str(port), str(Path(__file__).resolve())]
                  + sys.argv[1:])

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2510_20499_b200 import BoundsState, metrics, propagate
    from paper_2510_20499_b200 import _lib
    from paper_2510_20499_b200.propagation import FORCE_FRONTIER, device_problem, propagate_device

    torch.cuda.set_device(local)
    from paper_2510_20499_b200 import set_device
    set_device(local)  # every problem / LP this rank uploads lives on its own GPU
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    log(f"generating {args.workload}")
    p, desc = make_workload(args.workload)
    log(f"generated n={p.n_vars} m={p.n_cons} nnz={p.nnz()}; uploading")
    dp = device_problem(p, device=local)
    n, m, N = p.n_vars, p.n_cons, p.nnz()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    d_root = torch.from_numpy(p.root_bounds()).cuda()
    d_work = torch.empty_like(d_root)

    # 1) exact-frontier stats pass: the reference trajectory's dirty sets, for the work counts
    d_stats = torch.zeros(64 * metrics.STAT_COLS, dtype=torch.int64, device="cuda")
    d_work.copy_(d_root)
    r_stats, _ = propagate_device(p, d_work.data_ptr(), False, None, sptr, FORCE_FRONTIER,
                                  d_stats.data_ptr())
    stats = metrics.trim(d_stats.cpu().numpy(), r_stats.rounds)
    log(f"stats pass done: rounds={r_stats.rounds}")
    ref_bits = d_work.cpu().numpy().view(np.uint64).copy()
    visits = metrics.nnz_visits(stats)
    alg_bytes = metrics.algorithmic_bytes(stats, n, m)

    def step():
        d_work.copy_(d_root)
        return propagate_device(p, d_work.data_ptr(), False, None, sptr)

    for _ in range(args.warmup):
        r, _ = step()
    torch.cuda.synchronize()
    # the fast path (full-round substitution) must reproduce the exact-frontier result bit for bit
    assert (r.status, r.rounds, r.crossed_vars) == (r_stats.status, r_stats.rounds, r_stats.crossed_vars)
    assert np.array_equal(d_work.cpu().numpy().view(np.uint64), ref_bits), "fast path != exact frontier"

    L = _lib.lib()
    import ctypes as C
    tot0, nl0 = C.c_double(), C.c_int64()
    L.bp_kernel_time(dp.h, None, C.byref(tot0), C.byref(nl0))
    launches0 = _lib.kernel_launches()
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t_wall0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = _lib.kernel_launches() - launches0
    tot1, nl1 = C.c_double(), C.c_int64()
    L.bp_kernel_time(dp.h, None, C.byref(tot1), C.byref(nl1))
    kern_ms = (tot1.value - tot0.value) / max(1, nl1.value - nl0.value)
    clocks = sampler.stop(t_wall0, t_wall1) if rank == 0 else None
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        kt = torch.tensor([kern_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(kt, op=dist.ReduceOp.MAX)
        kern_ms = float(kt.item())

    log(f"timed region done: {ms / args.steps:.3f} ms/step")
    # 2) e2e: host (pinned) bounds through the C-ABI call bp_propagate, H2D + D2H every step
    host_root = p.root_bounds()
    pinned = torch.empty(host_root.size, dtype=torch.float64).pin_memory()
    hb = pinned.numpy()
    e2e_times = []
    for i in range(args.e2e_steps + 2):
        hb[:] = host_root
        b = BoundsState(raw=hb)
        b.b = hb  # operate on the pinned buffer in place
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rr = propagate(p, b)
        t1 = time.perf_counter()
        if i >= 2:
            e2e_times.append(t1 - t0)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    log("e2e done")
    probing = None if args.no_probing else run_probing(args, rank, world, local)
    log("probing done")
    rounding = None if args.no_rounding else run_rounding(args, rank, world, local)
    log("rounding done")
    # (the builder runs before the C5 batch: after the batch's 64 resident problems and host
    # threads its pageable host<->device copies measured 3-4x slower, 79 -> 285 ms)
    lp = None if args.no_lp or args.workload != "C2" else run_lp(args, rank, world, local, p)
    log("lp done")
    build = None if args.no_build or args.workload != "C2" else run_build(args, rank, world, local, p)
    log("build done")
    batch = None if args.no_batch else run_batch(args, rank, world, local)
    log("batch done")

    if rank == 0:
        peak, peak_kind = peaks()
        achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
        # DRAM traffic needs a profiler pass (ncu), not run inside the timed bench: the committed
        # per-launch dram__bytes_read/write sum of one propagate of the same code
        # (tools/gpu_profiles.sh -> tools/ncu_traffic.py -> profiles/r02/ncu_traffic_summary.json)
        traffic = None
        tj = ROOT / "profiles" / "r02" / "ncu_traffic_summary.json"
        if tj.exists():
            traffic = json.loads(tj.read_text()).get("dram_bytes_per_launch", {}).get(args.workload)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            res = cpu_reference_propagate(p, reps=1)
            if res is not None:
                times, out, cores = res
                cpu = {"value": visits / times[0], "unit": "nnz/s", "cores": cores,
                       "kind": "reference",
                       "sample": f"1 full propagate of {args.workload} ({out[3]} rounds, "
                                 f"{times[0]:.2f} s), reference compiled from /root/reference"}
                assert out[3] == r.rounds and out[2] == int(r.status), "reference trajectory differs"
                assert np.array_equal(out[0].view(np.uint64), ref_bits), "C2 bounds differ from the reference"
                one = cpu_reference_single_thread(args.workload)
                if one is not None:
                    cpu["single_thread"] = {"value": visits / one, "unit": "nnz/s", "cores": 1,
                                            "sample": f"1 propagate of {args.workload} with PULSE_THREADS=1 "
                                                      f"({one:.2f} s)"}
        value = world * visits * args.steps / (ms * 1e-3)
        line = {
            "metric": "BP nnz/s", "value": value, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": desc, "n_vars": n, "n_cons": m, "nnz": N,
                       "rounds": r.rounds, "status": int(r.status),
                       "nnz_visits_per_step": visits, "algorithmic_bytes_per_step": alg_bytes,
                       "full_rounds_in_reference_trajectory": int(stats[:, 0].sum()),
                       "l2": "no flush: CSR+CSC inputs (%.0f MB) exceed the 126 MB L2" % (N * 24 / 1e6),
                       "parallelism": f"replicas x{world}"},
            "e2e": {"value": world * visits / e2e_s, "unit": "nnz/s",
                    "h2d_bytes_per_step": int(host_root.nbytes), "d2h_bytes_per_step": int(host_root.nbytes),
                    "ms_per_step": e2e_s * 1e3, "api": "bp_propagate (C-ABI, host pinned bounds)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "one propagate = k_engine (cooperative) + per full round "
                                   "k_rows_full + k_cand_pieces, CUDA events around the sequence",
                         "kernel_ms": kern_ms},
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "probing": probing,
            "rounding": rounding,
            "batch": batch,
            "lp": lp,
            "build": build,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
