// Block-per-branch probing (probing.hpp:194-238) for the branches the warp kernel cannot hold:
// frontiers larger than its shared-memory overlays (C4: dirty knapsack rows of 20k entries, whose
// variables all become dirty), and every branch of an UNCERTIFIED root, whose first round must be
// a full round (propagation.hpp:442; the frontier-start lemma of SURVEY §8a A12 needs a fixpoint).
//
// One thread block runs one branch at a time with its state DENSE in global memory (a per-block
// scratch of O(n + m) words, L2-resident for mid-size problems): bounds and activity overlays valid
// under a per-branch tag, dirty-row / dirty-var dedup stamps under per-round tags. No capacity
// limits, no hashing. The rounds are the reference's: activities of the dirty rows in fixed
// 16384-entry segments, Jacobi tightening of the dirty vars (all reads before any write), the
// std::min/max folds in CSC order, counts_as_change, crossing -> infeasible, the 64-round cap.
// Deltas = the written variables that differ from the root, ascending (probing.hpp:213-217).
#include <algorithm>
#include <cmath>

#include "bp_engine.cuh"
#include "bp_probe.cuh"

namespace bp {

namespace {

constexpr unsigned FULL   = 0xffffffffu;
constexpr int kBThreads   = 512;
constexpr int kBWarps     = kBThreads / 32;
constexpr int kLaneItem   = 64;    // rows / columns up to this length: one thread
constexpr int kSortCap    = 4096;  // deltas sorted in shared memory up to this count

constexpr int kHugeItem = 2048;  // rows / columns longer than this: the whole block

struct BSmem {
  int n_a, n_b, n_long, n_huge, crossed, n_touch, tag;
  int hugeq[kBThreads];
  double red[kBWarps][4];
  int redi[kBWarps][2];
  int red_ok;
  unsigned long long wa, wb;  // block work counters: row nnz and column nnz of the dirty sets
  int longq[kBThreads];
  double stage[kBWarps][64];
  int sortbuf[kSortCap];
};

// Bounds of var i in this branch: the overlay's if stamped, else the root's. (Issuing all three
// loads unconditionally measured slower on C4: the extra traffic outweighs the latency.)
__device__ __forceinline__ double2 bb_get(const ProbeRoot& R, const BlockScratch& W, int i, unsigned bt)
{
  return __ldcg(W.bst + i) == bt ? __ldcg(W.bnd + i) : R.bounds[i];
}

// Activity of row k (reference order: sequential within 16384-entry segments, segments in order).
__device__ void act_thread(const DevProblem& P, const ProbeRoot& R, const BlockScratch& W, unsigned bt,
                           int k, double& smn, int& imn, double& smx, int& imx)
{
  const int rs = __ldg(P.row_start + k), re = __ldg(P.row_start + k + 1);
  double pmn = 0.0, pmx = 0.0;
  imn = imx = 0;
  for (int e = rs; e < re; ++e) {
    const double2 b = bb_get(R, W, __ldg(P.row_col + e), bt);
    double cm, cx;
    int i1, i2;
    contrib(__ldg(P.row_val + e), b.x, b.y, cm, cx, i1, i2);
    pmn = __dadd_rn(pmn, cm);
    pmx = __dadd_rn(pmx, cx);
    imn += i1;
    imx += i2;
  }
  smn = __dadd_rn(0.0, pmn);
  smx = __dadd_rn(0.0, pmx);
}

// Integer-exact fast path: when every finite contribution of a chain is an integer
// and their absolute sum stays below 2^52, every partial sum of the reference's sequential fold is
// exact, so any summation order gives its bits (a warp tree here). The running sum starts at +0.0
// and is never -0.0; `+ 0.0` maps a tree's -0.0 (sum of -0.0 contributions) back to +0.0.
__device__ __forceinline__ bool exact_warp_sum(const DevProblem& P, const ProbeRoot& R,
                                               const BlockScratch& W, unsigned bt, int rs, int L,
                                               int lane, double& smn, double& smx, int& imn, int& imx)
{
  double sm = 0.0, sx = 0.0, am = 0.0, ax = 0.0;
  int cmn = 0, cmx = 0;
  bool ok = true;
  for (int j = lane; j < L; j += 32) {
    const double2 b = bb_get(R, W, __ldg(P.row_col + rs + j), bt);
    double cm, cx;
    int i1, i2;
    contrib(__ldg(P.row_val + rs + j), b.x, b.y, cm, cx, i1, i2);
    ok = ok && cm == rint(cm) && cx == rint(cx);
    sm += cm;
    sx += cx;
    am += fabs(cm);
    ax += fabs(cx);
    cmn += i1;
    cmx += i2;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sm += __shfl_xor_sync(FULL, sm, o);
    sx += __shfl_xor_sync(FULL, sx, o);
    am += __shfl_xor_sync(FULL, am, o);
    ax += __shfl_xor_sync(FULL, ax, o);
    cmn += __shfl_xor_sync(FULL, cmn, o);
    cmx += __shfl_xor_sync(FULL, cmx, o);
  }
  ok = __all_sync(FULL, ok) && am < 0x1p52 && ax < 0x1p52;
  if (!ok) return false;
  smn = sm + 0.0;
  smx = sx + 0.0;
  imn = cmn;
  imx = cmx;
  return true;
}

__device__ void act_warp(const DevProblem& P, const ProbeRoot& R, const BlockScratch& W, unsigned bt,
                         int k, double* stage, int lane, double& smn, int& imn, double& smx, int& imx)
{
  const int rs = __ldg(P.row_start + k), L = __ldg(P.row_start + k + 1) - rs;
  if (exact_warp_sum(P, R, W, bt, rs, L, lane, smn, smx, imn, imx)) return;
  double tot = 0.0, part = 0.0;
  int cmn = 0, cmx = 0;
  for (int base = 0; base < L; base += 32) {
    if (base > 0 && (base % kSumSegment) == 0) {
      tot  = __dadd_rn(tot, part);
      part = 0.0;
    }
    const int j = base + lane;
    double cm = 0.0, cx = 0.0;
    if (j < L) {
      const double2 b = bb_get(R, W, __ldg(P.row_col + rs + j), bt);
      int i1, i2;
      contrib(__ldg(P.row_val + rs + j), b.x, b.y, cm, cx, i1, i2);
      cmn += i1;
      cmx += i2;
    }
    stage[lane]      = cm;
    stage[32 + lane] = cx;
    __syncwarp();
    if (lane < 2) {
      const int cnt = min(32, L - base);
      for (int q = 0; q < cnt; ++q) part = __dadd_rn(part, stage[32 * lane + q]);
    }
    __syncwarp();
  }
  tot = __dadd_rn(tot, part);
  smn = __shfl_sync(FULL, tot, 0);
  smx = __shfl_sync(FULL, tot, 1);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    cmn += __shfl_xor_sync(FULL, cmn, o);
    cmx += __shfl_xor_sync(FULL, cmx, o);
  }
  imn = cmn;
  imx = cmx;
}

// Activity of a huge row by the whole block: the integer-exact tree (see exact_warp_sum) when it
// applies, else the reference's sequential fold by the first warp.
__device__ void act_block(const DevProblem& P, const ProbeRoot& R, const BlockScratch& W, BSmem& sm,
                          unsigned bt, int k, double& smn, int& imn, double& smx, int& imx)
{
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rs = __ldg(P.row_start + k), L = __ldg(P.row_start + k + 1) - rs;
  double s0 = 0.0, s1 = 0.0, a0 = 0.0, a1 = 0.0;
  int c0 = 0, c1 = 0;
  bool ok = true;
#pragma unroll 4
  for (int j = tid; j < L; j += kBThreads) {
    const double2 b = bb_get(R, W, __ldg(P.row_col + rs + j), bt);
    double cm, cx;
    int i1, i2;
    contrib(__ldg(P.row_val + rs + j), b.x, b.y, cm, cx, i1, i2);
    ok = ok && cm == rint(cm) && cx == rint(cx);
    s0 += cm;
    s1 += cx;
    a0 += fabs(cm);
    a1 += fabs(cx);
    c0 += i1;
    c1 += i2;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s0 += __shfl_xor_sync(FULL, s0, o);
    s1 += __shfl_xor_sync(FULL, s1, o);
    a0 += __shfl_xor_sync(FULL, a0, o);
    a1 += __shfl_xor_sync(FULL, a1, o);
    c0 += __shfl_xor_sync(FULL, c0, o);
    c1 += __shfl_xor_sync(FULL, c1, o);
  }
  const bool wok = __all_sync(FULL, ok);
  if (tid == 0) sm.red_ok = 1;
  __syncthreads();
  if (lane == 0) {
    sm.red[warp][0] = s0;
    sm.red[warp][1] = s1;
    sm.red[warp][2] = a0;
    sm.red[warp][3] = a1;
    sm.redi[warp][0] = c0;
    sm.redi[warp][1] = c1;
    if (!wok) sm.red_ok = 0;
  }
  __syncthreads();
  double t0 = 0.0, t1 = 0.0, u0 = 0.0, u1 = 0.0;
  int d0 = 0, d1 = 0;
  for (int q = 0; q < kBWarps; ++q) {  // every thread folds the 16 partials the same way
    t0 += sm.red[q][0];
    t1 += sm.red[q][1];
    u0 += sm.red[q][2];
    u1 += sm.red[q][3];
    d0 += sm.redi[q][0];
    d1 += sm.redi[q][1];
  }
  const bool exact = sm.red_ok && u0 < 0x1p52 && u1 < 0x1p52;
  __syncthreads();
  if (exact) {
    smn = t0 + 0.0;
    smx = t1 + 0.0;
    imn = d0;
    imx = d1;
    return;
  }
  if (warp == 0) act_warp(P, R, W, bt, k, sm.stage[0], lane, smn, imn, smx, imx);
}

__device__ __forceinline__ void act_get(const DevProblem& P, const ProbeRoot& R, const BlockScratch& W,
                                        unsigned bt, int k, double& mnf, int& nmn, double& mxf,
                                        int& nmx, double& g, double& h)
{
  const double2 cb = __ldg(&P.cons[k]);
  g                = cb.y;
  h                = cb.x;
  if (__ldcg(W.ast + k) == bt) {
    const double2 a = __ldcg(W.act + k);
    const int2 c    = __ldcg(W.ainf + k);
    mnf = a.x;
    mxf = a.y;
    nmn = c.x;
    nmx = c.y;
  } else {
    const RowRec r = ld_rec(R.rec + k);
    decode_rec(r, R.aux, k, mnf, nmn, mxf, nmx);
  }
}

__device__ void fold_thread(const DevProblem& P, const ProbeRoot& R, const BlockScratch& W, unsigned bt,
                            int i, double lo, double up, bool integer, double& nl, double& nu)
{
  nl = lo;
  nu = up;
  const int cs = __ldg(P.col_start + i), ce = __ldg(P.col_start + i + 1);
  for (int e = cs; e < ce; ++e) {
    const int k = __ldg(P.col_row + e);
    double mnf, mxf, g, h, cl, cu;
    int nmn, nmx;
    act_get(P, R, W, bt, k, mnf, nmn, mxf, nmx, g, h);
    cand_explicit(lo, up, integer, __ldg(P.col_val + e), mnf, nmn, mxf, nmx, g, h, cl, cu);
    if (cu < nu) nu = cu;
    if (nl < cl) nl = cl;
  }
}

__device__ void fold_warp(const DevProblem& P, const ProbeRoot& R, const BlockScratch& W, unsigned bt,
                          int i, double lo, double up, bool integer, int lane, double& nl, double& nu)
{
  const int cs = __ldg(P.col_start + i), ce = __ldg(P.col_start + i + 1);
  Fold f{lo, -1, up, -1};
  for (int e = cs + lane; e < ce; e += 32) {
    const int k = __ldg(P.col_row + e);
    double mnf, mxf, g, h, cl, cu;
    int nmn, nmx;
    act_get(P, R, W, bt, k, mnf, nmn, mxf, nmx, g, h);
    cand_explicit(lo, up, integer, __ldg(P.col_val + e), mnf, nmn, mxf, nmx, g, h, cl, cu);
    if (cu < f.up) { f.up = cu; f.up_pos = e; }
    if (f.lo < cl) { f.lo = cl; f.lo_pos = e; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double olo = __shfl_xor_sync(FULL, f.lo, o);
    const int olp    = __shfl_xor_sync(FULL, f.lo_pos, o);
    const double oup = __shfl_xor_sync(FULL, f.up, o);
    const int oupp   = __shfl_xor_sync(FULL, f.up_pos, o);
    fold_combine(f, olo, olp, oup, oupp);
  }
  nl = f.lo;
  nu = f.up;
}

// Runs body(item, mode, idx, stride) over items list[0..cnt) (or 0..cnt when list == nullptr):
// mode 0 -- items whose range in `start` is <= kLaneItem, by one thread (idx 0, stride 1);
// mode 1 -- up to kHugeItem, by one warp (idx = lane, stride 32);
// mode 2 -- longer, by the whole block one after another (idx = thread, stride = block size; every
//           thread calls body, so it may use __syncthreads).
template <class F>
__device__ __forceinline__ void block_items(BSmem& sm, const int* list, int cnt, const int* start, F body)
{
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int base = 0; base < cnt; base += kBThreads) {
    const int j   = base + tid;
    const int it  = j < cnt ? (list ? list[j] : j) : -1;
    const int len = it >= 0 ? __ldg(start + it + 1) - __ldg(start + it) : 0;
    if (it >= 0 && len <= kLaneItem) body(it, 0, 0, 1);
    if (it >= 0 && len > kLaneItem && len <= kHugeItem) sm.longq[atomicAdd(&sm.n_long, 1)] = it;
    if (it >= 0 && len > kHugeItem) sm.hugeq[atomicAdd(&sm.n_huge, 1)] = it;
    __syncthreads();
    const int nl = sm.n_long, nh = sm.n_huge;
    for (int q = warp; q < nl; q += kBWarps) body(sm.longq[q], 1, lane, 32);
    __syncthreads();
    for (int q = 0; q < nh; ++q) body(sm.hugeq[q], 2, tid, kBThreads);
    __syncthreads();
    if (tid == 0) sm.n_long = sm.n_huge = 0;
    __syncthreads();
  }
}

__device__ __forceinline__ unsigned next_tag(BSmem& sm)
{
  __syncthreads();
  if (threadIdx.x == 0) sm.tag = sm.tag + 1;
  __syncthreads();
  return (unsigned)sm.tag;
}

// One branch on this block. Returns 0 feasible, 1 infeasible; *n_touch = written variables.
__device__ int block_branch(const DevProblem& P, const ProbeRoot& R, const BlockScratch& W, BSmem& sm,
                            const Limits& lim, int v, double blo, double bup, bool full_first,
                            unsigned& bt, unsigned long long* wk)
{
  const int tid = threadIdx.x;
  bt            = next_tag(sm);
  const double2 rb = R.bounds[v];
  const double2 nb = make_double2(smax(rb.x, blo), smin(rb.y, bup));
  if (nb.x > nb.y) return 1;  // probing.hpp:205-206
  if (tid == 0) {
    W.bnd[v]   = nb;
    W.bst[v]   = bt;
    W.touch[0] = v;
    W.chg[0]   = v;
    sm.n_touch = 1;
    sm.n_a     = 1;  // changed list: {v}
    sm.crossed = 0;
  }
  __syncthreads();
  int rounds = 0;
  for (;;) {
    const bool full = full_first && rounds == 0;
    int nr = P.m, nv = P.n;
    const int* rl = nullptr;
    const int* vl = nullptr;
    if (!full) {
      // frontier: rows(changed) -> drow, vars(drow) -> dvar (stamp-deduplicated)
      const unsigned rt = next_tag(sm);
      const int nch     = sm.n_a;
      if (tid == 0) sm.n_b = 0;
      __syncthreads();
      block_items(sm, W.chg, nch, P.col_start, [&](int i, int mode, int idx, int stride) {
        const int cs = __ldg(P.col_start + i), ce = __ldg(P.col_start + i + 1);
        for (int e = cs + idx; e < ce; e += stride) {
          const int k = __ldg(P.col_row + e);
          if (atomicExch(W.rmark + k, rt) != rt) W.drow[atomicAdd(&sm.n_b, 1)] = k;
        }
      });
      nr = sm.n_b;
      if (nr == 0) return 0;                   // dirty_rows.empty() (propagation.hpp:481)
      if (rounds >= lim.max_rounds) return 0;
      rl = W.drow;
    }
    ++rounds;
    // activities of the dirty rows (from the round-start bounds)
    block_items(sm, rl, nr, P.row_start, [&](int k, int mode, int idx, int stride) {
      double smn, smx;
      int imn, imx;
      bool writer = idx == 0;
      if (mode == 2) act_block(P, R, W, sm, bt, k, smn, imn, smx, imx);
      else if (mode == 1) act_warp(P, R, W, bt, k, sm.stage[threadIdx.x >> 5], idx, smn, imn, smx, imx);
      else act_thread(P, R, W, bt, k, smn, imn, smx, imx);
      if (writer) {
        W.act[k]  = make_double2(smn, smx);
        W.ainf[k] = make_int2(imn, imx);
        __threadfence_block();
        W.ast[k] = bt;
      }
    });
    // the vars to re-evaluate: vars of the dirty rows (propagation.hpp:476-479) whose candidate from
    // a dirty row is not provably non-improving (candidate gating, bp_device.cuh entry_quiet). A var
    // whose every dirty row is quiet for it folds to its current bounds -- its clean rows give the
    // candidates of its last evaluation, which made no change -- so skipping it is exact.
    {
      const unsigned vt = next_tag(sm);
      if (tid == 0) sm.n_a = 0;
      __syncthreads();
      block_items(sm, rl, nr, P.row_start, [&](int k, int mode, int idx, int stride) {
        double mnf, mxf, g, h;
        int nmn, nmx;
        act_get(P, R, W, bt, k, mnf, nmn, mxf, nmx, g, h);
        const int rs = __ldg(P.row_start + k), re = __ldg(P.row_start + k + 1);
#pragma unroll 4
        for (int e = rs + idx; e < re; e += stride) {
          const int i     = __ldg(P.row_col + e);
          const double2 b = bb_get(R, W, i, bt);
          double tw, pm;
          entry_reach(__ldg(P.row_val + e), b.x, b.y, __ldg(P.is_int + i) != 0, tw, pm);
          if (entry_quiet(tw, pm, mnf, nmn, mxf, nmx, g, h)) continue;
          if (atomicExch(W.vmark + i, vt) != vt) W.dvar[atomicAdd(&sm.n_a, 1)] = i;
        }
      });
      nv = sm.n_a;
      vl = W.dvar;
    }
    if (tid == 0) {  // work of this round (thread 0; R, V here, A and B below)
      wk[0] += nr;
      wk[2] += nv;
    }
    {
      unsigned long long a = 0, bs = 0;
      for (int j = tid; j < nr; j += kBThreads) {
        const int k = rl ? rl[j] : j;
        a += __ldg(P.row_start + k + 1) - __ldg(P.row_start + k);
      }
      for (int j = tid; j < nv; j += kBThreads) {
        const int i = vl[j];
        bs += __ldg(P.col_start + i + 1) - __ldg(P.col_start + i);
      }
      if (a) atomicAdd(&sm.wa, a);
      if (bs) atomicAdd(&sm.wb, bs);
    }
    // Jacobi tightening of the dirty vars: new values to the changed list, written afterwards
    __syncthreads();  // every thread has read nv = n_a
    if (tid == 0) sm.n_a = 0;
    __syncthreads();
    block_items(sm, vl, nv, P.col_start, [&](int i, int mode, int idx, int stride) {
      const double2 b    = bb_get(R, W, i, bt);
      const bool integer = __ldg(P.is_int + i) != 0;
      double nl, nu;
      if (mode == 0) {
        fold_thread(P, R, W, bt, i, b.x, b.y, integer, nl, nu);
      } else if (mode == 1 || threadIdx.x < 32) {  // huge columns: the block's first warp
        fold_warp(P, R, W, bt, i, b.x, b.y, integer, idx & 31, nl, nu);
      }
      if (idx == 0) {
        double2 out = b;
        const int r = finish_var(&out, b.x, b.y, nl, nu, integer, lim);
        if (r < 0) atomicAdd(&sm.crossed, 1);
        if (r > 0) {
          const int pos = atomicAdd(&sm.n_a, 1);
          W.chg[pos]    = i;
          W.chgv[pos]   = out;
        }
      }
    });
    if (sm.crossed > 0) return 1;  // propagation.hpp:448-452
    const int nc = sm.n_a;
    if (tid == 0) wk[4] += nc;
    if (nc == 0) return 0;         // fixpoint (propagation.hpp:453)
    for (int j = tid; j < nc; j += kBThreads) {
      const int i = W.chg[j];
      if (__ldcg(W.bst + i) != bt) W.touch[atomicAdd(&sm.n_touch, 1)] = i;
      W.bnd[i] = W.chgv[j];
      W.bst[i] = bt;
    }
    __syncthreads();
    if (rounds >= lim.max_rounds) return 0;
  }
}

__global__ void __launch_bounds__(kBThreads, 1)
    k_probe_block(DevProblem P, ProbeRoot R, ProbeBatch B, Limits lim, BlockScratch W0, int full_first)
{
  __shared__ BSmem sm;
  BlockScratch W = W0.for_block(blockIdx.x);
  const int tid  = threadIdx.x;
  unsigned long long wk[5] = {0, 0, 0, 0, 0};  // thread 0's work counters (R, -, V, -, C)
  if (tid == 0) {
    sm.tag    = (int)*W.tagc;
    sm.n_long = 0;
    sm.n_huge = 0;
    sm.wa = sm.wb = 0;
  }
  __syncthreads();
  for (;;) {
    __shared__ int t_sh;
    if (tid == 0) t_sh = atomicAdd(B.cursor, 1);
    __syncthreads();
    const int t = t_sh;
    __syncthreads();
    if (t >= B.n_task) break;
    unsigned bt      = 0;
    const int status = block_branch(P, R, W, sm, lim, B.var[t], B.lo[t], B.up[t], full_first != 0, bt, wk);
    __syncthreads();
    // deltas: written variables that differ from the root, ascending by var
    const int nt = sm.n_touch;
    int cnt      = 0;
    if (status == 0) {
      if (tid == 0) sm.n_b = 0;
      __syncthreads();
      for (int j = tid; j < nt; j += kBThreads) {
        const int i     = W.touch[j];
        const double2 b = __ldcg(W.bnd + i), r = R.bounds[i];
        if (b.x != r.x || b.y != r.y) W.dvar[atomicAdd(&sm.n_b, 1)] = i;
      }
      __syncthreads();
      cnt = sm.n_b;
    }
    __shared__ long long base_sh;
    if (tid == 0) {
      long long base = 0;
      if (cnt) base = (long long)atomicAdd(B.pool_cursor, (unsigned long long)cnt);
      B.status[t] = status;
      B.dcount[t] = cnt;
      B.doff[t]   = base;
      if (status == 0 && cnt && base + cnt > B.pool_cap) B.status[t] = 3;  // host grows and reruns
      base_sh = base;
    }
    __syncthreads();
    const long long base = base_sh;
    if (status == 0 && cnt && base + cnt <= B.pool_cap) {
      if (cnt <= kSortCap) {  // bitonic sort of the delta vars in shared memory
        int np2 = 1;
        while (np2 < cnt) np2 <<= 1;
        for (int j = tid; j < np2; j += kBThreads) sm.sortbuf[j] = j < cnt ? W.dvar[j] : 0x7FFFFFFF;
        __syncthreads();
        for (int ksz = 2; ksz <= np2; ksz <<= 1)
          for (int jj = ksz >> 1; jj > 0; jj >>= 1) {
            for (int x = tid; x < np2; x += kBThreads) {
              const int y = x ^ jj;
              if (y > x) {
                const int a = sm.sortbuf[x], b = sm.sortbuf[y];
                if (((x & ksz) == 0) == (a > b)) {
                  sm.sortbuf[x] = b;
                  sm.sortbuf[y] = a;
                }
              }
            }
            __syncthreads();
          }
        for (int j = tid; j < cnt; j += kBThreads) {
          const int i     = sm.sortbuf[j];
          const double2 b = __ldcg(W.bnd + i);
          B.pvar[base + j] = i;
          B.plo[base + j]  = b.x;
          B.pup[base + j]  = b.y;
        }
      } else {  // large: ordered sweep over all variables (block scan of the flags)
        __shared__ int wsum[kBWarps + 1];
        int run = 0;
        for (int i0 = 0; i0 < P.n; i0 += kBThreads) {
          const int i = i0 + tid;
          bool d      = false;
          double2 b   = make_double2(0.0, 0.0);
          if (i < P.n && __ldcg(W.bst + i) == bt) {
            b                = __ldcg(W.bnd + i);
            const double2 r  = R.bounds[i];
            d                = b.x != r.x || b.y != r.y;
          }
          const unsigned m = __ballot_sync(FULL, d);
          if ((tid & 31) == 0) wsum[tid >> 5] = __popc(m);
          __syncthreads();
          if (tid == 0) {
            int acc = 0;
            for (int q = 0; q < kBWarps; ++q) {
              const int c = wsum[q];
              wsum[q]     = acc;
              acc += c;
            }
            wsum[kBWarps] = acc;
          }
          __syncthreads();
          if (d) {
            const long long o = base + run + wsum[tid >> 5] + __popc(m & ((1u << (tid & 31)) - 1u));
            B.pvar[o] = i;
            B.plo[o]  = b.x;
            B.pup[o]  = b.y;
          }
          run += wsum[kBWarps];
          __syncthreads();
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    *W.tagc = (unsigned)sm.tag;
    if (B.work) {
      wk[1] = sm.wa;
      wk[3] = sm.wb;
      for (int q = 0; q < 5; ++q)
        if (wk[q]) atomicAdd(B.work + q, wk[q]);
    }
  }
}

}  // namespace

size_t block_scratch_bytes(int n, int m)
{
  const size_t nn = (size_t)std::max(n, 1), mm = (size_t)std::max(m, 1);
  auto r = [](size_t b) { return (b + 15) / 16 * 16; };
  return 2 * r(16 * nn) + r(16 * mm) + r(8 * mm) + 5 * r(4 * nn) + 3 * r(4 * mm) + 16 + 256;
}

void probe_block_launch(Problem& Pr, const ProbeRoot& R, ProbeBatch& B, const Limits& lim,
                        BlockScratch& W, int full_first, cudaStream_t s)
{
  k_probe_block<<<W.nblocks, kBThreads, 0, s>>>(Pr.dev(), R, B, lim, W, full_first);
  BP_CUDA(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace bp
