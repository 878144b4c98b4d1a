// Persistent, device-resident bound propagation for sm_100a.
//
// One cooperative kernel runs the whole `propagate` loop of the reference
// (propagation.hpp:418-486) with no host round trip per round:
//
//   round r:  Phase A  row activities      (propagation.hpp:226-251)   ─ grid.sync
//             Phase B  bound tightening    (propagation.hpp:378-412)   ─ grid.sync
//             decision: infeasible / fixpoint / round cap / empty frontier (uniform on every block)
//             Phase C  frontier: changed vars → dirty rows (+ segment/expansion tasks)  ─ grid.sync
//             Phase D  dirty rows → dirty vars                                            ─ grid.sync
//
// Work partition (replaces the reference's LRB bins, propagation.hpp:97-141):
//   rows  nnz <= 32        one lane per row, sequential fold (exact reference order)
//         32 < nnz <= 2048 one warp per row: lanes gather/multiply, lanes 0/1 fold min/max chains
//         nnz > 2048       one producer/consumer warp PAIR per 16384-entry segment; the last
//                          segment to finish sums the partials in segment order (heavy_row_activity,
//                          propagation.hpp:197-218) — identical bits to the sequential sum.
//   vars  col nnz <= 32    one lane per var, sequential CSC fold
//         col nnz > 32     one warp per var; the std::min/max fold is reduced as a lexicographic
//                          (value, CSC position) min/max, which reproduces "first operand wins on
//                          ties" (sign of tied zeros) exactly.
// Frontier rounds (propagation.hpp:456-479) touch only dirty rows / dirty vars; when the frontier
// would cover a large fraction of the matrix the engine runs a full round instead — evaluating a
// superset of the dirty sets yields bit-identical results (SURVEY §8a A12 lemma).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "bp_engine.cuh"

namespace cg = cooperative_groups;

namespace bp {

long long g_kernel_launches = 0;

namespace {

constexpr int kThreads   = 256;
constexpr int kWarps     = kThreads / 32;
constexpr int kPairs     = kWarps / 2;
constexpr unsigned FULL  = 0xffffffffu;
constexpr int kXChunk    = 256;  // entries per var-expansion task

__device__ __forceinline__ unsigned lanemask_lt()
{
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ void named_bar(int id, int count)
{
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ int warp_sum(int v)
{
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer()
{
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_volatile(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p)
{
  return *(const volatile unsigned long long*)p;
}

struct Smem {
  double pair_buf[kPairs][2][2][64];  // [pair][buffer][chain][entry]
  int pair_cnt[kPairs][2][2];
  int pair_inf[kPairs][2];
  double warp_buf[kWarps][2][128];    // medium-row fold staging
  int chg[kWarps][64];                // changed-var staging before a global append
  int blk_crossed;
  int blk_any_rows;
  unsigned long long blk_colnnz;
  int fetch[kWarps];
};

struct Ctx {
  const DevProblem& P;
  const DevState& S;
  const Limits& lim;
  Smem& sm;
  int lane, warp, gwarp, nwarps;
};

// ------------------------------------------------------------------ row activities

__device__ __forceinline__ void write_rec(const DevProblem& P, const DevState& S, int k, double smn,
                                          double smx, int imn, int imx)
{
  const double2 c = __ldg(&P.cons[k]);
  RowRec r;
  r.min = imn ? box_count(imn) : smn;
  r.max = imx ? box_count(imx) : smx;
  r.g   = c.y;
  r.h   = c.x;
  st_rec(S.rec + k, r);
  if (imn | imx) S.aux[k] = make_double2(smn, smx);
}

// nnz <= 32: one lane, sequential (single segment: total = 0.0 + part = part, part != -0.0).
__device__ void row_activity_lane(const DevProblem& P, const DevState& S, int k)
{
  const int rs = __ldg(P.row_start + k), re = __ldg(P.row_start + k + 1);
  double smn = 0.0, smx = 0.0;
  int imn = 0, imx = 0;
#pragma unroll 4
  for (int e = rs; e < re; ++e) {
    const int c    = __ldg(P.row_col + e);
    const double a = __ldg(P.row_val + e);
    const double2 b = S.bounds[c];
    double cmn, cmx;
    int i1, i2;
    contrib(a, b.x, b.y, cmn, cmx, i1, i2);
    smn = __dadd_rn(smn, cmn);
    smx = __dadd_rn(smx, cmx);
    imn += i1;
    imx += i2;
  }
  write_rec(P, S, k, smn, smx, imn, imx);
}

// 32 < nnz <= 2048: one warp; lanes produce 128 contributions per step, lanes 0/1 fold.
__device__ void row_activity_warp(Ctx& c, int k)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  double(*wb)[128]    = c.sm.warp_buf[c.warp];
  const int rs = __ldg(P.row_start + k), L = __ldg(P.row_start + k + 1) - rs;
  double acc = 0.0;
  int imn = 0, imx = 0;
  for (int base = 0; base < L; base += 128) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int j = base + h * 32 + c.lane;
      double cmn = 0.0, cmx = 0.0;
      if (j < L) {
        const int col  = __ldg(P.row_col + rs + j);
        const double a = __ldg(P.row_val + rs + j);
        const double2 b = S.bounds[col];
        int i1, i2;
        contrib(a, b.x, b.y, cmn, cmx, i1, i2);
        imn += i1;
        imx += i2;
      }
      wb[0][h * 32 + c.lane] = cmn;
      wb[1][h * 32 + c.lane] = cmx;
    }
    __syncwarp();
    if (c.lane < 2) {
      const int cnt     = min(128, L - base);
      const double* src = wb[c.lane];
#pragma unroll 8
      for (int j = 0; j < cnt; ++j) acc = __dadd_rn(acc, src[j]);
    }
    __syncwarp();
  }
  imn = warp_sum(imn);
  imx = warp_sum(imx);
  const double smx = __shfl_sync(FULL, acc, 1);
  if (c.lane == 0) write_rec(P, S, k, acc, smx, imn, imx);
}

// nnz > 2048: producer warp computes and zero-compacts contributions of 64 entries per step into a
// double buffer; consumer lanes 0/1 fold the min/max chains in entry order. Skipping zero
// contributions is exact: the running sum starts at +0.0 and is never -0.0.
__device__ void row_segment_pair(Ctx& c, int k, int seg, bool producer, int pair)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  double(*pb)[2][64]  = c.sm.pair_buf[pair];
  int(*pcnt)[2]       = c.sm.pair_cnt[pair];
  int* pinf           = c.sm.pair_inf[pair];
  const int bar       = 1 + pair;
  const int rs = __ldg(P.row_start + k), L = __ldg(P.row_start + k + 1) - rs;
  const int e0 = seg * kSumSegment, e1 = min(L, e0 + kSumSegment);
  const int nch = (e1 - e0 + 63) >> 6;
  double acc = 0.0;
  int imn = 0, imx = 0;
  const unsigned lt = lanemask_lt();
  for (int step = 0; step <= nch; ++step) {
    if (producer) {
      if (step < nch) {
        const int bb = step & 1, base = e0 + (step << 6);
        double cm[2], cx[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = base + h * 32 + c.lane;
          cm[h] = 0.0;
          cx[h] = 0.0;
          if (e < e1) {
            const int col  = __ldg(P.row_col + rs + e);
            const double a = __ldg(P.row_val + rs + e);
            const double2 b = S.bounds[col];
            int i1, i2;
            contrib(a, b.x, b.y, cm[h], cx[h], i1, i2);
            imn += i1;
            imx += i2;
          }
        }
        const unsigned m0 = __ballot_sync(FULL, cm[0] != 0.0);
        const unsigned m1 = __ballot_sync(FULL, cm[1] != 0.0);
        const unsigned x0 = __ballot_sync(FULL, cx[0] != 0.0);
        const unsigned x1 = __ballot_sync(FULL, cx[1] != 0.0);
        if (cm[0] != 0.0) pb[bb][0][__popc(m0 & lt)] = cm[0];
        if (cm[1] != 0.0) pb[bb][0][__popc(m0) + __popc(m1 & lt)] = cm[1];
        if (cx[0] != 0.0) pb[bb][1][__popc(x0 & lt)] = cx[0];
        if (cx[1] != 0.0) pb[bb][1][__popc(x0) + __popc(x1 & lt)] = cx[1];
        if (c.lane == 0) {
          pcnt[bb][0] = __popc(m0) + __popc(m1);
          pcnt[bb][1] = __popc(x0) + __popc(x1);
        }
      }
    } else if (step >= 1 && c.lane < 2) {
      const int bb      = (step - 1) & 1;
      const int cnt     = pcnt[bb][c.lane];
      const double* src = pb[bb][c.lane];
#pragma unroll 4
      for (int j = 0; j < cnt; ++j) acc = __dadd_rn(acc, src[j]);
    }
    named_bar(bar, 64);
  }
  if (producer) {
    imn = warp_sum(imn);
    imx = warp_sum(imx);
    if (c.lane == 0) {
      pinf[0] = imn;
      pinf[1] = imx;
    }
  }
  named_bar(bar, 64);
  if (!producer) {
    const double smx = __shfl_sync(FULL, acc, 1);
    if (c.lane == 0) {
      const int nseg = (L + kSumSegment - 1) / kSumSegment;
      if (nseg == 1) {
        write_rec(P, S, k, acc, smx, pinf[0], pinf[1]);
      } else {
        const int base = __ldg(P.seg_base + k);
        SegPart sp;
        sp.min  = acc;
        sp.max  = smx;
        sp.nmin = pinf[0];
        sp.nmax = pinf[1];
        sp.pad0 = sp.pad1 = 0;
        S.seg_part[base + seg] = sp;
        __threadfence();
        const int done = atomicAdd(&S.seg_done[k], 1);
        if (done == nseg - 1) {
          __threadfence();
          double tmn = 0.0, tmx = 0.0;
          int cmn = 0, cmx = 0;
          for (int s = 0; s < nseg; ++s) {  // row_activity's segment fold (propagation.hpp:182-188)
            const SegPart* q = S.seg_part + base + s;
            tmn = __dadd_rn(tmn, __ldcg(&q->min));
            tmx = __dadd_rn(tmx, __ldcg(&q->max));
            cmn += __ldcg(&q->nmin);
            cmx += __ldcg(&q->nmax);
          }
          write_rec(P, S, k, tmn, tmx, cmn, cmx);
          S.seg_done[k] = 0;
        }
      }
    }
  }
  named_bar(bar, 64);
}

// Dynamic work cursor shared by a warp.
__device__ __forceinline__ int warp_fetch(Ctx& c, int* cursor, int step)
{
  int t = 0;
  if (c.lane == 0) t = atomicAdd(cursor, step);
  return __shfl_sync(FULL, t, 0);
}

// Phase A. full: every row from the static partition tables; else: the frontier lists.
__device__ void phase_activity(Ctx& c, ParCtl* pc, bool full)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int par       = (&c.S.ctl->par[1] == pc) ? 1 : 0;
  // 1) segment tasks (longest rows first) on warp pairs, static stride.
  {
    const int n_seg   = full ? P.n_seg : ld_volatile(&pc->n_dseg);
    const int2* tasks = full ? P.seg_task : S.dseg[par];
    const int pair    = c.warp >> 1;
    const bool prod   = (c.warp & 1) == 0;
    const int gpair   = blockIdx.x * kPairs + pair;
    const int npairs  = gridDim.x * kPairs;
    for (int t = gpair; t < n_seg; t += npairs) {
      const int2 tk = tasks[t];
      row_segment_pair(c, tk.x, tk.y, prod, pair);
    }
  }
  // 2) medium rows, one warp each (dynamic).
  {
    const int n    = full ? P.n_mrow : ld_volatile(&pc->n_drow_m);
    const int* ids = full ? P.mrow : S.drow_m[par];
    for (int t = warp_fetch(c, &pc->cur_m, 1); t < n; t = warp_fetch(c, &pc->cur_m, 1))
      row_activity_warp(c, full ? __ldg(ids + t) : ids[t]);
  }
  // 3) short rows, one lane each, tiles of 32 (dynamic).
  {
    const int n    = full ? P.n_srow : ld_volatile(&pc->n_drow_s);
    const int* ids = full ? P.srow : S.drow_s[par];
    for (int t = warp_fetch(c, &pc->cur_s, 32); t < n; t = warp_fetch(c, &pc->cur_s, 32)) {
      const int j = t + c.lane;
      if (j < n) row_activity_lane(P, S, full ? __ldg(ids + j) : ids[j]);
    }
  }
}

// ------------------------------------------------------------------ tightening

__device__ int tighten_lane(const DevProblem& P, const DevState& S, int i, const Limits& lim)
{
  const double2 b    = S.bounds[i];
  const bool integer = __ldg(P.is_int + i) != 0;
  Fold f{b.x, -1, b.y, -1};
  const int cs = __ldg(P.col_start + i), ce = __ldg(P.col_start + i + 1);
#pragma unroll 2
  for (int e = cs; e < ce; ++e) {
    const int k    = __ldg(P.col_row + e);
    const double a = __ldg(P.col_val + e);
    const RowRec r = ld_rec(S.rec + k);
    fold_entry(f, b.x, b.y, integer, a, r, S.aux, k, e);
  }
  return finish_var(S.bounds + i, b.x, b.y, f.lo, f.up, integer, lim);
}

__device__ int tighten_warp(Ctx& c, int i)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const double2 b     = S.bounds[i];
  const bool integer  = __ldg(P.is_int + i) != 0;
  Fold f{b.x, -1, b.y, -1};
  const int cs = __ldg(P.col_start + i), ce = __ldg(P.col_start + i + 1);
  for (int e = cs + c.lane; e < ce; e += 32) {
    const int k    = __ldg(P.col_row + e);
    const double a = __ldg(P.col_val + e);
    const RowRec r = ld_rec(S.rec + k);
    fold_entry(f, b.x, b.y, integer, a, r, S.aux, k, e);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double olo = __shfl_xor_sync(FULL, f.lo, o);
    const int olp    = __shfl_xor_sync(FULL, f.lo_pos, o);
    const double oup = __shfl_xor_sync(FULL, f.up, o);
    const int oupp   = __shfl_xor_sync(FULL, f.up_pos, o);
    fold_combine(f, olo, olp, oup, oupp);
  }
  int res = 0;
  if (c.lane == 0) res = finish_var(S.bounds + i, b.x, b.y, f.lo, f.up, integer, c.lim);
  return __shfl_sync(FULL, res, 0);
}

struct Tally {
  int crossed;
  int any_rows;
  unsigned long long colnnz;
  int nbuf;  // warp-uniform count of staged changed vars
};

__device__ __forceinline__ void flush_changed(Ctx& c, ParCtl* pc, Tally& t)
{
  if (t.nbuf == 0) return;
  int base = 0;
  if (c.lane == 0) base = atomicAdd(&pc->n_changed, t.nbuf);
  base = __shfl_sync(FULL, base, 0);
  __syncwarp();
  for (int j = c.lane; j < t.nbuf; j += 32) c.S.changed[base + j] = c.sm.chg[c.warp][j];
  __syncwarp();
  t.nbuf = 0;
}

// Records the per-var outcomes of one warp step (each lane: var i or -1, result r).
__device__ __forceinline__ void tally(Ctx& c, ParCtl* pc, Tally& t, int i, int r)
{
  const unsigned ch = __ballot_sync(FULL, r > 0);
  if (r < 0) t.crossed++;
  if (r > 0) {
    const int nnz = __ldg(c.P.col_start + i + 1) - __ldg(c.P.col_start + i);
    t.colnnz += (unsigned long long)nnz;
    if (nnz > 0) t.any_rows = 1;
  }
  if (ch) {
    if (t.nbuf + __popc(ch) > 64) flush_changed(c, pc, t);
    if (r > 0) c.sm.chg[c.warp][t.nbuf + __popc(ch & lanemask_lt())] = i;
    t.nbuf += __popc(ch);
    __syncwarp();
  }
}

__device__ void phase_tighten(Ctx& c, ParCtl* pc, bool full)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int par       = (&c.S.ctl->par[1] == pc) ? 1 : 0;
  Tally t{0, 0, 0ull, 0};
  {
    const int n    = full ? P.n_mcol : ld_volatile(&pc->n_dvar_m);
    const int* ids = full ? P.mcol : S.dvar_m[par];
    for (int q = warp_fetch(c, &pc->cur_vm, 1); q < n; q = warp_fetch(c, &pc->cur_vm, 1)) {
      const int i = full ? __ldg(ids + q) : ids[q];
      const int r = tighten_warp(c, i);
      // lane 0 stands for the var; other lanes report nothing
      tally(c, pc, t, c.lane == 0 ? i : -1, c.lane == 0 ? r : 0);
    }
  }
  {
    const int n    = full ? P.n_scol : ld_volatile(&pc->n_dvar_s);
    const int* ids = full ? P.scol : S.dvar_s[par];
    for (int q = warp_fetch(c, &pc->cur_vs, 32); q < n; q = warp_fetch(c, &pc->cur_vs, 32)) {
      const int j = q + c.lane;
      int i = -1, r = 0;
      if (j < n) {
        i = full ? __ldg(ids + j) : ids[j];
        r = tighten_lane(P, S, i, c.lim);
      }
      tally(c, pc, t, i, r);
    }
  }
  flush_changed(c, pc, t);
  // block reduction of the tallies, one global atomic each
  int cr = warp_sum(t.crossed);
  int ar = __any_sync(FULL, t.any_rows);
  unsigned long long cn = t.colnnz;
#pragma unroll
  for (int o = 16; o; o >>= 1) cn += __shfl_xor_sync(FULL, cn, o);
  if (c.lane == 0) {
    if (cr) atomicAdd(&c.sm.blk_crossed, cr);
    if (ar) atomicOr(&c.sm.blk_any_rows, 1);
    if (cn) atomicAdd(&c.sm.blk_colnnz, cn);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (c.sm.blk_crossed) atomicAdd(&pc->n_crossed, c.sm.blk_crossed);
    if (c.sm.blk_any_rows) atomicOr(&pc->any_rows, 1);
    if (c.sm.blk_colnnz) atomicAdd(&pc->colnnz, c.sm.blk_colnnz);
    c.sm.blk_crossed  = 0;
    c.sm.blk_any_rows = 0;
    c.sm.blk_colnnz   = 0;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ frontier

__device__ __forceinline__ int warp_append(int* counter, bool pred, unsigned lt)
{
  const unsigned b = __ballot_sync(FULL, pred);
  if (!b) return -1;
  const int leader = __ffs(b) - 1;
  int base         = 0;
  if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(counter, __popc(b));
  base = __shfl_sync(FULL, base, leader);
  return pred ? base + __popc(b & lt) : -1;
}

// Phase C: rows(changed) → dirty rows of the next round, classified + var-expansion tasks.
__device__ void phase_expand_rows(Ctx& c, ParCtl* pc, ParCtl* qc, int qpar, unsigned stamp)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int nch       = ld_volatile(&pc->n_changed);
  const unsigned lt   = lanemask_lt();
  unsigned long long roww = 0;
  for (int t = warp_fetch(c, &pc->cur_x1, 32); t < nch; t = warp_fetch(c, &pc->cur_x1, 32)) {
    const int cnt = min(32, nch - t);
    for (int q = 0; q < cnt; ++q) {
      const int i  = S.changed[t + q];
      const int cs = __ldg(P.col_start + i), ce = __ldg(P.col_start + i + 1);
      for (int base = cs; base < ce; base += 32) {
        const int e   = base + c.lane;
        const bool ok = e < ce;
        const int k   = ok ? __ldg(P.col_row + e) : 0;
        const bool nw = ok && atomicExch(S.row_stamp + k, stamp) != stamp;
        if (!__ballot_sync(FULL, nw)) continue;
        const int L = nw ? __ldg(P.row_start + k + 1) - __ldg(P.row_start + k) : 0;
        if (nw) roww += (unsigned long long)L;
        int pos = warp_append(&qc->n_drow_all, nw, lt);
        if (nw) S.drow_all[qpar][pos] = k;
        const bool is_s = nw && L <= kShortNnz;
        const bool is_m = nw && L > kShortNnz && L <= kSegNnz;
        const bool is_g = nw && L > kSegNnz;
        pos = warp_append(&qc->n_drow_s, is_s, lt);
        if (is_s) S.drow_s[qpar][pos] = k;
        pos = warp_append(&qc->n_drow_m, is_m, lt);
        if (is_m) S.drow_m[qpar][pos] = k;
        if (is_g) {
          const int ns = (L + kSumSegment - 1) / kSumSegment;
          const int b0 = atomicAdd(&qc->n_dseg, ns);
          for (int s = 0; s < ns; ++s) S.dseg[qpar][b0 + s] = make_int2(k, s);
        }
        if (nw && L > 0) {
          const int nx = (L + kXChunk - 1) / kXChunk;
          const int b0 = atomicAdd(&qc->n_xtask, nx);
          for (int s = 0; s < nx; ++s) S.xtask[qpar][b0 + s] = make_int2(k, s);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) roww += __shfl_xor_sync(FULL, roww, o);
  if (c.lane == 0 && roww) atomicAdd(&qc->roww, roww);
}

// Phase D: dirty rows → dirty vars of the next round (classified by column length).
__device__ void phase_expand_vars(Ctx& c, ParCtl* pc, ParCtl* qc, int qpar, unsigned stamp)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int ntask     = ld_volatile(&qc->n_xtask);
  const unsigned lt   = lanemask_lt();
  unsigned long long colw = 0;
  for (int t = warp_fetch(c, &pc->cur_x2, 1); t < ntask; t = warp_fetch(c, &pc->cur_x2, 1)) {
    const int2 tk = S.xtask[qpar][t];
    const int rs  = __ldg(P.row_start + tk.x), re = __ldg(P.row_start + tk.x + 1);
    const int e0  = rs + tk.y * kXChunk, e1 = min(re, e0 + kXChunk);
    bool nw[kXChunk / 32];
    int vj[kXChunk / 32];
#pragma unroll
    for (int h = 0; h < kXChunk / 32; ++h) {
      const int e = e0 + h * 32 + c.lane;
      vj[h]       = e < e1 ? __ldg(P.row_col + e) : -1;
      nw[h]       = vj[h] >= 0 && atomicExch(S.var_stamp + vj[h], stamp) != stamp;
    }
#pragma unroll
    for (int h = 0; h < kXChunk / 32; ++h) {
      if (!__ballot_sync(FULL, nw[h])) continue;
      const int L     = nw[h] ? __ldg(P.col_start + vj[h] + 1) - __ldg(P.col_start + vj[h]) : 0;
      const bool is_s = nw[h] && L <= kShortNnz;
      const bool is_m = nw[h] && L > kShortNnz;
      colw += (unsigned long long)L;
      int pos         = warp_append(&qc->n_dvar_s, is_s, lt);
      if (is_s) S.dvar_s[qpar][pos] = vj[h];
      pos = warp_append(&qc->n_dvar_m, is_m, lt);
      if (is_m) S.dvar_m[qpar][pos] = vj[h];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) colw += __shfl_xor_sync(FULL, colw, o);
  if (c.lane == 0 && colw) atomicAdd(&qc->colw, colw);
}

__device__ void zero_par(ParCtl* q)
{
  int* w = reinterpret_cast<int*>(q);
  for (int j = 0; j < (int)(sizeof(ParCtl) / sizeof(int)); ++j) w[j] = 0;
}

__global__ void __launch_bounds__(kThreads, 2)
    k_engine(DevProblem P, DevState S, Limits lim, int mode, int full_first, unsigned stamp_base,
             unsigned long long dense_thr, long long* stats)
{
  __shared__ Smem sm;
  cg::grid_group grid = cg::this_grid();
  if (threadIdx.x == 0) {
    sm.blk_crossed  = 0;
    sm.blk_any_rows = 0;
    sm.blk_colnnz   = 0;
  }
  __syncthreads();
  Ctx c{P, S, lim, sm, (int)(threadIdx.x & 31), (int)(threadIdx.x >> 5),
        (int)((blockIdx.x * kThreads + threadIdx.x) >> 5), (int)(gridDim.x * kWarps)};

  if (mode == MODE_ACTIVITY) {
    phase_activity(c, &S.ctl->par[1], full_first != 0);
    return;
  }
  if (mode == MODE_TIGHTEN) {
    phase_tighten(c, &S.ctl->par[1], full_first != 0);
    return;
  }

  const unsigned long long t0 = globaltimer();
  const bool timed            = isfinite(lim.time_limit);
  bool full                   = true;  // round 1 is always a full sweep (propagation.hpp:442)
  bool any_change             = false;
  int status = BP_STATUS_UNSET, crossed_out = 0;
  int rounds = 0;
  while (rounds < lim.max_rounds) {
    ++rounds;
    const int ppar = rounds & 1, qpar = ppar ^ 1;
    ParCtl* pc     = &S.ctl->par[ppar];
    ParCtl* qc     = &S.ctl->par[qpar];
    phase_activity(c, pc, full || !lim.incremental);
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      zero_par(qc);
      if (timed && (double)(globaltimer() - t0) * 1e-9 >= lim.time_limit) pc->stop = 1;
    }
    phase_tighten(c, pc, full || !lim.incremental);
    grid.sync();
    const int cr = ld_volatile(&pc->n_crossed);
    const int nc = ld_volatile(&pc->n_changed);
    if (stats && blockIdx.x == 0 && threadIdx.x == 0) {
      const bool fr = full || !lim.incremental;
      long long* st = stats + (long long)(rounds - 1) * kStatCols;
      st[0] = fr ? 1 : 0;
      st[1] = fr ? P.m : ld_volatile(&pc->n_drow_all);
      st[2] = fr ? P.nnz : (long long)ld_volatile(&pc->roww);
      st[3] = fr ? P.n : ld_volatile(&pc->n_dvar_s) + ld_volatile(&pc->n_dvar_m);
      st[4] = fr ? P.nnz : (long long)ld_volatile(&pc->colw);
      st[5] = nc;
    }
    if (cr > 0) {
      status      = BP_STATUS_INFEASIBLE;
      crossed_out = cr;
      break;
    }
    if (nc == 0) break;
    any_change = true;
    if (!ld_volatile(&pc->any_rows)) break;          // dirty_rows.empty() (propagation.hpp:481)
    if (rounds >= lim.max_rounds) break;
    if (ld_volatile(&pc->stop)) break;             // time limit (propagation.hpp:439)
    if (!lim.incremental || ld_volatile(&pc->colnnz) > dense_thr) {
      full = true;
      continue;
    }
    const unsigned stamp = stamp_base + (unsigned)rounds;
    phase_expand_rows(c, pc, qc, qpar, stamp);
    grid.sync();
    if (ld_volatile(&qc->roww) > dense_thr) {
      full = true;
      continue;
    }
    phase_expand_vars(c, pc, qc, qpar, stamp);
    grid.sync();
    full = false;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (status == BP_STATUS_UNSET) status = any_change ? BP_STATUS_TIGHTENED : BP_STATUS_UNCHANGED;
    S.ctl->status     = status;
    S.ctl->rounds     = rounds;
    S.ctl->crossed    = crossed_out;
    S.ctl->any_change = any_change ? 1 : 0;
  }
}

}  // namespace

// ------------------------------------------------------------------ host side

DevProblem Problem::dev() const
{
  DevProblem d;
  d.n         = n;
  d.m         = m;
  d.nnz       = nnz;
  d.row_start = row_start.p;
  d.row_col   = row_col.p;
  d.row_val   = row_val.p;
  d.col_start = col_start.p;
  d.col_row   = col_row.p;
  d.col_val   = col_val.p;
  d.cons      = cons.p;
  d.is_int    = is_int.p;
  d.n_srow    = n_srow;
  d.srow      = srow.p;
  d.n_mrow    = n_mrow;
  d.mrow      = mrow.p;
  d.n_seg     = n_seg;
  d.seg_task  = seg_task.p;
  d.seg_base  = seg_base.p;
  d.n_scol    = n_scol;
  d.scol      = scol.p;
  d.n_mcol    = n_mcol;
  d.mcol      = mcol.p;
  return d;
}

void problem_build(Problem& P, int n, int m, const int* row_start, const int* row_col,
                   const double* row_val, const int* col_start_in, const int* col_row_in,
                   const double* col_val_in, const double* var_lower, const double* var_upper,
                   const uint8_t* is_integer, const double* cons_lower, const double* cons_upper)
{
  BP_CUDA(cudaSetDevice(P.device));
  P.n   = n;
  P.m   = m;
  P.nnz = row_start[m];
  const long long N = P.nnz;
  P.h_row_start.assign(row_start, row_start + m + 1);
  // CSC: caller-provided or the stable transpose of problem.hpp:211-225.
  std::vector<int> cst, crw;
  std::vector<double> cvl;
  if (col_start_in) {
    P.h_col_start.assign(col_start_in, col_start_in + n + 1);
  } else {
    cst.assign(n + 1, 0);
    for (long long e = 0; e < N; ++e) cst[row_col[e] + 1]++;
    for (int i = 0; i < n; ++i) cst[i + 1] += cst[i];
    crw.resize(N);
    cvl.resize(N);
    std::vector<int> cur(cst.begin(), cst.end() - 1);
    for (int k = 0; k < m; ++k)
      for (int e = row_start[k]; e < row_start[k + 1]; ++e) {
        const int d = cur[row_col[e]]++;
        crw[d]      = k;
        cvl[d]      = row_val[e];
      }
    P.h_col_start = cst;
    col_row_in    = crw.data();
    col_val_in    = cvl.data();
  }
  P.row_start.upload(row_start, m + 1);
  P.row_col.upload(row_col, N);
  P.row_val.upload(row_val, N);
  P.col_start.upload(P.h_col_start.data(), n + 1);
  P.col_row.upload(col_row_in, N);
  P.col_val.upload(col_val_in, N);
  std::vector<double2> cons(m);
  for (int k = 0; k < m; ++k) cons[k] = make_double2(cons_lower[k], cons_upper[k]);
  P.cons.upload(cons);
  P.is_int.upload(is_integer, n);

  // Partition tables.
  std::vector<int> srow, mrow, scol, mcol, seg_base(m, -1);
  std::vector<std::pair<int, int>> seg_rows;
  for (int k = 0; k < m; ++k) {
    const int L = row_start[k + 1] - row_start[k];
    if (L <= kShortNnz) srow.push_back(k);
    else if (L <= kSegNnz) mrow.push_back(k);
    else seg_rows.push_back({L, k});
  }
  std::stable_sort(mrow.begin(), mrow.end(), [&](int a, int b) {
    return row_start[a + 1] - row_start[a] > row_start[b + 1] - row_start[b];
  });
  std::stable_sort(seg_rows.begin(), seg_rows.end(),
                   [](auto& a, auto& b) { return a.first > b.first; });
  std::vector<int2> seg_task;
  int slot = 0;
  // segment-major order: the first segment of every long row first, so all long rows start early
  int max_seg = 0;
  for (auto& [L, k] : seg_rows) {
    seg_base[k] = slot;
    const int ns = (L + kSumSegment - 1) / kSumSegment;
    slot += ns;
    max_seg = std::max(max_seg, ns);
  }
  for (int s = 0; s < max_seg; ++s)
    for (auto& [L, k] : seg_rows)
      if (s * kSumSegment < L) seg_task.push_back(make_int2(k, s));
  for (int i = 0; i < n; ++i) {
    const int L = P.h_col_start[i + 1] - P.h_col_start[i];
    if (L <= kShortNnz) scol.push_back(i);
    else mcol.push_back(i);
  }
  std::stable_sort(mcol.begin(), mcol.end(), [&](int a, int b) {
    return P.h_col_start[a + 1] - P.h_col_start[a] > P.h_col_start[b + 1] - P.h_col_start[b];
  });
  P.n_srow = (int)srow.size();
  P.n_mrow = (int)mrow.size();
  P.n_seg  = (int)seg_task.size();
  P.n_scol = (int)scol.size();
  P.n_mcol = (int)mcol.size();
  P.srow.upload(srow);
  P.mrow.upload(mrow);
  P.scol.upload(scol);
  P.mcol.upload(mcol);
  P.seg_task.upload(seg_task);
  P.seg_base.upload(seg_base);
  P.h_seg_base = seg_base;

  // Workspace.
  P.bounds.alloc(std::max(n, 1));
  P.rec.alloc(std::max(m, 1));
  P.aux.alloc(std::max(m, 1));
  P.seg_part.alloc(std::max(slot, 1));
  P.seg_done.alloc(std::max(m, 1));
  BP_CUDA(cudaMemset(P.seg_done.p, 0, sizeof(int) * std::max(m, 1)));
  P.row_stamp.alloc(std::max(m, 1));
  P.var_stamp.alloc(std::max(n, 1));
  BP_CUDA(cudaMemset(P.row_stamp.p, 0, sizeof(unsigned) * std::max(m, 1)));
  BP_CUDA(cudaMemset(P.var_stamp.p, 0, sizeof(unsigned) * std::max(n, 1)));
  const size_t mm = (size_t)std::max(m, 1), nn = (size_t)std::max(n, 1);
  // int lists per parity: drow_all, drow_s, drow_m (m each), dvar_s, dvar_m (n each); changed (n)
  P.lists_i.alloc(2 * (3 * mm + 2 * nn) + nn);
  // int2 lists per parity: dseg (slot), xtask (N/256 + m)
  const size_t nseg_cap = (size_t)std::max(slot, 1);
  const size_t nx_cap   = (size_t)(N / kXChunk) + mm + 1;
  P.lists_i2.alloc(2 * (nseg_cap + nx_cap));
  P.ctl.alloc(1);
  DevState& S = P.st;
  S.bounds    = P.bounds.p;
  S.rec       = P.rec.p;
  S.aux       = P.aux.p;
  S.seg_part  = P.seg_part.p;
  S.seg_done  = P.seg_done.p;
  S.row_stamp = P.row_stamp.p;
  S.var_stamp = P.var_stamp.p;
  int* pi     = P.lists_i.p;
  int2* pi2   = P.lists_i2.p;
  for (int q = 0; q < 2; ++q) {
    S.drow_all[q] = pi; pi += mm;
    S.drow_s[q]   = pi; pi += mm;
    S.drow_m[q]   = pi; pi += mm;
    S.dvar_s[q]   = pi; pi += nn;
    S.dvar_m[q]   = pi; pi += nn;
    S.dseg[q]     = pi2; pi2 += nseg_cap;
    S.xtask[q]    = pi2; pi2 += nx_cap;
  }
  S.changed = pi;
  S.ctl     = P.ctl.p;

  int dev_sms = 0, per_sm = 0;
  BP_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, P.device));
  BP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_engine, kThreads, 0));
  if (per_sm < 1) throw cuda_error("engine kernel cannot be resident (occupancy 0)");
  P.grid_blocks = dev_sms * std::min(per_sm, 2);
  BP_CUDA(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
  BP_CUDA(cudaEventCreate(&P.ev0));
  BP_CUDA(cudaEventCreate(&P.ev1));
}

RunResult run_engine(Problem& P, Mode mode, bool full, const Limits& lim, cudaStream_t s, int flags,
                     long long* d_stats)
{
  DevProblem d                 = P.dev();
  DevState st                  = P.st;
  Limits l                     = lim;
  int md                       = (int)mode;
  int ff                       = full ? 1 : 0;
  // stamps: one value per round, never reused until wrap-around (then the stamp arrays reset)
  if (P.stamp_base > 0xF0000000u - (unsigned)lim.max_rounds - 2) {
    BP_CUDA(cudaMemsetAsync(P.row_stamp.p, 0, sizeof(unsigned) * P.row_stamp.n, s));
    BP_CUDA(cudaMemsetAsync(P.var_stamp.p, 0, sizeof(unsigned) * P.var_stamp.n, s));
    P.stamp_base = 1;
  }
  unsigned sb                  = P.stamp_base;
  P.stamp_base += (unsigned)std::max(lim.max_rounds, 1) + 1;
  unsigned long long dense_thr = (flags & ENGINE_FORCE_FRONTIER) ? ~0ull
                                                                 : (unsigned long long)(P.nnz / 4);
  long long* stp = d_stats;
  void* args[] = {&d, &st, &l, &md, &ff, &sb, &dense_thr, &stp};
  BP_CUDA(cudaEventRecord(P.ev0, s));
  BP_CUDA(cudaLaunchCooperativeKernel((void*)k_engine, P.grid_blocks, kThreads, args, 0, s));
  BP_CUDA(cudaEventRecord(P.ev1, s));
  ++g_kernel_launches;
  RunResult r{0, 0, 0};
  if (mode == MODE_PROPAGATE) {
    int h[4];
    BP_CUDA(cudaMemcpyAsync(h, &P.st.ctl->status, sizeof(h), cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaStreamSynchronize(s));
    r.status  = h[0];
    r.rounds  = h[1];
    r.crossed = h[2];
  } else {
    BP_CUDA(cudaStreamSynchronize(s));
  }
  float ms = 0.f;
  BP_CUDA(cudaEventElapsedTime(&ms, P.ev0, P.ev1));
  P.last_kernel_ms = ms;
  P.total_kernel_ms += ms;
  P.n_launch++;
  return r;
}

void stage_rows(Problem& P, const int* rows, int nrows, cudaStream_t s)
{
  std::vector<int> all, sr, mr;
  std::vector<int2> sg;
  for (int j = 0; j < nrows; ++j) {
    const int k = rows[j];
    const int L = P.h_row_start[k + 1] - P.h_row_start[k];
    all.push_back(k);
    if (L <= kShortNnz) sr.push_back(k);
    else if (L <= kSegNnz) mr.push_back(k);
    else
      for (int q = 0; q * kSumSegment < L; ++q) sg.push_back(make_int2(k, q));
  }
  DevState& S = P.st;
  auto up = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) BP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  };
  up(S.drow_all[1], all.data(), all.size() * 4);
  up(S.drow_s[1], sr.data(), sr.size() * 4);
  up(S.drow_m[1], mr.data(), mr.size() * 4);
  up(S.dseg[1], sg.data(), sg.size() * 8);
  int cnt[4] = {(int)all.size(), (int)sr.size(), (int)mr.size(), (int)sg.size()};
  up(&S.ctl->par[1].n_drow_all, cnt, sizeof(cnt));
}

void stage_vars(Problem& P, const int* vars, int nvars, cudaStream_t s)
{
  std::vector<int> sv, mv;
  for (int j = 0; j < nvars; ++j) {
    const int i = vars[j];
    const int L = P.h_col_start[i + 1] - P.h_col_start[i];
    (L <= kShortNnz ? sv : mv).push_back(i);
  }
  DevState& S = P.st;
  if (!sv.empty())
    BP_CUDA(cudaMemcpyAsync(S.dvar_s[1], sv.data(), sv.size() * 4, cudaMemcpyHostToDevice, s));
  if (!mv.empty())
    BP_CUDA(cudaMemcpyAsync(S.dvar_m[1], mv.data(), mv.size() * 4, cudaMemcpyHostToDevice, s));
  int cnt[2] = {(int)sv.size(), (int)mv.size()};
  BP_CUDA(cudaMemcpyAsync(&S.ctl->par[1].n_dvar_s, cnt, sizeof(cnt), cudaMemcpyHostToDevice, s));
}

}  // namespace bp
