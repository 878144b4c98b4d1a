// Persistent, device-resident bound propagation for sm_100a.
//
// One cooperative kernel runs the whole `propagate` loop of the reference
// (propagation.hpp:418-486) with no host round trip per round:
//
//   round r:  Phase A  row activities      (propagation.hpp:226-251)   ─ grid.sync
//             Phase B  bound tightening    (propagation.hpp:378-412)   ─ grid.sync
//             decision: infeasible / fixpoint / round cap / empty frontier (uniform on every block)
//             Phase C  frontier: changed vars → dirty rows (+ segment / expansion tasks) ─ grid.sync
//             Phase D  dirty rows → dirty vars                                           ─ grid.sync
//
// The path is a sparse gather: its cost is memory-level parallelism, not arithmetic. Work is
// therefore organised so every warp keeps 4 independent gathers per lane in flight:
//   rows  nnz <= 32   packed tiles (<= 32 rows, <= 128 entries): the warp loads a tile coalesced,
//                     gathers all bounds at once, and each lane folds one row in reference order
//                     from shared memory (exact: same sequential sum).
//         nnz > 32    one warp per 16384-entry segment (the reference's fixed summation tree,
//                     problem.hpp:274), software-pipelined in 128-entry chunks (loads two chunks
//                     ahead, gathers one chunk ahead of the fold); zero contributions are
//                     compacted away (exact: the running sum starts at +0.0 and is never -0.0);
//                     lanes 0/1 fold the min/max chains. Multi-segment rows are summed by the
//                     last segment to finish, in segment order (heavy_row_activity, :197-218).
//   vars  nnz <= 32   packed tiles; lanes gather row records (one LDG.256 each) and compute
//                     per-entry candidates; each lane folds one variable in CSC order.
//         nnz > 32    one warp per variable; the std::min/max fold is reduced as a lexicographic
//                     (value, CSC position) min/max, which reproduces "first operand wins on
//                     ties" (sign of tied zeros) exactly.
// Frontier rounds (propagation.hpp:456-479) touch only dirty rows / dirty vars; when the frontier
// would cost about as much as the whole matrix the engine runs a full round instead — evaluating a
// superset of the dirty sets yields bit-identical results (SURVEY §8a A12 lemma).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "bp_engine.cuh"

namespace cg = cooperative_groups;

namespace bp {

long long g_kernel_launches = 0;

namespace {

constexpr int kThreads  = 256;
constexpr int kWarps    = kThreads / 32;
constexpr unsigned FULL = 0xffffffffu;
constexpr int kXChunk   = 256;  // entries per var-expansion task
constexpr int kEPL      = kTile / 32;

__device__ __forceinline__ unsigned lanemask_lt()
{
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int warp_sum(int v)
{
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ int warp_incl_scan(int v, int lane)
{
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer()
{
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ldv(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ unsigned long long ldv(const unsigned long long* p)
{
  return *(const volatile unsigned long long*)p;
}

struct WarpSmem {
  double b0[kTile];          // min contributions / lower-bound candidates
  double b1[kTile];          // max contributions / upper-bound candidates
  unsigned char fl[kTile];   // infinite-contributor flags (bit 0 min, bit 1 max)
  int off[32];               // list tiles: exclusive entry offsets of the 32 items
  int st[32];                //             their first entry
  double2 vb[32];            // tighten tiles: the 32 variables' bounds
  unsigned char vint[32];    //                and integrality
  int chg[64];               // changed-var staging before a global append
};

struct Smem {
  WarpSmem w[kWarps];
  int blk_crossed;
  int blk_any_rows;
  unsigned long long blk_colnnz;
};

struct Ctx {
  const DevProblem& P;
  const DevState& S;
  const Limits& lim;
  Smem& sm;
  WarpSmem& w;
  int lane, warp;
};

// Allocates `cnt` slots per lane in a global list with one atomic per warp; returns this lane's
// first slot.
__device__ __forceinline__ int warp_alloc(int* counter, int cnt, int lane)
{
  const int incl  = warp_incl_scan(cnt, lane);
  const int total = __shfl_sync(FULL, incl, 31);
  int base        = 0;
  if (total) {
    if (lane == 31) base = atomicAdd(counter, total);
    base = __shfl_sync(FULL, base, 31);
  }
  return base + incl - cnt;
}

// Largest o with off[o] <= f (off non-decreasing, off[0] = 0): the list item owning entry f.
__device__ __forceinline__ int owner_of(const int* off, int f)
{
  int o = 0;
#pragma unroll
  for (int step = 16; step; step >>= 1)
    if (off[o + step] <= f) o += step;
  return o;
}

__device__ __forceinline__ int warp_fetch(Ctx& c, int* cursor, int step)
{
  int t = 0;
  if (c.lane == 0) t = atomicAdd(cursor, step);
  return __shfl_sync(FULL, t, 0);
}

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

// One 16384-entry segment of a long row, streamed by one warp.
__device__ void row_stream(Ctx& c, int k, int seg)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int lane      = c.lane;
  const int rs = __ldg(P.row_start + k), L = __ldg(P.row_start + k + 1) - rs;
  const int e0 = rs + seg * kSumSegment, e1 = rs + min(L, (seg + 1) * kSumSegment);
  const int nch = (e1 - e0 + kTile - 1) / kTile;
  int ca[kEPL], cb[kEPL];
  double va[kEPL], vb[kEPL];
  double2 bd[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    const int e = e0 + h * 32 + lane;
    ca[h]       = e < e1 ? __ldg(P.row_col + e) : -1;
    va[h]       = e < e1 ? __ldg(P.row_val + e) : 0.0;
  }
#pragma unroll
  for (int h = 0; h < kEPL; ++h) bd[h] = ca[h] >= 0 ? S.bounds[ca[h]] : make_double2(0.0, 0.0);
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    const int e = e0 + kTile + h * 32 + lane;
    cb[h]       = e < e1 ? __ldg(P.row_col + e) : -1;
    vb[h]       = e < e1 ? __ldg(P.row_val + e) : 0.0;
  }
  double acc = 0.0;
  int imn = 0, imx = 0;
  const unsigned lt = lanemask_lt();
  for (int s = 0; s < nch; ++s) {
    double cm[kEPL], cx[kEPL];
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      cm[h] = 0.0;
      cx[h] = 0.0;
      if (ca[h] >= 0) {
        int i1, i2;
        contrib(va[h], bd[h].x, bd[h].y, cm[h], cx[h], i1, i2);
        imn += i1;
        imx += i2;
      }
    }
    // gather chunk s+1 (its columns arrived one iteration ago), load chunk s+2
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      bd[h] = cb[h] >= 0 ? S.bounds[cb[h]] : make_double2(0.0, 0.0);
      ca[h] = cb[h];
      va[h] = vb[h];
    }
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const int e = e0 + (s + 2) * kTile + h * 32 + lane;
      cb[h]       = e < e1 ? __ldg(P.row_col + e) : -1;
      vb[h]       = e < e1 ? __ldg(P.row_val + e) : 0.0;
    }
    // order-preserving compaction of the non-zero contributions of each chain
    int pm = 0, px = 0;
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const unsigned m = __ballot_sync(FULL, cm[h] != 0.0);
      const unsigned x = __ballot_sync(FULL, cx[h] != 0.0);
      if (cm[h] != 0.0) c.w.b0[pm + __popc(m & lt)] = cm[h];
      if (cx[h] != 0.0) c.w.b1[px + __popc(x & lt)] = cx[h];
      pm += __popc(m);
      px += __popc(x);
    }
    __syncwarp();
    if (lane < 2) {
      const int cnt     = lane ? px : pm;
      const double* src = lane ? c.w.b1 : c.w.b0;
#pragma unroll 4
      for (int j = 0; j < cnt; ++j) acc = __dadd_rn(acc, src[j]);
    }
    __syncwarp();
  }
  imn              = warp_sum(imn);
  imx              = warp_sum(imx);
  const double smx = __shfl_sync(FULL, acc, 1);
  if (lane == 0) {
    const int nseg = (L + kSumSegment - 1) / kSumSegment;
    if (nseg == 1) {
      write_rec(P, S, k, acc, smx, imn, imx);  // 0.0 + part == part (part is never -0.0)
    } else {
      const int base = __ldg(P.seg_base + k);
      SegPart sp;
      sp.min  = acc;
      sp.max  = smx;
      sp.nmin = imn;
      sp.nmax = imx;
      sp.pad0 = sp.pad1 = 0;
      S.seg_part[base + seg] = sp;
      __threadfence();
      const int done = atomicAdd(&S.seg_done[k], 1);
      if (done == nseg - 1) {
        __threadfence();
        double tmn = 0.0, tmx = 0.0;
        int cmn = 0, cmx = 0;
        for (int q = 0; q < nseg; ++q) {  // row_activity's segment fold (propagation.hpp:182-188)
          const SegPart* p = S.seg_part + base + q;
          tmn = __dadd_rn(tmn, __ldcg(&p->min));
          tmx = __dadd_rn(tmx, __ldcg(&p->max));
          cmn += __ldcg(&p->nmin);
          cmx += __ldcg(&p->nmax);
        }
        write_rec(P, S, k, tmn, tmx, cmn, cmx);
        S.seg_done[k] = 0;
      }
    }
  }
}

// Contributions of up to 128 gathered entries into shared memory (slot h*32+lane).
__device__ __forceinline__ void stage_contribs(Ctx& c, const int* col, const double* a)
{
  double2 bd[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) bd[h] = col[h] >= 0 ? c.S.bounds[col[h]] : make_double2(0.0, 0.0);
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    double cm = 0.0, cx = 0.0;
    int i1 = 0, i2 = 0;
    if (col[h] >= 0) contrib(a[h], bd[h].x, bd[h].y, cm, cx, i1, i2);
    c.w.b0[h * 32 + c.lane] = cm;
    c.w.b1[h * 32 + c.lane] = cx;
    c.w.fl[h * 32 + c.lane] = (unsigned char)(i1 | (i2 << 1));
  }
}

// A packed tile of short rows (full rounds).
__device__ void act_tile_packed(Ctx& c, int t)
{
  const DevProblem& P = c.P;
  const int r0 = __ldg(P.sr_tile + t), r1 = __ldg(P.sr_tile + t + 1);
  const int p0 = __ldg(P.sr_ptr + r0), p1 = __ldg(P.sr_ptr + r1);
  int col[kEPL];
  double a[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    const int f = p0 + h * 32 + c.lane;
    col[h]      = f < p1 ? __ldg(P.sr_col + f) : -1;
    a[h]        = f < p1 ? __ldg(P.sr_val + f) : 0.0;
  }
  stage_contribs(c, col, a);
  __syncwarp();
  if (c.lane < r1 - r0) {
    const int r  = r0 + c.lane;
    const int q0 = __ldg(P.sr_ptr + r) - p0, q1 = __ldg(P.sr_ptr + r + 1) - p0;
    double smn = 0.0, smx = 0.0;
    int imn = 0, imx = 0;
    for (int q = q0; q < q1; ++q) {
      smn = __dadd_rn(smn, c.w.b0[q]);
      smx = __dadd_rn(smx, c.w.b1[q]);
      imn += c.w.fl[q] & 1;
      imx += c.w.fl[q] >> 1;
    }
    write_rec(P, c.S, __ldg(P.srow + r), smn, smx, imn, imx);
  }
  __syncwarp();
}

// Up to 32 listed items (rows or columns) as one flattened entry stream: returns this lane's
// item range [excl, excl + L) and the stream length; fills w.off / w.st.
__device__ __forceinline__ int list_tile_setup(Ctx& c, int first, int len, int& excl)
{
  const int incl = warp_incl_scan(len, c.lane);
  excl           = incl - len;
  c.w.off[c.lane] = excl;
  c.w.st[c.lane]  = first;
  __syncwarp();
  return __shfl_sync(FULL, incl, 31);
}

// Listed short rows (frontier rounds): flattened 128-entry windows, each lane folds its row.
__device__ void act_list_tile(Ctx& c, const int* ids, int base, int n)
{
  const DevProblem& P = c.P;
  const int j = base + c.lane;
  const int k = j < n ? ids[j] : -1;
  int rs = 0, L = 0;
  if (k >= 0) {
    rs = __ldg(P.row_start + k);
    L  = __ldg(P.row_start + k + 1) - rs;
  }
  int excl;
  const int T = list_tile_setup(c, rs, L, excl);
  double smn = 0.0, smx = 0.0;
  int imn = 0, imx = 0;
  for (int w0 = 0; w0 < T; w0 += kTile) {
    int col[kEPL];
    double a[kEPL];
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const int f = w0 + h * 32 + c.lane;
      col[h]      = -1;
      a[h]        = 0.0;
      if (f < T) {
        const int o = owner_of(c.w.off, f);
        const int e = c.w.st[o] + (f - c.w.off[o]);
        col[h]      = __ldg(P.row_col + e);
        a[h]        = __ldg(P.row_val + e);
      }
    }
    stage_contribs(c, col, a);
    __syncwarp();
    if (k >= 0) {
      const int q0 = max(excl, w0) - w0, q1 = min(excl + L, w0 + kTile) - w0;
      for (int q = q0; q < q1; ++q) {
        smn = __dadd_rn(smn, c.w.b0[q]);
        smx = __dadd_rn(smx, c.w.b1[q]);
        imn += c.w.fl[q] & 1;
        imx += c.w.fl[q] >> 1;
      }
    }
    __syncwarp();
  }
  if (k >= 0) write_rec(P, c.S, k, smn, smx, imn, imx);
}

// Phase A. full: every row from the static partition tables; else the frontier lists.
__device__ void phase_activity(Ctx& c, ParCtl* pc, int par, bool full)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  {
    const int n       = full ? P.n_seg : ldv(&pc->n_dseg);
    const int2* tasks = full ? P.seg_task : S.dseg[par];
    for (int t = warp_fetch(c, &pc->cur_seg, 1); t < n; t = warp_fetch(c, &pc->cur_seg, 1)) {
      const int2 tk = tasks[t];
      row_stream(c, tk.x, tk.y);
    }
  }
  if (full) {
    for (int t = warp_fetch(c, &pc->cur_s, 1); t < P.n_srtile; t = warp_fetch(c, &pc->cur_s, 1))
      act_tile_packed(c, t);
  } else {
    const int n = ldv(&pc->n_drow_s);
    for (int t = warp_fetch(c, &pc->cur_s, 32); t < n; t = warp_fetch(c, &pc->cur_s, 32))
      act_list_tile(c, S.drow_s[par], t, n);
  }
}

// ------------------------------------------------------------------ tightening

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
  for (int j = c.lane; j < t.nbuf; j += 32) c.S.changed[base + j] = c.w.chg[j];
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
    if (r > 0) c.w.chg[t.nbuf + __popc(ch & lanemask_lt())] = i;
    t.nbuf += __popc(ch);
    __syncwarp();
  }
}

// Long column: one warp, 4 row-record gathers per lane in flight, (value, position) reduction.
__device__ int tighten_warp(Ctx& c, int i)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const double2 b     = S.bounds[i];
  const bool integer  = __ldg(P.is_int + i) != 0;
  Fold f{b.x, -1, b.y, -1};
  const int cs = __ldg(P.col_start + i), ce = __ldg(P.col_start + i + 1);
  for (int base = cs; base < ce; base += kTile) {
    int k[kEPL];
    double a[kEPL];
    RowRec r[kEPL];
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const int e = base + h * 32 + c.lane;
      k[h]        = e < ce ? __ldg(P.col_row + e) : -1;
      a[h]        = e < ce ? __ldg(P.col_val + e) : 0.0;
    }
#pragma unroll
    for (int h = 0; h < kEPL; ++h)
      if (k[h] >= 0) r[h] = ld_rec(S.rec + k[h]);
#pragma unroll
    for (int h = 0; h < kEPL; ++h)
      if (k[h] >= 0) fold_entry(f, b.x, b.y, integer, a[h], r[h], S.aux, k[h], base + h * 32 + c.lane);
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

// Candidates of up to 128 entries (row k[h], coefficient a[h], owner variable own[h] whose bounds
// are in w.vb) into shared memory: b0 = lower-bound candidates, b1 = upper-bound candidates.
__device__ __forceinline__ void stage_candidates(Ctx& c, const int* k, const double* a, const int* own)
{
  RowRec r[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h)
    if (k[h] >= 0) r[h] = ld_rec(c.S.rec + k[h]);
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    double cl = -INFINITY, cu = INFINITY;
    if (k[h] >= 0) {
      const double2 b = c.w.vb[own[h]];
      entry_candidates(b.x, b.y, c.w.vint[own[h]] != 0, a[h], r[h], c.S.aux, k[h], cl, cu);
    }
    c.w.b0[h * 32 + c.lane] = cl;
    c.w.b1[h * 32 + c.lane] = cu;
  }
}

// Packed tile of short columns (full rounds).
__device__ void tighten_tile_packed(Ctx& c, int t, ParCtl* pc, Tally& ty)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int v0 = __ldg(P.sc_tile + t), v1 = __ldg(P.sc_tile + t + 1);
  const int p0 = __ldg(P.sc_ptr + v0), p1 = __ldg(P.sc_ptr + v1);
  int i = -1;
  if (c.lane < v1 - v0) {
    i                  = __ldg(P.scol + v0 + c.lane);
    c.w.vb[c.lane]     = S.bounds[i];
    c.w.vint[c.lane]   = __ldg(P.is_int + i);
  }
  int k[kEPL], own[kEPL];
  double a[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    const int f = p0 + h * 32 + c.lane;
    k[h]        = f < p1 ? __ldg(P.sc_row + f) : -1;
    a[h]        = f < p1 ? __ldg(P.sc_val + f) : 0.0;
    own[h]      = f < p1 ? __ldg(P.sc_own + f) : 0;
  }
  __syncwarp();
  stage_candidates(c, k, a, own);
  __syncwarp();
  int res = 0;
  if (i >= 0) {
    const double2 b = c.w.vb[c.lane];
    double nl = b.x, nu = b.y;
    const int q0 = __ldg(P.sc_ptr + v0 + c.lane) - p0, q1 = __ldg(P.sc_ptr + v0 + c.lane + 1) - p0;
    for (int q = q0; q < q1; ++q) {
      const double cl = c.w.b0[q], cu = c.w.b1[q];
      if (nl < cl) nl = cl;
      if (cu < nu) nu = cu;
    }
    res = finish_var(S.bounds + i, b.x, b.y, nl, nu, c.w.vint[c.lane] != 0, c.lim);
  }
  tally(c, pc, ty, i, res);
  __syncwarp();
}

// Listed short columns (frontier rounds).
__device__ void tighten_list_tile(Ctx& c, const int* ids, int base, int n, ParCtl* pc, Tally& ty)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int j = base + c.lane;
  const int i = j < n ? ids[j] : -1;
  int cs = 0, L = 0;
  double2 b = make_double2(0.0, 0.0);
  bool integer = false;
  if (i >= 0) {
    cs      = __ldg(P.col_start + i);
    L       = __ldg(P.col_start + i + 1) - cs;
    b       = S.bounds[i];
    integer = __ldg(P.is_int + i) != 0;
  }
  c.w.vb[c.lane]   = b;
  c.w.vint[c.lane] = integer ? 1 : 0;
  int excl;
  const int T = list_tile_setup(c, cs, L, excl);
  double nl = b.x, nu = b.y;
  for (int w0 = 0; w0 < T; w0 += kTile) {
    int k[kEPL], own[kEPL];
    double a[kEPL];
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const int f = w0 + h * 32 + c.lane;
      k[h]        = -1;
      a[h]        = 0.0;
      own[h]      = 0;
      if (f < T) {
        const int o = owner_of(c.w.off, f);
        const int e = c.w.st[o] + (f - c.w.off[o]);
        k[h]        = __ldg(P.col_row + e);
        a[h]        = __ldg(P.col_val + e);
        own[h]      = o;
      }
    }
    stage_candidates(c, k, a, own);
    __syncwarp();
    if (i >= 0) {
      const int q0 = max(excl, w0) - w0, q1 = min(excl + L, w0 + kTile) - w0;
      for (int q = q0; q < q1; ++q) {
        const double cl = c.w.b0[q], cu = c.w.b1[q];
        if (nl < cl) nl = cl;
        if (cu < nu) nu = cu;
      }
    }
    __syncwarp();
  }
  int res = 0;
  if (i >= 0) res = finish_var(S.bounds + i, b.x, b.y, nl, nu, integer, c.lim);
  tally(c, pc, ty, i, res);
}

__device__ void phase_tighten(Ctx& c, ParCtl* pc, int par, bool full)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  Tally t{0, 0, 0ull, 0};
  {
    const int n    = full ? P.n_mcol : ldv(&pc->n_dvar_m);
    const int* ids = full ? P.mcol : S.dvar_m[par];
    for (int q = warp_fetch(c, &pc->cur_vm, 1); q < n; q = warp_fetch(c, &pc->cur_vm, 1)) {
      const int i = ids[q];
      const int r = tighten_warp(c, i);
      tally(c, pc, t, c.lane == 0 ? i : -1, c.lane == 0 ? r : 0);
    }
  }
  if (full) {
    for (int q = warp_fetch(c, &pc->cur_vs, 1); q < P.n_sctile; q = warp_fetch(c, &pc->cur_vs, 1))
      tighten_tile_packed(c, q, pc, t);
  } else {
    const int n = ldv(&pc->n_dvar_s);
    for (int q = warp_fetch(c, &pc->cur_vs, 32); q < n; q = warp_fetch(c, &pc->cur_vs, 32))
      tighten_list_tile(c, S.dvar_s[par], q, n, pc, t);
  }
  flush_changed(c, pc, t);
  const int cr = warp_sum(t.crossed);
  const int ar = __any_sync(FULL, t.any_rows);
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

// Phase C: rows(changed) → next round's dirty rows: short rows, long-row segment tasks, and
// 256-entry var-expansion tasks. 4 incidences per lane in flight.
__device__ void phase_expand_rows(Ctx& c, ParCtl* pc, ParCtl* qc, int qpar, unsigned stamp)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int nch       = ldv(&pc->n_changed);
  unsigned long long roww = 0;
  for (int t = warp_fetch(c, &pc->cur_x1, 32); t < nch; t = warp_fetch(c, &pc->cur_x1, 32)) {
    const int j = t + c.lane;
    const int i = j < nch ? S.changed[j] : -1;
    int cs = 0, L = 0;
    if (i >= 0) {
      cs = __ldg(P.col_start + i);
      L  = __ldg(P.col_start + i + 1) - cs;
    }
    int excl;
    const int T = list_tile_setup(c, cs, L, excl);
    for (int w0 = 0; w0 < T; w0 += kTile) {
      int k[kEPL];
      bool nw[kEPL];
#pragma unroll
      for (int h = 0; h < kEPL; ++h) {
        const int f = w0 + h * 32 + c.lane;
        k[h]        = -1;
        if (f < T) {
          const int o = owner_of(c.w.off, f);
          k[h]        = __ldg(P.col_row + c.w.st[o] + (f - c.w.off[o]));
        }
      }
#pragma unroll
      for (int h = 0; h < kEPL; ++h) nw[h] = k[h] >= 0 && atomicExch(S.row_stamp + k[h], stamp) != stamp;
      int RL[kEPL], n_s = 0, n_g = 0, n_x = 0, n_a = 0;
#pragma unroll
      for (int h = 0; h < kEPL; ++h) {
        RL[h] = nw[h] ? __ldg(P.row_start + k[h] + 1) - __ldg(P.row_start + k[h]) : 0;
        roww += (unsigned long long)RL[h];
        n_a += nw[h];
        n_s += nw[h] && RL[h] <= kShortNnz;
        n_g += (nw[h] && RL[h] > kShortNnz) ? (RL[h] + kSumSegment - 1) / kSumSegment : 0;
        n_x += (nw[h] && RL[h] > 0) ? (RL[h] + kXChunk - 1) / kXChunk : 0;
      }
      warp_alloc(&qc->n_drow_all, n_a, c.lane);
      int ps = warp_alloc(&qc->n_drow_s, n_s, c.lane);
      int pg = warp_alloc(&qc->n_dseg, n_g, c.lane);
      int px = warp_alloc(&qc->n_xtask, n_x, c.lane);
#pragma unroll
      for (int h = 0; h < kEPL; ++h) {
        if (!nw[h]) continue;
        if (RL[h] <= kShortNnz) S.drow_s[qpar][ps++] = k[h];
        else
          for (int s = 0; s * kSumSegment < RL[h]; ++s) S.dseg[qpar][pg++] = make_int2(k[h], s);
        for (int s = 0; s * kXChunk < RL[h]; ++s) S.xtask[qpar][px++] = make_int2(k[h], s);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) roww += __shfl_xor_sync(FULL, roww, o);
  if (c.lane == 0 && roww) atomicAdd(&qc->roww, roww);
}

// Phase D: dirty rows → next round's dirty vars (classified by column length).
__device__ void phase_expand_vars(Ctx& c, ParCtl* pc, ParCtl* qc, int qpar, unsigned stamp)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int ntask     = ldv(&qc->n_xtask);
  unsigned long long colw = 0;
  constexpr int H = kXChunk / 32;
  for (int t = warp_fetch(c, &pc->cur_x2, 1); t < ntask; t = warp_fetch(c, &pc->cur_x2, 1)) {
    const int2 tk = S.xtask[qpar][t];
    const int rs = __ldg(P.row_start + tk.x), re = __ldg(P.row_start + tk.x + 1);
    const int e0 = rs + tk.y * kXChunk, e1 = min(re, e0 + kXChunk);
    int vj[H];
    bool nw[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int e = e0 + h * 32 + c.lane;
      vj[h]       = e < e1 ? __ldg(P.row_col + e) : -1;
    }
#pragma unroll
    for (int h = 0; h < H; ++h) nw[h] = vj[h] >= 0 && atomicExch(S.var_stamp + vj[h], stamp) != stamp;
    int CL[H], n_s = 0, n_m = 0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      CL[h] = nw[h] ? __ldg(P.col_start + vj[h] + 1) - __ldg(P.col_start + vj[h]) : 0;
      colw += (unsigned long long)CL[h];
      n_s += nw[h] && CL[h] <= kShortNnz;
      n_m += nw[h] && CL[h] > kShortNnz;
    }
    int ps = warp_alloc(&qc->n_dvar_s, n_s, c.lane);
    int pm = warp_alloc(&qc->n_dvar_m, n_m, c.lane);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      if (!nw[h]) continue;
      if (CL[h] <= kShortNnz) S.dvar_s[qpar][ps++] = vj[h];
      else S.dvar_m[qpar][pm++] = vj[h];
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

#ifndef BP_MIN_BLOCKS
#define BP_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(kThreads, BP_MIN_BLOCKS)
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
  const int warp = threadIdx.x >> 5;
  Ctx c{P, S, lim, sm, sm.w[warp], (int)(threadIdx.x & 31), warp};

  if (mode == MODE_ACTIVITY) {
    phase_activity(c, &S.ctl->par[1], 1, full_first != 0);
    return;
  }
  if (mode == MODE_TIGHTEN) {
    phase_tighten(c, &S.ctl->par[1], 1, full_first != 0);
    return;
  }

  const unsigned long long t0 = globaltimer();
  const bool timed            = isfinite(lim.time_limit);
  const bool lead             = blockIdx.x == 0 && threadIdx.x == 0;
  bool full                   = true;  // round 1 is always a full sweep (propagation.hpp:442)
  bool any_change             = false;
  int status = BP_STATUS_UNSET, crossed_out = 0;
  int rounds = 0;
  while (rounds < lim.max_rounds) {
    ++rounds;
    const int ppar = rounds & 1, qpar = ppar ^ 1;
    ParCtl* pc     = &S.ctl->par[ppar];
    ParCtl* qc     = &S.ctl->par[qpar];
    long long* st  = stats ? stats + (long long)(rounds - 1) * kStatCols : nullptr;
    const bool fr  = full || !lim.incremental;
    phase_activity(c, pc, ppar, fr);
    grid.sync();
    if (st && lead) st[6] = (long long)(globaltimer() - t0);
    if (lead) {
      zero_par(qc);  // safe: every block has finished reading the previous round's counters
      if (timed && (double)(globaltimer() - t0) * 1e-9 >= lim.time_limit) pc->stop = 1;
    }
    phase_tighten(c, pc, ppar, fr);
    grid.sync();
    const int cr = ldv(&pc->n_crossed);
    const int nc = ldv(&pc->n_changed);
    if (st && lead) {
      st[7] = (long long)(globaltimer() - t0);
      st[8] = st[9] = st[7];
      st[0] = fr ? 1 : 0;
      st[1] = fr ? P.m : ldv(&pc->n_drow_all);
      st[2] = fr ? P.nnz : (long long)ldv(&pc->roww);
      st[3] = fr ? P.n : ldv(&pc->n_dvar_s) + ldv(&pc->n_dvar_m);
      st[4] = fr ? P.nnz : (long long)ldv(&pc->colw);
      st[5] = nc;
    }
    if (cr > 0) {
      status      = BP_STATUS_INFEASIBLE;
      crossed_out = cr;
      break;
    }
    if (nc == 0) break;
    any_change = true;
    if (!ldv(&pc->any_rows)) break;  // dirty_rows.empty() (propagation.hpp:481)
    if (rounds >= lim.max_rounds) break;
    if (ldv(&pc->stop)) break;       // time limit (propagation.hpp:439)
    if (!lim.incremental || ldv(&pc->colnnz) > dense_thr) {
      full = true;
      continue;
    }
    const unsigned stamp = stamp_base + (unsigned)rounds;
    phase_expand_rows(c, pc, qc, qpar, stamp);
    grid.sync();
    if (st && lead) st[8] = st[9] = (long long)(globaltimer() - t0);
    if (ldv(&qc->roww) > dense_thr) {
      full = true;
      continue;
    }
    phase_expand_vars(c, pc, qc, qpar, stamp);
    grid.sync();
    if (st && lead) st[9] = (long long)(globaltimer() - t0);
    // a frontier round costs ~ its gathers (row nnz + col nnz); a full round ~ 2 N = 8 dense_thr
    full = dense_thr != ~0ull && ldv(&qc->roww) + ldv(&qc->colw) > 6 * dense_thr;
  }
  if (lead) {
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
  d.n_srtile  = n_srtile;
  d.srow      = srow.p;
  d.sr_ptr    = sr_ptr.p;
  d.sr_col    = sr_col.p;
  d.sr_val    = sr_val.p;
  d.sr_tile   = sr_tile.p;
  d.n_seg     = n_seg;
  d.seg_task  = seg_task.p;
  d.seg_base  = seg_base.p;
  d.n_scol    = n_scol;
  d.n_sctile  = n_sctile;
  d.scol      = scol.p;
  d.sc_ptr    = sc_ptr.p;
  d.sc_row    = sc_row.p;
  d.sc_val    = sc_val.p;
  d.sc_own    = sc_own.p;
  d.sc_tile   = sc_tile.p;
  d.n_mcol    = n_mcol;
  d.mcol      = mcol.p;
  return d;
}

namespace {

// Packs the short items (nnz <= kShortNnz) of a compressed matrix view contiguously, in natural
// order, and groups them into tiles of <= 32 items and <= kTile entries.
struct Packed {
  std::vector<int> ids, ptr, idx, tile;
  std::vector<double> val;
  std::vector<uint8_t> own;
};

Packed pack_short(int count, const int* start, const int* idx, const double* val)
{
  Packed pk;
  pk.ptr.push_back(0);
  for (int k = 0; k < count; ++k) {
    const int L = start[k + 1] - start[k];
    if (L > kShortNnz) continue;
    pk.ids.push_back(k);
    for (int e = start[k]; e < start[k + 1]; ++e) {
      pk.idx.push_back(idx[e]);
      pk.val.push_back(val[e]);
    }
    pk.ptr.push_back((int)pk.idx.size());
  }
  pk.own.resize(pk.idx.size());
  const int ns = (int)pk.ids.size();
  int r = 0;
  while (r < ns) {
    pk.tile.push_back(r);
    const int base = pk.ptr[r];
    int q          = r;
    while (q < ns && q - r < 32 && pk.ptr[q + 1] - base <= kTile) {
      for (int e = pk.ptr[q]; e < pk.ptr[q + 1]; ++e) pk.own[e] = (uint8_t)(q - r);
      ++q;
    }
    r = q;
  }
  pk.tile.push_back(ns);
  return pk;
}

}  // namespace

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
  const int* col_start = P.h_col_start.data();
  P.row_start.upload(row_start, m + 1);
  P.row_col.upload(row_col, N);
  P.row_val.upload(row_val, N);
  P.col_start.upload(col_start, n + 1);
  P.col_row.upload(col_row_in, N);
  P.col_val.upload(col_val_in, N);
  std::vector<double2> cons(m);
  for (int k = 0; k < m; ++k) cons[k] = make_double2(cons_lower[k], cons_upper[k]);
  P.cons.upload(cons);
  P.is_int.upload(is_integer, n);

  // Short rows / columns: packed tiles.
  {
    Packed r = pack_short(m, row_start, row_col, row_val);
    P.n_srow   = (int)r.ids.size();
    P.n_srtile = (int)r.tile.size() - 1;
    P.srow.upload(r.ids);
    P.sr_ptr.upload(r.ptr);
    P.sr_col.upload(r.idx);
    P.sr_val.upload(r.val);
    P.sr_tile.upload(r.tile);
    Packed c = pack_short(n, col_start, col_row_in, col_val_in);
    P.n_scol   = (int)c.ids.size();
    P.n_sctile = (int)c.tile.size() - 1;
    P.scol.upload(c.ids);
    P.sc_ptr.upload(c.ptr);
    P.sc_row.upload(c.idx);
    P.sc_val.upload(c.val);
    P.sc_own.upload(c.own);
    P.sc_tile.upload(c.tile);
  }
  // Long rows: one task per 16384-entry segment, longest segments first (the fold of a segment
  // is a sequential chain, so long chains must start early).
  std::vector<int> seg_base(m, -1);
  std::vector<std::pair<int, int2>> tasks;  // (segment length, task)
  int slot = 0;
  for (int k = 0; k < m; ++k) {
    const int L = row_start[k + 1] - row_start[k];
    if (L <= kShortNnz) continue;
    const int ns = (L + kSumSegment - 1) / kSumSegment;
    if (ns > 1) {
      seg_base[k] = slot;
      slot += ns;
    }
    for (int s = 0; s < ns; ++s)
      tasks.push_back({std::min(L - s * kSumSegment, kSumSegment), make_int2(k, s)});
  }
  std::stable_sort(tasks.begin(), tasks.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<int2> seg_task(tasks.size());
  for (size_t j = 0; j < tasks.size(); ++j) seg_task[j] = tasks[j].second;
  P.n_seg  = (int)seg_task.size();
  P.n_part = slot;
  P.seg_task.upload(seg_task);
  P.seg_base.upload(seg_base);
  // Long columns, longest first.
  std::vector<int> mcol;
  for (int i = 0; i < n; ++i)
    if (col_start[i + 1] - col_start[i] > kShortNnz) mcol.push_back(i);
  std::stable_sort(mcol.begin(), mcol.end(), [&](int a, int b) {
    return col_start[a + 1] - col_start[a] > col_start[b + 1] - col_start[b];
  });
  P.n_mcol = (int)mcol.size();
  P.mcol.upload(mcol);

  // Workspace.
  const size_t mm = (size_t)std::max(m, 1), nn = (size_t)std::max(n, 1);
  P.bounds.alloc(nn);
  P.rec.alloc(mm);
  P.aux.alloc(mm);
  P.seg_part.alloc(std::max(slot, 1));
  P.seg_done.alloc(mm);
  BP_CUDA(cudaMemset(P.seg_done.p, 0, sizeof(int) * mm));
  P.row_stamp.alloc(mm);
  P.var_stamp.alloc(nn);
  BP_CUDA(cudaMemset(P.row_stamp.p, 0, sizeof(unsigned) * mm));
  BP_CUDA(cudaMemset(P.var_stamp.p, 0, sizeof(unsigned) * nn));
  // int lists per parity: drow_s (m), dvar_s, dvar_m (n each); changed (n)
  P.lists_i.alloc(2 * (mm + 2 * nn) + nn);
  // int2 lists per parity: dseg (all segment tasks), xtask (N/256 + m)
  const size_t nseg_cap = (size_t)std::max(P.n_seg, 1);
  const size_t nx_cap   = (size_t)(N / 256) + mm + 1;
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
    S.drow_s[q] = pi; pi += mm;
    S.dvar_s[q] = pi; pi += nn;
    S.dvar_m[q] = pi; pi += nn;
    S.dseg[q]   = pi2; pi2 += nseg_cap;
    S.xtask[q]  = pi2; pi2 += nx_cap;
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
  DevProblem d = P.dev();
  DevState st  = P.st;
  Limits l     = lim;
  int md       = (int)mode;
  int ff       = full ? 1 : 0;
  // stamps: one value per round, never reused until wrap-around (then the stamp arrays reset)
  if (P.stamp_base > 0xF0000000u - (unsigned)std::max(lim.max_rounds, 1) - 2) {
    BP_CUDA(cudaMemsetAsync(P.row_stamp.p, 0, sizeof(unsigned) * P.row_stamp.n, s));
    BP_CUDA(cudaMemsetAsync(P.var_stamp.p, 0, sizeof(unsigned) * P.var_stamp.n, s));
    P.stamp_base = 1;
  }
  unsigned sb = P.stamp_base;
  P.stamp_base += (unsigned)std::max(lim.max_rounds, 1) + 1;
  unsigned long long dense_thr =
      (flags & ENGINE_FORCE_FRONTIER) ? ~0ull : (unsigned long long)(P.nnz / 4);
  long long* stp = d_stats;
  void* args[]   = {&d, &st, &l, &md, &ff, &sb, &dense_thr, &stp};
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
  std::vector<int> sr;
  std::vector<int2> sg;
  for (int j = 0; j < nrows; ++j) {
    const int k = rows[j];
    const int L = P.h_row_start[k + 1] - P.h_row_start[k];
    if (L <= kShortNnz) sr.push_back(k);
    else
      for (int q = 0; q * kSumSegment < L; ++q) sg.push_back(make_int2(k, q));
  }
  DevState& S = P.st;
  if (!sr.empty())
    BP_CUDA(cudaMemcpyAsync(S.drow_s[1], sr.data(), sr.size() * 4, cudaMemcpyHostToDevice, s));
  if (!sg.empty())
    BP_CUDA(cudaMemcpyAsync(S.dseg[1], sg.data(), sg.size() * 8, cudaMemcpyHostToDevice, s));
  int cnt[3] = {(int)sr.size(), (int)sg.size(), nrows};
  BP_CUDA(cudaMemcpyAsync(&S.ctl->par[1].n_drow_s, cnt, sizeof(cnt), cudaMemcpyHostToDevice, s));
  BP_CUDA(cudaStreamSynchronize(s));
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
  BP_CUDA(cudaStreamSynchronize(s));
}

}  // namespace bp
