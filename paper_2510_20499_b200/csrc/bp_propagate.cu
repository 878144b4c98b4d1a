// Persistent, device-resident bound propagation for sm_100a.
//
// One cooperative kernel runs the whole `propagate` loop of the reference
// (propagation.hpp:418-486) with no host round trip per round. The path is a sparse fp64 gather
// whose cost is memory-level parallelism and two serial chains (the reference's sequential
// activity sums and the std::min/max fold of each column), so the kernel is organised around
// keeping gathers in flight and taking those chains off the critical path.
//
// FULL round (round 1, and any round whose frontier is a large part of the matrix):
//   F2  rows: per 16384-entry segment of a long row, one warp streams the row's indices and
//       coefficients coalesced and gathers its bounds (two chunks in flight) while lanes 0/1 run
//       the reference's sequential min/max sums (zero contributions skipped: exact, the running
//       sum is never -0.0); packed tiles of short rows fold one row per lane. Right after a
//       row's activity is known, every entry's candidate bounds for its variable are computed
//       (unless provably non-improving: candidate gating) and the ones strictly improving the
//       round-start bound are published into per-variable slots with order-preserving 64-bit
//       atomics (fused tightening: no CSC pass, no second gather of row records). ─ grid.sync
//   F4  finalize: per variable, the slot gives the std::min/max fold result (ties at +-0.0 are
//       resolved by the smallest row = first CSC position), then the reference's crossing /
//       hair-crossing / threshold rules (propagation.hpp:354-369).                  ─ grid.sync
// FRONTIER round (propagation.hpp:442-447 with dirty rows / dirty vars):
//   P2 activities (dirty rows) ─ B tighten the dirty vars over the
//   CSC (row-record gathers; long columns reduced as a lexicographic (value, CSC position)
//   min/max) ─ C/D frontier expansion.
// Evaluating a superset of the reference's dirty sets yields bit-identical results (DESIGN.md §2,
// SURVEY §8a A12 lemma), so the engine may pick either round type for any round.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "bp_engine.cuh"

namespace cg = cooperative_groups;

namespace bp {

std::atomic<long long> g_kernel_launches{0};

namespace {

constexpr int kThreads  = 256;
constexpr int kWarps    = kThreads / 32;
constexpr unsigned FULL = 0xffffffffu;
constexpr int kEPL      = kTile / 32;
constexpr int kIntBit   = (int)0x80000000u;
#ifndef BP_ROW_GATE
#define BP_ROW_GATE 1
#endif
constexpr bool kRowGate = BP_ROW_GATE != 0;  // row-level candidate gating (maxima in the fold pass)

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
__device__ __forceinline__ unsigned ldv(const unsigned* p) { return *(const volatile unsigned*)p; }
__device__ __forceinline__ unsigned long long ldv(const unsigned long long* p)
{
  return *(const volatile unsigned long long*)p;
}
__device__ __forceinline__ RowRec ld_rec_cg(const RowRec* p)
{
  RowRec r;
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.min), "=d"(r.max), "=d"(r.g), "=d"(r.h)
               : "l"(p));
  return r;
}

struct WarpSmem {
  double b0[kFoldChunk];     // min contributions / lower-bound candidates
  double b1[kFoldChunk];     // max contributions / upper-bound candidates
  unsigned char fl[kTile];   // infinite-contributor flags (bit 0 min, bit 1 max)
  int off[32];               // list tiles: exclusive entry offsets of the 32 items
  int st[32];                //             their first entry
  double2 vb[32];            // tighten tiles: the 32 variables' bounds
  double ract[32][2];        // short-row tiles: finite parts of each row's min/max activity
  int rinf[32][2];           //                  and infinite-contributor counts
  int rk[32];                //                  and row ids (row bounds go to vb)
  unsigned char vint[32];    // tighten tiles: integrality
  int chg[64];               // changed-var staging before a global append
};

struct Smem {
  WarpSmem w[kWarps];
  int blk_crossed;
  int blk_any_rows;
  unsigned long long blk_colnnz;
  unsigned long long blk_reach, blk_hreach;
};

struct Ctx {
  const DevProblem& P;
  const DevState& S;
  const Limits& lim;
  Smem& sm;
  WarpSmem& w;
  int lane, warp;
  unsigned touch = 0;  // dirty-filtered round stamp: publishes list their variables (finalize)
};

// Debug counters (BP_DEBUG=1): per task kind total / max cycles and count.
// Task / gate statistics (BP_DEBUG=1) only exist in builds with -DBP_DBG_STATS=1: compiled into the
// unrolled row loops they cost code size (instruction-cache misses) even when disabled at run time.
#ifndef BP_DBG_STATS
#define BP_DBG_STATS 0
#endif
#define DBG_ON(S) (BP_DBG_STATS && (S).dbg)

__device__ __forceinline__ void dbg_task(Ctx& c, int kind, long long c0)
{
  if (DBG_ON(c.S) && c.lane == 0) {
    const unsigned long long d = (unsigned long long)(clock64() - c0);
    atomicAdd(c.S.dbg + 3 * kind, d);
    atomicMax(c.S.dbg + 3 * kind + 1, d);
    atomicAdd(c.S.dbg + 3 * kind + 2, 1ull);
  }
}

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

// Work cursor over `lim` items in chunks of `step`: a grid-wide atomic cursor with the next fetch
// in flight while the current chunk runs (and no fetch past the end). With `may_static`, when the
// whole range fits one chunk per warp of the grid, warps take chunks statically (no atomics: an
// empty or small list costs nothing) -- only for tasks no other warp waits on: a task that spins on
// another task's result (heavy segment folds on their pieces) must follow the dynamic order, in
// which every producer is claimed by a running warp before any consumer is (progress without
// grid-wide co-residency, e.g. next to other streams' kernels).
struct Prefetch {
  Ctx& c;
  int* cur;
  int step, t, nx, lim;
  bool stat;
  __device__ Prefetch(Ctx& c_, int* cur_, int step_, int lim_ = 0x3FFFFFFF, bool may_static = false)
      : c(c_), cur(cur_), step(step_), lim(lim_)
  {
    const int nw = gridDim.x * kWarps;
    stat         = lim <= 0 || (may_static && (long long)lim <= (long long)step * nw);
    if (stat) {
      t = lim <= 0 ? 0x3FFFFFFF : (blockIdx.x * kWarps + c.warp) * step;
    } else {
      t = 0x3FFFFFFF;
      if (c.lane == 0) t = claim();
      t = __shfl_sync(FULL, t, 0);
      issue();
    }
  }
  // an exhausted cursor is only read: with short lists most of the grid's warps would otherwise
  // queue atomics on one address for nothing (a value >= lim is a claim past the end either way)
  __device__ __forceinline__ int claim() { return ldv(cur) < lim ? atomicAdd(cur, step) : lim; }
  __device__ __forceinline__ void issue()
  {
    nx = 0x3FFFFFFF;
    if (c.lane == 0 && t < lim) nx = claim();
  }
  __device__ __forceinline__ void advance()
  {
    if (stat) {
      t = 0x3FFFFFFF;
    } else {
      t = __shfl_sync(FULL, nx, 0);
      issue();
    }
  }
};

// Up to 32 listed items as one flattened entry stream: returns the stream length and this lane's
// item offset; fills w.off / w.st.
__device__ __forceinline__ int list_tile_setup(Ctx& c, int first, int len, int& excl)
{
  const int incl  = warp_incl_scan(len, c.lane);
  excl            = incl - len;
  c.w.off[c.lane] = excl;
  c.w.st[c.lane]  = first;
  __syncwarp();
  return __shfl_sync(FULL, incl, 31);
}

// ------------------------------------------------------------------ candidate publication

// Records a zero candidate of row k in a slot's zero-tie word: the smallest row wins (the first CSC
// position, i.e. the reference's fold keeps it), and a row replaces its own earlier record -- with
// persistent slots (dirty-filtered rounds) a dirty row republishes, and its zero may change sign.
__device__ __forceinline__ void publish_zero(unsigned* z, int k, bool neg)
{
  const unsigned nv = ((unsigned)k << 1) | (neg ? 1u : 0u);
  unsigned cur      = *(volatile unsigned*)z;
  while (cur != nv && (cur >> 1) >= (unsigned)k) {  // kZeroEmpty >> 1 exceeds every row id
    const unsigned prev = atomicCAS(z, cur, nv);
    if (prev == cur) break;
    cur = prev;
  }
}

// Publishes the candidates of one (row k, variable) entry that strictly improve the round-start
// bounds (lo, up) into the variable's slot.
__device__ __forceinline__ bool publish(CandSlot* s, double cl, double cu, double lo, double up,
                                       int k)
{
  if (cu < up) {
    atomicMin(&s->up_key, okey(cu == 0.0 ? 0.0 : cu));
    if (cu == 0.0) publish_zero(&s->up_zero, k, signbit(cu));
  }
  if (lo < cl) {
    atomicMax(&s->lo_key, okey(cl == 0.0 ? 0.0 : cl));
    if (cl == 0.0) publish_zero(&s->lo_zero, k, signbit(cl));
  }
  return cu < up || lo < cl;
}

#ifndef BP_EMIT_NOINLINE
#define BP_EMIT_NOINLINE 0
#endif
// The candidates of one non-quiet entry (cand_explicit + publish). Inlined: an out-of-line copy
// (BP_EMIT_NOINLINE=1) shrinks k_rows_full's code by a fifth but costs C2 5% (call overhead and
// register saves around the call in the row loops; tools/gpu_ab.sh).
#if BP_EMIT_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void emit_cand(const DevState& S, unsigned touch, int ci, double a, double lo, double up, double mnf,
               int nmn, double mxf, int nmx, double g, double h, int k)
{
  double cl, cu;
  cand_explicit(lo, up, ci < 0, a, mnf, nmn, mxf, nmx, g, h, cl, cu);
  const int v = ci & ~kIntBit;
  // a dirty-filtered round lists the variables it publishes to: only their slots can have changed,
  // so its finalize visits them alone (the others' slots and bounds are those of the last finalize)
  if (publish(S.slot + v, cl, cu, lo, up, k) && touch && atomicExch(S.vtouch + v, touch) != touch)
    S.touched[atomicAdd(&S.ctl->n_touch, 1)] = v;
}

// Dirty filter of a full round's row tasks: ds = 0 (true full round) or the stamp the previous
// round's finalize wrote into row_stamp for the rows of its changed vars.
__device__ __forceinline__ bool row_live(const DevState& S, int k, unsigned ds)
{
  return ds == 0 || __ldcg(S.row_stamp + k) == ds;
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

// Candidates of entries [e0, e1) of long row k whose activity is (mnf, nmn, mxf, nmx, g, h).
// Bounds are gathered straight from the (L2-resident) bounds array.
__device__ void long_candidates(Ctx& c, int k, int e0, int e1, double mnf, int nmn, double mxf,
                                int nmx, double g, double hh)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int rs        = __ldg(P.row_start + k);
  for (int j0 = e0; j0 < e1; j0 += kTile) {
    int ci[kEPL];
    double a[kEPL];
    double2 bd[kEPL];
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const int e = j0 + h * 32 + c.lane;
      ci[h]       = e < e1 ? __ldg(P.row_ci + rs + e) : -1;
      a[h]        = e < e1 ? __ldg(P.row_val + rs + e) : 0.0;
    }
#pragma unroll
    for (int h = 0; h < kEPL; ++h)
      bd[h] = ci[h] != -1 ? S.bounds[ci[h] & ~kIntBit] : make_double2(0.0, 0.0);
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      if (ci[h] == -1) continue;
      double tw, pm;
      entry_reach(a[h], bd[h].x, bd[h].y, ci[h] < 0, tw, pm);
      if (entry_quiet(tw, pm, mnf, nmn, mxf, nmx, g, hh)) continue;
      emit_cand(S, c.touch, ci[h], a[h], bd[h].x, bd[h].y, mnf, nmn, mxf, nmx, g, hh, k);
    }
  }
}

// Sequential left-to-right sum of src[0..cnt) onto acc (the reference's fold order), with the
// shared-memory loads of the next 8 values in flight while the current 8 are added.
__device__ __forceinline__ double fold_seq(const double* src, int cnt, double acc)
{
  const double2* s2 = reinterpret_cast<const double2*>(src);
  int j             = 0;
  if (cnt >= 8) {
    double2 v0 = s2[0], v1 = s2[1], v2 = s2[2], v3 = s2[3];
    for (j = 8; j + 8 <= cnt; j += 8) {
      const double2 w0 = s2[j / 2], w1 = s2[j / 2 + 1], w2 = s2[j / 2 + 2], w3 = s2[j / 2 + 3];
      acc = __dadd_rn(acc, v0.x); acc = __dadd_rn(acc, v0.y);
      acc = __dadd_rn(acc, v1.x); acc = __dadd_rn(acc, v1.y);
      acc = __dadd_rn(acc, v2.x); acc = __dadd_rn(acc, v2.y);
      acc = __dadd_rn(acc, v3.x); acc = __dadd_rn(acc, v3.y);
      v0 = w0; v1 = w1; v2 = w2; v3 = w3;
    }
    acc = __dadd_rn(acc, v0.x); acc = __dadd_rn(acc, v0.y);
    acc = __dadd_rn(acc, v1.x); acc = __dadd_rn(acc, v1.y);
    acc = __dadd_rn(acc, v2.x); acc = __dadd_rn(acc, v2.y);
    acc = __dadd_rn(acc, v3.x); acc = __dadd_rn(acc, v3.y);
  }
  for (; j < cnt; ++j) acc = __dadd_rn(acc, src[j]);
  return acc;
}

// Tail of a segment fold (warp-uniform inputs): combines the segment partials of multi-segment
// rows in segment order (propagation.hpp:182-188), writes the row record, and continues with the
// candidates (gated; inline for rows <= kCandSplit, else by publishing the row to the candidate
// pieces).
__device__ void fold_finish(Ctx& c, int k, int L, int seg, double smn, double smx, int imn, int imx,
                            double gtw, double gpm, bool cand, unsigned stamp)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int lane      = c.lane;
  const int nseg = (L + kSumSegment - 1) / kSumSegment;
  int final_row  = 0;  // 1 if this warp holds the row's final activity
  if (nseg == 1) {
    final_row = 1;
  } else {
    if (lane == 0) {
      const int base = __ldg(P.seg_base + k);
      SegPart sp;
      sp.min  = smn;
      sp.max  = smx;
      sp.nmin = imn;
      sp.nmax = imx;
      sp.tmax = gtw;
      sp.pmax = gpm;
      S.seg_part[base + seg] = sp;
      __threadfence();
      const int done = atomicAdd(&S.seg_done[k], 1);
      if (done == nseg - 1) {
        __threadfence();
        double tmn = 0.0, tmx = 0.0;
        int cmn = 0, cmx = 0;
        for (int q = 0; q < nseg; ++q) {  // row_activity's segment fold (propagation.hpp:182-188)
          const SegPart* sq = S.seg_part + base + q;
          tmn = __dadd_rn(tmn, __ldcg(&sq->min));
          tmx = __dadd_rn(tmx, __ldcg(&sq->max));
          cmn += __ldcg(&sq->nmin);
          cmx += __ldcg(&sq->nmax);
          gtw = fmax(gtw, __ldcg(&sq->tmax));
          gpm = fmax(gpm, __ldcg(&sq->pmax));
        }
        smn           = tmn;
        smx           = tmx;
        imn           = cmn;
        imx           = cmx;
        S.seg_done[k] = 0;
        final_row     = 1;
      }
    }
    final_row = __shfl_sync(FULL, final_row, 0);
    smn       = __shfl_sync(FULL, smn, 0);
    smx       = __shfl_sync(FULL, smx, 0);
    imn       = __shfl_sync(FULL, imn, 0);
    imx       = __shfl_sync(FULL, imx, 0);
    gtw       = __shfl_sync(FULL, gtw, 0);
    gpm       = __shfl_sync(FULL, gpm, 0);
  }
  if (!final_row) return;
  if (lane == 0) write_rec(P, S, k, smn, smx, imn, imx);
  if (!cand) return;
  const double2 cb = __ldg(&P.cons[k]);
  // row-level gating: no entry of the row can publish a candidate -> skip the candidate pass
  const bool quiet = kRowGate && entry_quiet(gtw, gpm, smn, imn, smx, imx, cb.y, cb.x);
  if (L > kCandSplit) {
    if (lane == 0) {
      S.rquiet[k] = quiet ? 1 : 0;
      __threadfence();
      atomicExch(S.ready + k, stamp);
    }
    return;
  }
  if (quiet) return;
  long_candidates(c, k, 0, L, smn, imn, smx, imx, cb.y, cb.x);
}

// F2 / P2: one 16384-entry segment of a long row, streamed in 128-entry chunks: the indices of
// chunk j+2 and the bound gathers of chunk j+1 are in flight while lanes 0/1 run the reference's
// sequential min/max sums over chunk j (zero contributions skipped: exact, the running sum is
// never -0.0). With `cand`, a single-segment row of <= kCandSplit entries publishes its
// candidates right away; longer rows publish their activity (ready stamp) for the parallel
// candidate pieces.
__device__ void long_fold(Ctx& c, int k, int seg, bool cand, unsigned stamp)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int lane      = c.lane;
  const int rs = __ldg(P.row_start + k), L = __ldg(P.row_start + k + 1) - rs;
  const int e0 = seg * kSumSegment, e1 = min(L, e0 + kSumSegment);
  constexpr int H = kEPL;
  int ci[H], ci2[H];
  double a[H], a2[H];
  double2 bd[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const int e  = e0 + h * 32 + lane;
    const int e2 = e + kTile;
    ci[h]        = e < e1 ? __ldg(P.row_ci + rs + e) : -1;
    a[h]         = e < e1 ? __ldg(P.row_val + rs + e) : 0.0;
    ci2[h]       = e2 < e1 ? __ldg(P.row_ci + rs + e2) : -1;
    a2[h]        = e2 < e1 ? __ldg(P.row_val + rs + e2) : 0.0;
  }
#pragma unroll
  for (int h = 0; h < H; ++h) bd[h] = ci[h] != -1 ? S.bounds[ci[h] & ~kIntBit] : make_double2(0.0, 0.0);
  double acc = 0.0;
  int imn = 0, imx = 0;
  double gtw = 0.0, gpm = 0.0;  // row-level gating maxima
  const unsigned lt = lanemask_lt();
  for (int base = e0; base < e1; base += kTile) {
    // order-preserving compaction of the non-zero contributions of each chain
    int pm = 0, px = 0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      double cm = 0.0, cx = 0.0;
      if (ci[h] != -1) {
        int i1, i2;
        contrib(a[h], bd[h].x, bd[h].y, cm, cx, i1, i2);
        imn += i1;
        imx += i2;
        if (cand && kRowGate) {
          double tw, pw;
          entry_reach(a[h], bd[h].x, bd[h].y, ci[h] < 0, tw, pw);
          gtw = fmax(gtw, tw);
          gpm = fmax(gpm, pw);
        }
      }
      const unsigned m = __ballot_sync(FULL, cm != 0.0);
      const unsigned x = __ballot_sync(FULL, cx != 0.0);
      if (cm != 0.0) c.w.b0[pm + __popc(m & lt)] = cm;
      if (cx != 0.0) c.w.b1[px + __popc(x & lt)] = cx;
      pm += __popc(m);
      px += __popc(x);
    }
    __syncwarp();
    // next chunk's gathers and the chunk after's indices in flight during the fold
#pragma unroll
    for (int h = 0; h < H; ++h) {
      ci[h] = ci2[h];
      a[h]  = a2[h];
    }
#pragma unroll
    for (int h = 0; h < H; ++h) bd[h] = ci[h] != -1 ? S.bounds[ci[h] & ~kIntBit] : make_double2(0.0, 0.0);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int e2 = base + 2 * kTile + h * 32 + lane;
      ci2[h]       = e2 < e1 ? __ldg(P.row_ci + rs + e2) : -1;
      a2[h]        = e2 < e1 ? __ldg(P.row_val + rs + e2) : 0.0;
    }
    if (lane < 2) acc = fold_seq(lane ? c.w.b1 : c.w.b0, lane ? px : pm, acc);
    __syncwarp();
  }
  if (cand) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      gtw = fmax(gtw, __shfl_xor_sync(FULL, gtw, o));
      gpm = fmax(gpm, __shfl_xor_sync(FULL, gpm, o));
    }
  }
  imn            = warp_sum(imn);
  imx            = warp_sum(imx);
  double smn     = __shfl_sync(FULL, acc, 0);
  double smx     = __shfl_sync(FULL, acc, 1);
  fold_finish(c, k, L, seg, smn, smx, imn, imx, gtw, gpm, cand, stamp);
}

// F2a (heavy rows): contributions of piece p (kPiece entries) of row k, with the per-128-chunk
// aggregates. The non-zero min / max contributions are compacted in entry order into the piece's
// slots of the two contribution streams (gmin / gmax at off + e0, counts in pcnt[p]): the segment
// fold then runs its chains over dense streams (the compaction off its critical path; see
// tools/microbench/mb_fold.cu: 139 -> 81 us per 16384-entry segment). The piece is published with
// this round's stamp.
__device__ void heavy_piece(Ctx& c, int pi, unsigned stamp)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int2 tk       = P.piece_task[pi];
  // (dirty-filtered rounds call only the pieces holding a variable changed last round: the others'
  // contributions, chunk aggregates and checkpoints are current)
  const int k = tk.x, rs = __ldg(P.row_start + k), L = __ldg(P.row_start + k + 1) - rs;
  const int off = __ldg(P.long_off + k);
  const int e0 = tk.y * kPiece, e1 = min(L, e0 + kPiece);
  double* gmn = S.gmin + off + e0;
  double* gmx = S.gmax + off + e0;
  const unsigned lt = lanemask_lt();
  int pm = 0, px = 0;
  PieceAgg ag{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0, 0};  // this lane's part of the piece aggregates
  // software pipeline over the piece's chunks: chunk j+1's bound gathers and chunk j+2's index /
  // value loads are in flight while chunk j is evaluated
  int ci[kEPL], ci2[kEPL];
  double a[kEPL], a2[kEPL];
  double2 bd[kEPL];
  auto load = [&](int j0, int (&ci_)[kEPL], double (&a_)[kEPL]) {
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const int e = j0 + h * 32 + c.lane;
      ci_[h]      = e < e1 ? __ldg(P.row_ci + rs + e) : -1;
      a_[h]       = e < e1 ? __ldg(P.row_val + rs + e) : 0.0;
    }
  };
  load(e0, ci, a);
  load(e0 + kTile, ci2, a2);
#pragma unroll
  for (int h = 0; h < kEPL; ++h) bd[h] = ci[h] != -1 ? S.bounds[ci[h] & ~kIntBit] : make_double2(0.0, 0.0);
  for (int j0 = e0; j0 < e1; j0 += kTile) {
    double cmv[kEPL], cxv[kEPL];
    int imn = 0, imx = 0;
    double gtw = 0.0, gpm = 0.0;
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      double cm = 0.0, cx = 0.0;
      if (ci[h] != -1) {
        int i1, i2;
        contrib(a[h], bd[h].x, bd[h].y, cm, cx, i1, i2);
        imn += i1;
        imx += i2;
        double tw, pw;
        entry_reach(a[h], bd[h].x, bd[h].y, ci[h] < 0, tw, pw);
        gtw = fmax(gtw, tw);
        gpm = fmax(gpm, pw);
      }
      cmv[h] = cm;
      cxv[h] = cx;
    }
    // next chunk: its gathers (indices loaded one chunk ago) and the loads of the one after
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      ci[h] = ci2[h];
      a[h]  = a2[h];
      bd[h] = ci[h] != -1 ? S.bounds[ci[h] & ~kIntBit] : make_double2(0.0, 0.0);
    }
    load(j0 + 2 * kTile, ci2, a2);
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const double cm = cmv[h], cx = cxv[h];
      ag.smin = __dadd_rn(ag.smin, cm);
      ag.amin = __dadd_rn(ag.amin, fabs(cm));
      ag.smax = __dadd_rn(ag.smax, cx);
      ag.amax = __dadd_rn(ag.amax, fabs(cx));
      // zero contributions are skipped: exact, the running sums are never -0.0
      const unsigned m = __ballot_sync(FULL, cm != 0.0);
      const unsigned x = __ballot_sync(FULL, cx != 0.0);
      if (cm != 0.0) gmn[pm + __popc(m & lt)] = cm;
      if (cx != 0.0) gmx[px + __popc(x & lt)] = cx;
      pm += __popc(m);
      px += __popc(x);
    }
    imn = warp_sum(imn);
    imx = warp_sum(imx);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      gtw = fmax(gtw, __shfl_xor_sync(FULL, gtw, o));
      gpm = fmax(gpm, __shfl_xor_sync(FULL, gpm, o));
    }
    if (c.lane == 0) {
      ChunkInfo ci_{gtw, gpm, imn, imx};
      S.cinfo[(off + j0) / kTile] = ci_;
    }
    ag.gtw = fmax(ag.gtw, gtw);  // (warp-uniform after the reductions above)
    ag.gpm = fmax(ag.gpm, gpm);
    ag.imn += imn;
    ag.imx += imx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    ag.smin = __dadd_rn(ag.smin, __shfl_xor_sync(FULL, ag.smin, o));
    ag.amin = __dadd_rn(ag.amin, __shfl_xor_sync(FULL, ag.amin, o));
    ag.smax = __dadd_rn(ag.smax, __shfl_xor_sync(FULL, ag.smax, o));
    ag.amax = __dadd_rn(ag.amax, __shfl_xor_sync(FULL, ag.amax, o));
  }
  __syncwarp();
  if (c.lane == 0) {
    S.pagg[pi] = ag;
    S.pcnt[pi] = make_int2(pm, px);
    __threadfence();
    atomicExch(S.pstamp + pi, stamp);
  }
}

// F2b (heavy rows): one 16384-entry segment. Waits for the segment's pieces, then runs the
// reference's sequential min / max sums (lanes 0 / 1) over the pieces' compacted contribution
// streams in chunks of kFoldVals values: every lane stages chunk t + 1 into shared memory (the
// other buffer) and has chunk t + 2's loads in flight while the chains fold chunk t.
constexpr int kFoldVals = 96;  // 4 buffers fill the 3 KB row-task staging region (kRowsWarpBytes)
static_assert(kFoldVals % 32 == 0 && 4 * kFoldVals * 8 <= 3072, "fold staging buffers");
// Fold modes: exact (frontier rounds, activity calls), lazy (full / dirty-filtered rounds: a row
// certified quiet skips its chains and keeps a stale record), refresh (stale rows only, chains
// from the first piece changed since their segment's last exact fold).
enum { kFoldExact = 0, kFoldLazy = 1, kFoldRefresh = 2 };

// Quietness certificate of a heavy row without its sequential sums: from the pieces'
// any-order sums S and absolute sums A of the min / max contributions, the reference's segmented
// sequential sum lies within eps*A of S (both err by at most L u sum|x|; eps = 8 (L + 1024) u also
// covers the bound's own rounding), so the row-level gate (entry_quiet with the row's reach
// maxima) evaluated in directed rounding over that interval proves that no entry of the row can
// publish a candidate -- exactly what the gate with the exact activity would prove, or more.
// Waits for this round's recomputed pieces of the row. Infinite contributors: only counts of 0
// (side usable with finite parts) or >= 2 (side unusable) are certified.
__device__ bool heavy_row_quiet(Ctx& c, int k, int L, unsigned stamp, unsigned ds)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int lane = c.lane;
  const int hp = __ldg(P.hpiece + k), npr = (L + kPiece - 1) / kPiece;
  for (int q = lane; q < npr; q += 32)
    if (ds == 0 || __ldcg(S.piece_dirty + hp + q) == ds)
      while (ldv(S.pstamp + hp + q) != stamp) __nanosleep(100);
  __syncwarp();
  __threadfence();
  double sm = 0.0, am = 0.0, sx = 0.0, ax = 0.0, gtw = 0.0, gpm = 0.0;
  int imn = 0, imx = 0;
  for (int q = lane; q < npr; q += 32) {
    const PieceAgg* a = S.pagg + hp + q;
    sm = __dadd_rn(sm, __ldcg(&a->smin));
    am = __dadd_rn(am, __ldcg(&a->amin));
    sx = __dadd_rn(sx, __ldcg(&a->smax));
    ax = __dadd_rn(ax, __ldcg(&a->amax));
    gtw = fmax(gtw, __ldcg(&a->gtw));
    gpm = fmax(gpm, __ldcg(&a->gpm));
    imn += __ldcg(&a->imn);
    imx += __ldcg(&a->imx);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sm  = __dadd_rn(sm, __shfl_xor_sync(FULL, sm, o));
    am  = __dadd_rn(am, __shfl_xor_sync(FULL, am, o));
    sx  = __dadd_rn(sx, __shfl_xor_sync(FULL, sx, o));
    ax  = __dadd_rn(ax, __shfl_xor_sync(FULL, ax, o));
    gtw = fmax(gtw, __shfl_xor_sync(FULL, gtw, o));
    gpm = fmax(gpm, __shfl_xor_sync(FULL, gpm, o));
    imn += __shfl_xor_sync(FULL, imn, o);
    imx += __shfl_xor_sync(FULL, imx, o);
  }
  const double2 cb  = __ldg(&P.cons[k]);
  const double g = cb.y, h = cb.x;
  const double eps  = (double)(L + 1024) * 0x1p-50;
  const double rtw  = __dmul_ru(gtw, 1.0 + 1e-12);
  bool qg = !isfinite(g) || imn >= 2;
  if (!qg && imn == 0) {  // side g: slack g - act_min over act_min in [lo, hi]
    const double e  = __dmul_ru(eps, am);
    const double hi = __dadd_ru(sm, e), lo = __dsub_rd(sm, e);
    const double mg = __dmul_ru(1e-12, __dadd_ru(__dadd_ru(fabs(g), fmax(fabs(lo), fabs(hi))), gpm));
    qg = __dsub_rd(g, hi) >= __dadd_ru(__dadd_ru(rtw, mg), 1e-300);
  }
  bool qh = !isfinite(h) || imx >= 2;
  if (!qh && imx == 0) {  // side h: slack act_max - h
    const double e  = __dmul_ru(eps, ax);
    const double hi = __dadd_ru(sx, e), lo = __dsub_rd(sx, e);
    const double mg = __dmul_ru(1e-12, __dadd_ru(__dadd_ru(fabs(h), fmax(fabs(lo), fabs(hi))), gpm));
    qh = __dsub_rd(lo, h) >= __dadd_ru(__dadd_ru(rtw, mg), 1e-300);
  }
  return qg && qh;
}

// True when a piece of row k changed after its segment's last exact fold (stale record).
__device__ bool heavy_row_stale(Ctx& c, int k, int L)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int hp = __ldg(P.hpiece + k), npr = (L + kPiece - 1) / kPiece;
  constexpr int kSegPieces = kSumSegment / kPiece;
  bool st = false;
  for (int q = c.lane; q < npr; q += 32)
    st = st || ldv(S.pstamp + hp + q) > ldv(S.sfold + hp + q / kSegPieces * kSegPieces);
  return __any_sync(FULL, st);
}

__device__ void heavy_fold(Ctx& c, int k, int seg, bool cand, unsigned stamp, unsigned ds, int mode)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int lane      = c.lane;
  const int L   = __ldg(P.row_start + k + 1) - __ldg(P.row_start + k);
  const int off = __ldg(P.long_off + k);
  const int e0 = seg * kSumSegment, e1 = min(L, e0 + kSumSegment);
  const int p0 = __ldg(P.hpiece + k) + e0 / kPiece, np = (e1 - e0 + kPiece - 1) / kPiece;
  if (mode == kFoldRefresh) {
    if (!heavy_row_stale(c, k, L)) return;
  } else if (mode == kFoldLazy && cand && heavy_row_quiet(c, k, L, stamp, ds)) {
    // every segment's warp reaches the same verdict: no chain, no record, no candidates; the
    // record is refreshed before anything reads it (phase_refresh)
    if (seg == 0 && lane == 0) {
      if (L > kCandSplit) {
        S.rquiet[k] = 1;
        __threadfence();
        atomicExch(S.ready + k, stamp);
      }
      S.ctl->stale = 1;
    }
    return;
  }
  if (mode != kFoldRefresh) {
    // this round's recomputed pieces of the segment (dirty-filtered round: the marked ones)
    const bool mine = lane < np && (ds == 0 || __ldcg(S.piece_dirty + p0 + lane) == ds);
    if (mine)
      while (ldv(S.pstamp + p0 + lane) != stamp) __nanosleep(100);
    __syncwarp();
    __threadfence();
  }
  // the sum is replayed from the checkpoint of the first piece that changed after the segment's
  // last exact fold (the prefix before it is unchanged); a segment without one keeps its partial
  const unsigned fs = ldv(S.sfold + p0);
  unsigned dm = __ballot_sync(FULL, lane < np && ldv(S.pstamp + p0 + lane) > fs);
  const int sb = __ldg(P.seg_base + k);
  if (dm == 0 && sb < 0) dm = 1u;  // (single-segment rows always have a changed piece when folded)
  if (dm == 0) {
    double smn = 0.0, smx = 0.0, gtw = 0.0, gpm = 0.0;
    int imn = 0, imx = 0;
    if (lane == 0) {
      const SegPart* sq = S.seg_part + sb + seg;
      smn = __ldcg(&sq->min);
      smx = __ldcg(&sq->max);
      imn = __ldcg(&sq->nmin);
      imx = __ldcg(&sq->nmax);
      gtw = __ldcg(&sq->tmax);
      gpm = __ldcg(&sq->pmax);
    }
    fold_finish(c, k, L, seg, smn, smx, imn, imx, gtw, gpm, cand, stamp);
    return;
  }
  const int pf             = __ffs(dm) - 1;  // first changed piece
  const long long c_stream = DBG_ON(S) ? clock64() : 0;
  double acc = 0.0, gtw = 0.0, gpm = 0.0;
  if (pf > 0 && lane < 2) acc = __ldcg(reinterpret_cast<const double*>(S.ckpt + p0 + pf) + lane);
  int imn = 0, imx = 0;
  // chunk aggregates of the segment: lanes read them strided (off the fold's critical path)
  for (int q = (off + e0) / kTile + lane; q < (off + e1 + kTile - 1) / kTile; q += 32) {
    const ChunkInfo* ch = S.cinfo + q;
    imn += __ldcg(&ch->imn);
    imx += __ldcg(&ch->imx);
    gtw = fmax(gtw, __ldcg(&ch->gtw));
    gpm = fmax(gpm, __ldcg(&ch->gpm));
  }
  // the chunk list from piece pf on (kFoldVals values per chunk and stream): lane q holds piece q's
  // counts and its chunks' inclusive prefix (at least one chunk per piece, possibly empty: its
  // checkpoint is written when it starts)
  const int2 cnt = lane < np ? __ldcg(S.pcnt + p0 + lane) : make_int2(0, 0);
  const int nck  = lane >= pf && lane < np ? max(1, (max(cnt.x, cnt.y) + kFoldVals - 1) / kFoldVals) : 0;
  const int incl = warp_incl_scan(nck, lane);
  const int T    = __shfl_sync(FULL, incl, 31);
  const double* gmn = S.gmin + off + e0;
  const double* gmx = S.gmax + off + e0;
  // chunk t -> piece q, chunk cc of the piece, and this chunk's value counts (warp-uniform)
  auto locate = [&](int t, int& q, int& cc, int& nm, int& nx) {
    q  = __popc(__ballot_sync(FULL, incl <= t));
    cc = t - (__shfl_sync(FULL, incl, q) - __shfl_sync(FULL, nck, q));
    nm = min(kFoldVals, max(0, __shfl_sync(FULL, cnt.x, q) - cc * kFoldVals));
    nx = min(kFoldVals, max(0, __shfl_sync(FULL, cnt.y, q) - cc * kFoldVals));
  };
  constexpr int V = kFoldVals / 32;
  double rm[V], rx[V];
  auto fetch = [&](int t) {  // chunk t's values into registers (zeros past the counts / the list)
    int q = 0, cc = 0, nm = 0, nx = 0;
    if (t < T) locate(t, q, cc, nm, nx);
    const int base = q * kPiece + cc * kFoldVals;
#pragma unroll
    for (int h = 0; h < V; ++h) {
      const int j = h * 32 + lane;
      rm[h]       = j < nm ? __ldcg(gmn + base + j) : 0.0;
      rx[h]       = j < nx ? __ldcg(gmx + base + j) : 0.0;
    }
  };
  // two buffers per stream in the warp's staging region (b0 / b1 are contiguous)
  double* buf = c.w.b0;
  auto stage = [&](int bi) {
#pragma unroll
    for (int h = 0; h < V; ++h) {
      buf[bi * kFoldVals + h * 32 + lane]                 = rm[h];
      buf[(2 + bi) * kFoldVals + h * 32 + lane]           = rx[h];
    }
  };
  fetch(0);
  stage(0);
  fetch(1);
  __syncwarp();
  for (int t = 0; t < T; ++t) {
    const int bi = t & 1;
    stage(bi ^ 1);  // chunk t + 1 (its buffers were last read in iteration t - 1)
    int q, cc, nm, nx;
    locate(t, q, cc, nm, nx);
    fetch(t + 2);
    if (lane < 2) {
      if (cc == 0) reinterpret_cast<double*>(S.ckpt + p0 + q)[lane] = acc;  // the sums before piece q
      acc = fold_seq(buf + (2 * lane + bi) * kFoldVals, lane ? nx : nm, acc);
    }
    __syncwarp();
  }
  imn = warp_sum(imn);
  imx = warp_sum(imx);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    gtw = fmax(gtw, __shfl_xor_sync(FULL, gtw, o));
    gpm = fmax(gpm, __shfl_xor_sync(FULL, gpm, o));
  }
  const double smn = __shfl_sync(FULL, acc, 0);
  const double smx = __shfl_sync(FULL, acc, 1);
  if (lane == 0) S.sfold[p0] = stamp;  // the segment's partial and checkpoints are exact as of now
  dbg_task(c, 3, c_stream);  // streaming part of a heavy segment (after its pieces are ready)
  fold_finish(c, k, L, seg, smn, smx, imn, imx, gtw, gpm, cand, stamp);
}

// Four medium rows (kPackNnz < nnz <= kHeavyFold, single segment) per warp, eight lanes per row:
// each group streams its row in 32-entry chunks (next chunk's indices in flight), compacts the
// non-zero contributions into its own shared-memory slice, and its lanes 0/1 run the row's
// sequential min/max sums -- the four rows' chains advance in the same instructions. Then the
// candidates of the non-quiet rows.
#ifndef BP_WARP_ROW_MIN
#define BP_WARP_ROW_MIN 256  // C2: off 5.61, 128 5.60, 256 5.60, 512 5.60 ms (late rounds 63-130 -> 57-65 us)
#endif
constexpr int kWarpRowMin = BP_WARP_ROW_MIN;  // medium rows above: a warp per row (group_fold)

__device__ void group_fold(Ctx& c, int t0, int nt, bool cand, unsigned ds = 0)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int lane = c.lane, g = lane >> 3, gl = lane & 7;
  const unsigned gmask = 0xFFu << (8 * g);
  const int k          = g < nt ? __ldg(&P.fold_task[t0 + g].x) : -1;
  // dirty-filtered round: clean rows of the group stay idle (see sell_slice)
  const bool act = k >= 0 && (ds == 0 || __ldcg(S.row_flag + k) == (unsigned char)ds);
  int rs = 0, L = 0;
  if (act) {
    rs = __ldg(P.row_start + k);
    L  = __ldg(P.row_start + k + 1) - rs;
  }
  int Lmax = L;
#pragma unroll
  for (int o = 16; o; o >>= 1) Lmax = max(Lmax, __shfl_xor_sync(FULL, Lmax, o));
  if (Lmax > kWarpRowMin) {
    // long medium rows (the group's rows have similar lengths): one after another with the whole
    // warp (128-entry chunks, two in flight) -- 4x fewer dependent load steps per row than 8 lanes
    const unsigned am = __ballot_sync(FULL, act && gl == 0);
    for (int q = 0; q < 4; ++q) {
      const int kq = __shfl_sync(FULL, k, 8 * q);
      if ((am >> (8 * q)) & 1u) long_fold(c, kq, 0, cand, 0u);
    }
    return;
  }
  double* gb0 = c.w.b0 + 32 * g;  // group slices of the staging buffers (<= 32 per chunk)
  double* gb1 = c.w.b1 + 32 * g;
  int ci[4], cn[4];
  double a[4], an[4];
  double2 bd[4];
  auto load = [&](int base, int* ci_, double* a_) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int e = base + h * 8 + gl;
      ci_[h]      = e < L ? __ldg(P.row_ci + rs + e) : -1;
      a_[h]       = e < L ? __ldg(P.row_val + rs + e) : 0.0;
    }
  };
  auto gather = [&]() {
#pragma unroll
    for (int h = 0; h < 4; ++h) bd[h] = ci[h] != -1 ? S.bounds[ci[h] & ~kIntBit] : make_double2(0.0, 0.0);
  };
  load(0, ci, a);
  gather();
  load(32, cn, an);
  const unsigned lt = lanemask_lt() & gmask;
  double acc = 0.0, gtw = 0.0, gpm = 0.0;
  int imn = 0, imx = 0;
  for (int base = 0; base < Lmax; base += 32) {
    int pm = 0, px = 0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      double cm = 0.0, cx = 0.0;
      if (ci[h] != -1) {
        int i1, i2;
        contrib(a[h], bd[h].x, bd[h].y, cm, cx, i1, i2);
        imn += i1;
        imx += i2;
        if (cand && kRowGate) {
          double tw, pw;
          entry_reach(a[h], bd[h].x, bd[h].y, ci[h] < 0, tw, pw);
          gtw = fmax(gtw, tw);
          gpm = fmax(gpm, pw);
        }
      }
      const unsigned m = __ballot_sync(FULL, cm != 0.0) & gmask;
      const unsigned x = __ballot_sync(FULL, cx != 0.0) & gmask;
      if (cm != 0.0) gb0[pm + __popc(m & lt)] = cm;
      if (cx != 0.0) gb1[px + __popc(x & lt)] = cx;
      pm += __popc(m);
      px += __popc(x);
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      ci[h] = cn[h];
      a[h]  = an[h];
    }
    gather();
    load(base + 64, cn, an);
    if (gl < 2 && act) acc = fold_seq(gl ? gb1 : gb0, gl ? px : pm, acc);
    __syncwarp();
  }
#pragma unroll
  for (int o = 4; o; o >>= 1) {
    imn += __shfl_xor_sync(FULL, imn, o);
    imx += __shfl_xor_sync(FULL, imx, o);
    gtw = fmax(gtw, __shfl_xor_sync(FULL, gtw, o));
    gpm = fmax(gpm, __shfl_xor_sync(FULL, gpm, o));
  }
  const double smn = __shfl_sync(FULL, acc, 8 * g);
  const double smx = __shfl_sync(FULL, acc, 8 * g + 1);
  double2 cb       = make_double2(0.0, 0.0);
  if (act) {
    cb = __ldg(&P.cons[k]);
    if (gl == 0) write_rec(P, S, k, smn, smx, imn, imx);
  }
  if (!cand) return;
  const bool quiet = !act || (kRowGate && entry_quiet(gtw, gpm, smn, imn, smx, imx, cb.y, cb.x));
  if (__all_sync(FULL, quiet)) return;
  for (int base = 0; base < Lmax; base += 32) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int e = base + h * 8 + gl;
      ci[h]       = !quiet && e < L ? __ldg(P.row_ci + rs + e) : -1;
      a[h]        = !quiet && e < L ? __ldg(P.row_val + rs + e) : 0.0;
    }
    gather();
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      if (ci[h] == -1) continue;
      double tw, pw;
      entry_reach(a[h], bd[h].x, bd[h].y, ci[h] < 0, tw, pw);
      if (entry_quiet(tw, pw, smn, imn, smx, imx, cb.y, cb.x)) continue;
      emit_cand(S, c.touch, ci[h], a[h], bd[h].x, bd[h].y, smn, imn, smx, imx, cb.y, cb.x, k);
    }
  }
}

// F2 tail: candidate piece p of a row with > kCandSplit entries, once its activity is published.
__device__ void long_cand_piece(Ctx& c, int k, int p, unsigned stamp, unsigned ds = 0)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  if (!row_live(S, k, ds)) return;  // clean row: no activity published this round
  if (c.lane == 0)
    while (ldv(S.ready + k) != stamp) __nanosleep(200);
  __syncwarp();
  __threadfence();
  if (*(const volatile unsigned char*)(S.rquiet + k)) return;  // the whole row is quiet
  const RowRec r = ld_rec_cg(S.rec + k);
  double mnf = r.min, mxf = r.max;
  const int nmn = is_box(r.min) ? box_value(r.min) : 0;
  const int nmx = is_box(r.max) ? box_value(r.max) : 0;
  if (nmn | nmx) {
    const double2 x = __ldcg(S.aux + k);
    if (nmn) mnf = x.x;
    if (nmx) mxf = x.y;
  }
  const int L = __ldg(P.row_start + k + 1) - __ldg(P.row_start + k);
  long_candidates(c, k, p * kPiece, min(L, (p + 1) * kPiece), mnf, nmn, mxf, nmx, r.g, r.h);
}

// One SELL-32 slice (32 rows of similar length <= kPackNnz, entries column-interleaved: entry j
// of lane i at base + 32 j + i): thread per row. Each lane streams its row in order with 4
// entries' loads and bound gathers in flight, runs the reference's sequential min/max sums in
// registers (rows here are single-segment), writes the row record, then -- with `cand`, unless
// every row of the slice is provably quiet -- streams the row again for the candidates.
#ifndef BP_SELL_UNROLL
#define BP_SELL_UNROLL 4
#endif
constexpr int kSellUnroll = BP_SELL_UNROLL;  // entries per lane in flight
// The thread-per-row SELL evaluation of row k (-1: idle lane) whose entries are at ciq / aq + 32 j
// for j < Lm (padding entries are -1), the loop running Lw >= Lm steps (warp-uniform).
__device__ __forceinline__ void sell_core(Ctx& c, int k, const int* ciq, const double* aq, int Lm, int Lw, bool cand)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  double smn = 0.0, smx = 0.0, gtw = 0.0, gpm = 0.0;
  int imn = 0, imx = 0;
  constexpr int U = kSellUnroll;
  for (int j = 0; j < Lw; j += U) {
    int ci[U];
    double a[U];
    double2 bd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ci[u] = k >= 0 && j + u < Lm ? __ldg(ciq + 32 * (j + u)) : -1;
      a[u]  = k >= 0 && j + u < Lm ? __ldg(aq + 32 * (j + u)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) bd[u] = ci[u] != -1 ? S.bounds[ci[u] & ~kIntBit] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (ci[u] == -1) continue;  // padding only follows a row's last entry
      double cm, cx;
      int i1, i2;
      contrib(a[u], bd[u].x, bd[u].y, cm, cx, i1, i2);
      smn = __dadd_rn(smn, cm);
      smx = __dadd_rn(smx, cx);
      imn += i1;
      imx += i2;
      if (cand && kRowGate) {
        double tw, pw;
        entry_reach(a[u], bd[u].x, bd[u].y, ci[u] < 0, tw, pw);
        gtw = fmax(gtw, tw);
        gpm = fmax(gpm, pw);
      }
    }
  }
  double2 cb = make_double2(0.0, 0.0);
  if (k >= 0) {
    cb = __ldg(&P.cons[k]);
    RowRec r;
    r.min = imn ? box_count(imn) : smn;
    r.max = imx ? box_count(imx) : smx;
    r.g   = cb.y;
    r.h   = cb.x;
    st_rec(S.rec + k, r);
    if (imn | imx) S.aux[k] = make_double2(smn, smx);
  }
  if (!cand) return;
  const bool quiet = k < 0 || (kRowGate && entry_quiet(gtw, gpm, smn, imn, smx, imx, cb.y, cb.x));
  if (DBG_ON(S)) {  // gate statistics (BP_DEBUG=1, built with -DBP_DBG_STATS=1)
    const unsigned nr = __popc(__ballot_sync(FULL, k >= 0)), nq = __popc(__ballot_sync(FULL, !quiet));
    if (c.lane == 0) {
      atomicAdd(S.dbg + 16, (unsigned long long)nr);
      atomicAdd(S.dbg + 17, (unsigned long long)nq);
    }
  }
  if (__all_sync(FULL, quiet)) return;
  for (int j = 0; j < Lw; j += U) {
    int ci[U];
    double a[U];
    double2 bd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ci[u] = !quiet && j + u < Lm ? __ldg(ciq + 32 * (j + u)) : -1;
      a[u]  = !quiet && j + u < Lm ? __ldg(aq + 32 * (j + u)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) bd[u] = ci[u] != -1 ? S.bounds[ci[u] & ~kIntBit] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (ci[u] == -1) continue;
      double tw, pw;
      entry_reach(a[u], bd[u].x, bd[u].y, ci[u] < 0, tw, pw);
      if (DBG_ON(S)) atomicAdd(S.dbg + 18, 1ull);
      if (entry_quiet(tw, pw, smn, imn, smx, imx, cb.y, cb.x)) continue;
      if (DBG_ON(S)) atomicAdd(S.dbg + 19, 1ull);
      emit_cand(S, c.touch, ci[u], a[u], bd[u].x, bd[u].y, smn, imn, smx, imx, cb.y, cb.x, k);
    }
  }
}

__device__ void sell_slice(Ctx& c, int sl, bool cand, unsigned ds = 0)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  // dirty-filtered round: the slice is dirty; its clean rows (byte flag != the round's mark; a stale
  // byte matching by wrap-around only recomputes a clean row, which is exact) are idle lanes
  int k = __ldg(P.srow + 32 * sl + c.lane);
  if (ds != 0 && k >= 0 && __ldcg(S.row_flag + k) != (unsigned char)ds) k = -1;
  const int b0 = __ldg(P.sr_tile + sl), b1 = __ldg(P.sr_tile + sl + 1);
  const int Lm = (b1 - b0) >> 5;
  sell_core(c, k, P.sr_ci + b0 + c.lane, P.sr_val + b0 + c.lane, Lm, Lm, cand);
}

// Dirty-filtered round with few dirty short rows: 32 listed rows per warp, each lane reading its
// row where it lies in its SELL slice (sell_pos) -- no idle lanes, at the price of uncoalesced
// index / value loads.
__device__ void sell_rows(Ctx& c, int base, int n, bool cand)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int i = base + c.lane;
  int k = -1, b = 0, Lm = 0;
  if (i < n) {
    k             = __ldcg(S.df_rows + i);
    const int pos = __ldg(P.sell_pos + k);
    const int b0 = __ldg(P.sr_tile + (pos >> 5)), b1 = __ldg(P.sr_tile + (pos >> 5) + 1);
    Lm            = (b1 - b0) >> 5;
    b             = b0 + (pos & 31);
  }
  int Lw = Lm;
#pragma unroll
  for (int o = 16; o; o >>= 1) Lw = max(Lw, __shfl_xor_sync(FULL, Lw, o));
  sell_core(c, k, P.sr_ci + b, P.sr_val + b, Lm, Lw, cand);
}

// Listed short rows (frontier rounds): flattened 128-entry windows, each lane folds its row.
__device__ void short_list_tile(Ctx& c, const int* ids, int base, int n)
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

#ifndef BP_SELL_ROWS_PER_SLICE
#define BP_SELL_ROWS_PER_SLICE 16
#endif
constexpr int kSellRowsPerSlice = BP_SELL_ROWS_PER_SLICE;  // listed rows below this many per dirty slice

#ifndef BP_PIECE_STEP
#define BP_PIECE_STEP 1
#endif
#ifndef BP_GROUP_STEP
#define BP_GROUP_STEP 1
#endif
// heavy pieces / groups of four medium rows per cursor claim in full rounds (measured on C2: 4
// pieces 5.67 -> 5.80 ms, 4 groups -> 6.95 ms: the medium rows balance only at one group a claim)
constexpr int kPieceStep = BP_PIECE_STEP;
constexpr int kGroupStep = BP_GROUP_STEP;
// SELL slices (k_rows_sell) statically assigned: 6.31 -> 5.55 ms on C2 against one shared cursor
// (every claim an atomic on one address, 7k claims per round)
#ifndef BP_MULTI_CURSORS
#define BP_MULTI_CURSORS 8
#endif
constexpr int kMultiCursors = BP_MULTI_CURSORS;  // medium-row group cursors in full rounds (1: one)
static_assert(kMultiCursors <= kMaxMultiCursors, "Ctl::mcur holds kMaxMultiCursors per parity");
#ifndef BP_STATIC_SELL
#define BP_STATIC_SELL 1
#endif
constexpr bool kStaticSell = BP_STATIC_SELL != 0;

// SELL slices of a full round, longest first: slices of rows > 32 entries one per fetch, the rest
// four per fetch (one cursor shared by the whole grid is the contended resource).
__device__ void phase_sell(Ctx& c, ParCtl* pc, bool cand, unsigned ds = 0)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int ns = P.n_srtile, nsl = P.n_srow_long;
  if (ds != 0) {  // dirty-filtered round
    const int nr = ldv(&S.ctl->df_cnt[3]), nd = ldv(&S.ctl->df_cnt[0]);
    const int gw = blockIdx.x * kWarps + c.warp, nw = gridDim.x * kWarps;
    if (nr <= kSellRowsPerSlice * nd) {  // few dirty rows per dirty slice: the listed rows, 32 per warp
      for (int t = 32 * gw; t < nr; t += 32 * nw) sell_rows(c, t, nr, cand);
      return;
    }
    // else the engine's list of dirty slices (clean lanes idle)
    for (int q = gw; q < nd; q += nw) sell_slice(c, __ldcg(S.df_slice + q), cand, ds);
    return;
  }
  if (kStaticSell) {
    // slices are independent (no task waits on another): a static grid-stride assignment, no
    // shared cursor; the slices are sorted by length, so every warp gets one of each length class
    const int gw = blockIdx.x * kWarps + c.warp, nw = gridDim.x * kWarps;
    for (int q = gw; q < ns; q += nw) sell_slice(c, q, cand);
    return;
  }
  for (Prefetch it_t(c, &pc->cur_s, 1, nsl, true); it_t.t < nsl; it_t.advance()) {
    const long long c0 = DBG_ON(S) ? clock64() : 0;
    sell_slice(c, it_t.t, cand);
    dbg_task(c, 1, c0);
  }
  for (Prefetch it_t(c, &pc->cur_a, 4, ns - nsl, true); nsl + it_t.t < ns; it_t.advance()) {
    const long long c0 = DBG_ON(S) ? clock64() : 0;
    for (int q = nsl + it_t.t; q < min(ns, nsl + it_t.t + 4); ++q) sell_slice(c, q, cand);
    dbg_task(c, 1, c0);
  }
}

// Phase 2 (F2 / P2): activities of all rows (full) or the dirty ones; `cand` fuses tightening.
// pieces_here = false: the candidate pieces of rows above kCandSplit are left to a following
// k_cand_pieces launch (no warp spins on an unfinished row's activity).
__device__ void phase_rows(Ctx& c, ParCtl* pc, int par, bool full, bool cand, unsigned stamp,
                           bool pieces_here = true, bool sell_here = true, unsigned ds = 0)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int nf        = full ? P.n_fold : ldv(&pc->n_dfold);
  const int2* folds   = full ? P.fold_task : S.dfold[par];
  if (full) {
    // long folds first (longest chains start first), then the SELL slices (4 per fetch: one
    // cursor shared by the whole grid is the contended resource), then candidate pieces of rows
    // above kCandSplit (they wait for their row's fold, all of which have been fetched by then)
    // heavy rows' contribution pieces first: the segment folds that wait for them are fetched
    // only after every piece has been fetched by a running warp (no deadlock)
    if (ds == 0) {  // (pieces from 8 interleaved cursors like the groups below: 5.50 -> 6.01 ms on C2
                    // -- a row's pieces then finish scattered in time and its folds wait longer)
      for (Prefetch it_t(c, &pc->cur_p, kPieceStep, P.n_piece); it_t.t < P.n_piece; it_t.advance())
        for (int q = it_t.t; q < min(P.n_piece, it_t.t + kPieceStep); ++q) heavy_piece(c, q, stamp);
    } else {  // dirty-filtered round: the engine's list of dirty pieces
      const int nd = ldv(&S.ctl->df_cnt[2]);
      for (Prefetch it_t(c, &pc->cur_p, 1, nd); it_t.t < nd; it_t.advance()) heavy_piece(c, __ldcg(S.df_piece + it_t.t), stamp);
    }
    const int nfh = P.n_fold_heavy;
    for (Prefetch it_t(c, &pc->cur_b, 1, nfh); it_t.t < nfh; it_t.advance()) {
      const long long c0 = DBG_ON(S) ? clock64() : 0;
      const int2 tk      = folds[it_t.t];
      if (row_live(S, tk.x, ds)) heavy_fold(c, tk.x, tk.y, cand, stamp, ds, kFoldLazy);
      dbg_task(c, 0, c0);
    }
    if (ds == 0 && kMultiCursors > 1) {
      // groups claimed one at a time (balance) from kMultiCursors interleaved sub-ranges, each with
      // its own cursor on its own line: a warp starts on sub-range (warp mod K) and moves on when
      // it is exhausted -- K times fewer atomics queue on any one address
      const int ng = (nf - nfh + 3) / 4;
      int* mc      = S.ctl->mcur + par * kMultiCursors * 32;
      int k        = (blockIdx.x * kWarps + c.warp) % kMultiCursors;
      for (int tried = 0; tried < kMultiCursors;) {
        int g = 0;
        if (c.lane == 0) g = atomicAdd(mc + 32 * k, 1);
        const int item = k + kMultiCursors * __shfl_sync(FULL, g, 0);
        if (item >= ng) {
          k = (k + 1) % kMultiCursors;
          ++tried;
          continue;
        }
        tried = 0;
        group_fold(c, nfh + 4 * item, min(4, nf - nfh - 4 * item), cand);
      }
    } else if (ds == 0) {
      for (Prefetch it_t(c, &pc->cur_g, 4 * kGroupStep, nf - nfh, true); nfh + it_t.t < nf; it_t.advance()) {
        const long long c0 = DBG_ON(S) ? clock64() : 0;
        for (int q = it_t.t; q < min(nf - nfh, it_t.t + 4 * kGroupStep); q += 4)
          group_fold(c, nfh + q, min(4, nf - nfh - q), cand);
        dbg_task(c, 4, c0);
      }
    } else {  // dirty-filtered round: the engine's list of dirty groups of four medium rows
      const int nd = ldv(&S.ctl->df_cnt[1]);
      for (Prefetch it_t(c, &pc->cur_g, 1, nd, true); it_t.t < nd; it_t.advance()) {
        const int t0 = 4 * __ldcg(S.df_group + it_t.t);
        group_fold(c, nfh + t0, min(4, nf - nfh - t0), cand, ds);
      }
    }
    if (sell_here) phase_sell(c, pc, cand, ds);
    const int nc = cand && pieces_here ? P.n_cpiece : 0;
    for (Prefetch it_t(c, &pc->cur_c, 1, nc); it_t.t < nc; it_t.advance()) {
      const long long c0 = DBG_ON(S) ? clock64() : 0;
      const int2 tk      = P.cpiece_task[it_t.t];
      long_cand_piece(c, tk.x, tk.y, stamp, ds);
      dbg_task(c, 2, c0);
    }
  } else {
    // dirty heavy rows: contribution pieces first (the folds waiting for them are fetched after)
    const int ndp = ldv(&pc->n_dpiece);
    for (Prefetch it_t(c, &pc->cur_p, 1, ndp); it_t.t < ndp; it_t.advance())
      heavy_piece(c, S.dpiece[par][it_t.t].x, stamp);
    for (Prefetch it_t(c, &pc->cur_b, 1, nf); it_t.t < nf; it_t.advance()) {
      const int2 tk = folds[it_t.t];
      if (__ldg(P.long_off + tk.x) >= 0) heavy_fold(c, tk.x, tk.y, false, stamp, 0, kFoldExact);
      else long_fold(c, tk.x, tk.y, false, stamp);
    }
    const int n = ldv(&pc->n_drow_s);
    for (Prefetch it_t(c, &pc->cur_c, 32, n); it_t.t < n; it_t.advance())
      short_list_tile(c, S.drow_s[par], it_t.t, n);
  }
}

// Exact records for the heavy rows a lazy full round left stale (certified quiet, chains skipped):
// every segment of such a row replays its sum from the first piece changed since its last exact
// fold (the pieces' streams are current). Run before anything reads the records: a frontier
// round's tightening, and the end of the call.
__device__ void phase_refresh(Ctx& c, unsigned stamp)
{
  const DevProblem& P = c.P;
  const int gw = blockIdx.x * kWarps + c.warp, nw = gridDim.x * kWarps;
  for (int t = gw; t < P.n_fold_heavy; t += nw) {
    const int2 tk = P.fold_task[t];
    heavy_fold(c, tk.x, tk.y, false, stamp, 0, kFoldRefresh);
  }
}

// ------------------------------------------------------------------ tightening

struct Tally {
  int crossed;
  int any_rows;
  unsigned long long colnnz;
  unsigned long long reach, hreach;  // Σ over changed vars of their light / heavy-row reach
  int nbuf;  // warp-uniform count of staged changed vars
};

// Appends the staged changed vars to the changed list and their columns, in kTile-entry chunks,
// to the row-expansion task list (no long serial chain in the frontier expansion).
__device__ __forceinline__ void flush_changed(Ctx& c, ParCtl* pc, Tally& t)
{
  if (t.nbuf == 0) return;
  int base = 0;
  if (c.lane == 0) base = atomicAdd(&pc->n_changed, t.nbuf);
  base = __shfl_sync(FULL, base, 0);
  __syncwarp();
  for (int j0 = 0; j0 < t.nbuf; j0 += 32) {
    const int j = j0 + c.lane;
    int i = -1, nch = 0;
    if (j < t.nbuf) {
      i                         = c.w.chg[j];
      c.S.changed[base + j]     = i;
      const int L               = __ldg(c.P.col_start + i + 1) - __ldg(c.P.col_start + i);
      nch                       = L > kTile ? (L + kTile - 1) / kTile : 0;
    }
    const int pos = warp_alloc(&pc->n_ctask, nch, c.lane);
    for (int q = 0; q < nch; ++q) c.S.ctask[pos + q] = make_int2(i, q);
  }
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
    t.reach += __ldg(c.P.reach + 2 * i);
    t.hreach += __ldg(c.P.reach + 2 * i + 1);
    if (nnz > 0) t.any_rows = 1;
  }
  if (ch) {
    if (t.nbuf + __popc(ch) > 64) flush_changed(c, pc, t);
    if (r > 0) c.w.chg[t.nbuf + __popc(ch & lanemask_lt())] = i;
    t.nbuf += __popc(ch);
    __syncwarp();
  }
}

__device__ void tally_flush_block(Ctx& c, ParCtl* pc, Tally& t)
{
  flush_changed(c, pc, t);
  const int cr = warp_sum(t.crossed);
  const int ar = __any_sync(FULL, t.any_rows);
  unsigned long long cn = t.colnnz, rh = t.reach, hh = t.hreach;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    rh += __shfl_xor_sync(FULL, rh, o);
    hh += __shfl_xor_sync(FULL, hh, o);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) cn += __shfl_xor_sync(FULL, cn, o);
  if (c.lane == 0) {
    if (cr) atomicAdd(&c.sm.blk_crossed, cr);
    if (ar) atomicOr(&c.sm.blk_any_rows, 1);
    if (cn) atomicAdd(&c.sm.blk_colnnz, cn);
    if (rh) atomicAdd(&c.sm.blk_reach, rh);
    if (hh) atomicAdd(&c.sm.blk_hreach, hh);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (c.sm.blk_crossed) atomicAdd(&pc->n_crossed, c.sm.blk_crossed);
    if (c.sm.blk_any_rows) atomicOr(&pc->any_rows, 1);
    if (c.sm.blk_colnnz) atomicAdd(&pc->colnnz, c.sm.blk_colnnz);
    if (c.sm.blk_reach) atomicAdd(&pc->reach, c.sm.blk_reach);
    if (c.sm.blk_hreach) atomicAdd(&pc->hreach, c.sm.blk_hreach);
    c.sm.blk_reach    = 0;
    c.sm.blk_hreach   = 0;
    c.sm.blk_crossed  = 0;
    c.sm.blk_any_rows = 0;
    c.sm.blk_colnnz   = 0;
  }
  __syncthreads();
}

// F4: per variable, the fold result from its candidate slot, then the reference's rules.
__device__ void phase_finalize(Ctx& c, ParCtl* pc, const int* list = nullptr, int nlist = 0)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  Tally t{0, 0, 0ull, 0ull, 0ull, 0};
  // uniform per-variable work: a static grid-stride sweep (no shared work cursor) over every
  // variable, or over the listed (touched) ones of a dirty-filtered round
  const int gw = blockIdx.x * kWarps + c.warp, nw = gridDim.x * kWarps;
  const int N  = list ? nlist : P.n;
  for (int q = 32 * gw; q < N; q += 32 * nw) {
    const int i = list ? (q + c.lane < nlist ? __ldcg(list + q + c.lane) : P.n) : q + c.lane;
    int res     = 0;
    if (i < P.n) {
      CandSlot* s                 = S.slot + i;
      const unsigned long long uk = s->up_key, lk = s->lo_key;
      if (uk != kUpEmpty || lk != kLoEmpty) {
        const double2 b = __ldcg(S.bounds + i);
        double nl = b.x, nu = b.y;
        if (uk != kUpEmpty) {
          nu = dekey(uk);
          if (nu == 0.0) nu = (s->up_zero & 1u) ? -0.0 : 0.0;
        }
        if (lk != kLoEmpty) {
          nl = dekey(lk);
          if (nl == 0.0) nl = (s->lo_zero & 1u) ? -0.0 : 0.0;
        }
        res = finish_var(S.bounds + i, b.x, b.y, nl, nu, __ldg(P.is_int + i) != 0, c.lim);
        // the slot of an unchanged variable persists: next round only its dirty rows republish,
        // and (candidates being monotone in the bounds of the other variables) the
        // kept values never undercut a fresh one, so the slot stays the exact fold
        if (res != 0) {
          s->up_key  = kUpEmpty;
          s->lo_key  = kLoEmpty;
          s->up_zero = kZeroEmpty;
          s->lo_zero = kZeroEmpty;
        }
      }
    }
    tally(c, pc, t, i < P.n ? i : -1, res);
  }
  tally_flush_block(c, pc, t);
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

// Packed tile of short columns (tighten-only calls with every variable).
__device__ void tighten_tile_packed(Ctx& c, int t, ParCtl* pc, Tally& ty)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int v0 = __ldg(P.sc_tile + t), v1 = __ldg(P.sc_tile + t + 1);
  const int p0 = __ldg(P.sc_ptr + v0), p1 = __ldg(P.sc_ptr + v1);
  int i = -1;
  if (c.lane < v1 - v0) {
    i                = __ldg(P.scol + v0 + c.lane);
    c.w.vb[c.lane]   = S.bounds[i];
    c.w.vint[c.lane] = __ldg(P.is_int + i);
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
  double2 b    = make_double2(0.0, 0.0);
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

// Phase B of frontier rounds (and tighten-only calls): CSC tightening of listed / all variables.
__device__ void phase_tighten(Ctx& c, ParCtl* pc, int par, bool full)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  Tally t{0, 0, 0ull, 0ull, 0ull, 0};
  {
    const int n    = full ? P.n_mcol : ldv(&pc->n_dvar_m);
    const int* ids = full ? P.mcol : S.dvar_m[par];
    for (Prefetch it_q(c, &pc->cur_vm, 1, n); it_q.t < n; it_q.advance()) {
    const int q = it_q.t;
      const int i = ids[q];
      const int r = tighten_warp(c, i);
      tally(c, pc, t, c.lane == 0 ? i : -1, c.lane == 0 ? r : 0);
    }
  }
  if (full) {
    for (Prefetch it_q(c, &pc->cur_vs, 1, P.n_sctile); it_q.t < P.n_sctile; it_q.advance())
      tighten_tile_packed(c, it_q.t, pc, t);
  } else {
    const int n = ldv(&pc->n_dvar_s);
    for (Prefetch it_q(c, &pc->cur_vs, 32, n); it_q.t < n; it_q.advance())
      tighten_list_tile(c, S.dvar_s[par], it_q.t, n, pc, t);
  }
  tally_flush_block(c, pc, t);
}

// ------------------------------------------------------------------ frontier

// One 128-incidence window of the row expansion: marks rows k[h] dirty for the next round and
// appends the new ones (short rows to drow_s; long rows as gather / fold / var-expansion tasks).
__device__ __forceinline__ void expand_rows_window(Ctx& c, ParCtl* qc, int qpar, unsigned stamp,
                                                   const int* k, unsigned long long& roww, int& nall)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  bool nw[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) nw[h] = k[h] >= 0 && atomicExch(S.row_stamp + k[h], stamp) != stamp;
  int RL[kEPL], n_s = 0, n_p = 0, n_f = 0, n_x = 0;
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    RL[h] = nw[h] ? __ldg(P.row_start + k[h] + 1) - __ldg(P.row_start + k[h]) : 0;
    roww += (unsigned long long)RL[h];
    nall += nw[h];
    const bool lg = nw[h] && RL[h] > kShortNnz;
    n_s += nw[h] && !lg;
    n_p += lg && RL[h] > kHeavyFold ? (RL[h] + kPiece - 1) / kPiece : 0;
    n_f += lg ? (RL[h] + kSumSegment - 1) / kSumSegment : 0;
    n_x += lg ? (RL[h] + kTile - 1) / kTile : 0;
  }
  int ps = warp_alloc(&qc->n_drow_s, n_s, c.lane);
#pragma unroll
  for (int h = 0; h < kEPL; ++h)
    if (nw[h] && RL[h] <= kShortNnz) S.drow_s[qpar][ps++] = k[h];
  if (__any_sync(FULL, n_f > 0)) {  // rare: a long row became dirty
    int pf = warp_alloc(&qc->n_dfold, n_f, c.lane);
    int px = warp_alloc(&qc->n_xtask, n_x, c.lane);
    int pp = warp_alloc(&qc->n_dpiece, n_p, c.lane);
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      if (!nw[h] || RL[h] <= kShortNnz) continue;
      if (RL[h] > kHeavyFold) {  // heavy: buffered fold, fed by contribution pieces
        const int p0 = __ldg(P.hpiece + k[h]);
        for (int s = 0; s * kPiece < RL[h]; ++s) S.dpiece[qpar][pp++] = make_int2(p0 + s, 0);
      }
      for (int s = 0; s * kSumSegment < RL[h]; ++s) S.dfold[qpar][pf++] = make_int2(k[h], s);
      for (int s = 0; s * kTile < RL[h]; ++s) S.xtask[qpar][px++] = make_int2(k[h], s);
    }
  }
}

// Adds this warp's accumulated expansion work to *total. Returns (warp-uniform) whether the
// expansion should stop early: the total crossed `budget` (the next round will be a full round, so
// the frontier lists are not needed) or another warp already stopped. budget = ~0: never stops.
__device__ __forceinline__ bool flush_work(Ctx& c, unsigned long long& acc, unsigned long long* total,
                                           int* abort_flag, unsigned long long budget)
{
  unsigned long long w = acc;
#pragma unroll
  for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(FULL, w, o);
  acc      = 0;
  int stop = 0;
  if (c.lane == 0) {
    if (w) {
      const unsigned long long old = atomicAdd(total, w);
      if (budget != ~0ull && old + w > budget) {
        stop = 1;
        atomicExch(abort_flag, 1);
      }
    }
    if (!stop && budget != ~0ull) stop = ldv(abort_flag);
  }
  return __shfl_sync(FULL, stop, 0) != 0;
}

// Phase C: rows(changed) → next round's dirty rows. Changed vars with short columns go 32 per
// warp (flattened 128-entry windows); longer columns were split into chunk tasks at append time.
__device__ void phase_expand_rows(Ctx& c, ParCtl* pc, ParCtl* qc, int qpar, unsigned stamp,
                                  unsigned long long budget)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  unsigned long long roww = 0;
  int nall                = 0;
  bool stop               = false;
  const bool eager        = budget != ~0ull;  // early exit enabled: flush per task
  const int nch = ldv(&pc->n_changed);
  for (Prefetch it_t(c, &pc->cur_x1, 32); it_t.t < nch && !stop; it_t.advance()) {
    const int t = it_t.t;
    const int j = t + c.lane;
    const int i = j < nch ? S.changed[j] : -1;
    int cs = 0, L = 0;
    if (i >= 0) {
      cs = __ldg(P.col_start + i);
      L  = __ldg(P.col_start + i + 1) - cs;
      if (L > kTile) L = 0;  // chunk tasks
    }
    int excl;
    const int T = list_tile_setup(c, cs, L, excl);
    for (int w0 = 0; w0 < T; w0 += kTile) {
      int k[kEPL];
#pragma unroll
      for (int h = 0; h < kEPL; ++h) {
        const int f = w0 + h * 32 + c.lane;
        k[h]        = -1;
        if (f < T) {
          const int o = owner_of(c.w.off, f);
          k[h]        = __ldg(P.col_row + c.w.st[o] + (f - c.w.off[o]));
        }
      }
      expand_rows_window(c, qc, qpar, stamp, k, roww, nall);
    }
    __syncwarp();
    if (eager) stop = flush_work(c, roww, &qc->roww, &qc->xabort, budget);
  }
  const int ntask = stop ? 0 : ldv(&pc->n_ctask);
  for (Prefetch it_t(c, &pc->cur_x2, 1); it_t.t < ntask && !stop; it_t.advance()) {
    const int t = it_t.t;
    const int2 tk = S.ctask[t];
    const int ce  = __ldg(P.col_start + tk.x + 1);
    const int e0  = __ldg(P.col_start + tk.x) + tk.y * kTile, e1 = min(ce, e0 + kTile);
    int k[kEPL];
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const int e = e0 + h * 32 + c.lane;
      k[h]        = e < e1 ? __ldg(P.col_row + e) : -1;
    }
    expand_rows_window(c, qc, qpar, stamp, k, roww, nall);
    if (eager) stop = flush_work(c, roww, &qc->roww, &qc->xabort, budget);
  }
  flush_work(c, roww, &qc->roww, &qc->xabort, ~0ull);
  nall = warp_sum(nall);
  if (c.lane == 0 && nall) atomicAdd(&qc->n_drow_all, nall);
}

// One 128-entry window of the var expansion: marks vars v[h] dirty and appends the new ones.
__device__ __forceinline__ void expand_vars_window(Ctx& c, ParCtl* qc, int qpar, unsigned stamp,
                                                   const int* v, unsigned long long& colw)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  bool nw[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) nw[h] = v[h] >= 0 && atomicExch(S.var_stamp + v[h], stamp) != stamp;
  int CL[kEPL], n_s = 0, n_m = 0;
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    CL[h] = nw[h] ? __ldg(P.col_start + v[h] + 1) - __ldg(P.col_start + v[h]) : 0;
    colw += (unsigned long long)CL[h];
    n_s += nw[h] && CL[h] <= kShortNnz;
    n_m += nw[h] && CL[h] > kShortNnz;
  }
  int ps = warp_alloc(&qc->n_dvar_s, n_s, c.lane);
  int pm = warp_alloc(&qc->n_dvar_m, n_m, c.lane);
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    if (!nw[h]) continue;
    if (CL[h] <= kShortNnz) S.dvar_s[qpar][ps++] = v[h];
    else S.dvar_m[qpar][pm++] = v[h];
  }
}

// Phase D: dirty rows → next round's dirty vars: short rows 32 per warp, long rows by chunk tasks.
__device__ void phase_expand_vars(Ctx& c, ParCtl* pc, ParCtl* qc, int qpar, unsigned stamp,
                                  unsigned long long budget)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  unsigned long long colw = 0;
  bool stop               = false;
  const bool eager        = budget != ~0ull;
  const int nr = ldv(&qc->n_drow_s);
  for (Prefetch it_t(c, &pc->cur_x3, 32); it_t.t < nr && !stop; it_t.advance()) {
    const int t = it_t.t;
    const int j = t + c.lane;
    const int k = j < nr ? S.drow_s[qpar][j] : -1;
    int rs = 0, L = 0;
    if (k >= 0) {
      rs = __ldg(P.row_start + k);
      L  = __ldg(P.row_start + k + 1) - rs;
    }
    int excl;
    const int T = list_tile_setup(c, rs, L, excl);
    for (int w0 = 0; w0 < T; w0 += kTile) {
      int v[kEPL];
#pragma unroll
      for (int h = 0; h < kEPL; ++h) {
        const int f = w0 + h * 32 + c.lane;
        v[h]        = -1;
        if (f < T) {
          const int o = owner_of(c.w.off, f);
          v[h]        = __ldg(P.row_col + c.w.st[o] + (f - c.w.off[o]));
        }
      }
      expand_vars_window(c, qc, qpar, stamp, v, colw);
    }
    __syncwarp();
    if (eager) stop = flush_work(c, colw, &qc->colw, &qc->xabort, budget);
  }
  const int ntask = stop ? 0 : ldv(&qc->n_xtask);
  for (Prefetch it_t(c, &pc->cur_x4, 1); it_t.t < ntask && !stop; it_t.advance()) {
    const int t = it_t.t;
    const int2 tk = S.xtask[qpar][t];
    const int re  = __ldg(P.row_start + tk.x + 1);
    const int e0  = __ldg(P.row_start + tk.x) + tk.y * kTile, e1 = min(re, e0 + kTile);
    int v[kEPL];
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const int e = e0 + h * 32 + c.lane;
      v[h]        = e < e1 ? __ldg(P.row_col + e) : -1;
    }
    expand_vars_window(c, qc, qpar, stamp, v, colw);
    if (eager) stop = flush_work(c, colw, &qc->colw, &qc->xabort, budget);
  }
  flush_work(c, colw, &qc->colw, &qc->xabort, ~0ull);
}

// Dirty marks for a dirty-filtered full round: row_stamp[k] = stamp for every row of a variable
// that changed this round (the reference's dirty_rows, propagation.hpp:474-476). Changed vars with
// short columns go 32 per warp (flattened 128-entry windows); longer columns by their chunk tasks.
// Appends id to dirty list q (0 slices, 1 groups, 2 pieces, 3 rows of SELL slices) for the lanes
// with `fresh`: one atomic per warp.
__device__ __forceinline__ void df_append(const DevState& S, int q, bool fresh, int id, int lane)
{
  const unsigned b = __ballot_sync(FULL, fresh);
  if (!b) return;
  int base = 0;
  if (lane == 0) base = atomicAdd(&S.ctl->df_cnt[q], __popc(b));
  base = __shfl_sync(FULL, base, 0);
  int* list = q == 0 ? S.df_slice : q == 1 ? S.df_group : q == 2 ? S.df_piece : S.df_rows;
  if (fresh) list[base + __popc(b & lanemask_lt())] = id;
}

// Marks the entries [e0, e1) (at most kTile) of a column, 32 lanes x kEPL loads in flight; rows of
// SELL slices are also appended, once per round (sell_stamp), to the dirty-row list (one atomic per
// warp and step).
__device__ __forceinline__ void mark_window(const DevProblem& P, const DevState& S, int e0, int e1,
                                            int lane, unsigned stamp)
{
  int mk[kEPL], rw[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    const int e = e0 + h * 32 + lane;
    mk[h]       = e < e1 ? __ldg(P.col_mark + e) : 0;
    rw[h]       = e < e1 ? __ldg(P.col_row + e) : -1;
  }
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    const bool on = rw[h] >= 0, light = on && mk[h] >= 0, sell = light && mk[h] < P.n_srtile;
    // the task (SELL slice / medium-row group / heavy-row piece) and the row: listed once per round
    bool task_new = false;
    if (light) {
      task_new = atomicExch(S.task_stamp + mk[h], stamp) != stamp;
      S.row_flag[rw[h]] = (unsigned char)stamp;
    } else if (on) {
      task_new = atomicExch(S.piece_dirty + (-mk[h] - 2), stamp) != stamp;
      S.row_stamp[rw[h]] = stamp;  // heavy row: its segment folds run (row_live)
    }
    df_append(S, 0, task_new && sell, mk[h], lane);
    df_append(S, 1, task_new && light && !sell, mk[h] - P.n_srtile, lane);
    df_append(S, 2, task_new && !light, -mk[h] - 2, lane);
    df_append(S, 3, sell && atomicExch(S.sell_stamp + rw[h], stamp) != stamp, rw[h], lane);
  }
}

// Dirty marks for a dirty-filtered full round: every row task (SELL slice, group of four medium rows,
// heavy-row piece + row) holding a variable that changed this round gets `stamp` (a superset of the
// reference's dirty_rows, propagation.hpp:474-476: recomputing a clean row is exact). One lane per
// changed var (columns <= kTile; longer ones by their chunk tasks).
__device__ void phase_mark_rows(Ctx& c, ParCtl* pc, unsigned stamp)
{
  const DevProblem& P = c.P;
  const DevState& S   = c.S;
  const int nch       = ldv(&pc->n_changed);
  const int gw = blockIdx.x * kWarps + c.warp, nw = gridDim.x * kWarps;
  // a warp per changed var (a lane walking its column serially costs a load latency per entry)
  for (int j = gw; j < nch; j += nw) {
    const int i  = S.changed[j];
    const int cs = __ldg(P.col_start + i), ce = __ldg(P.col_start + i + 1);
    if (ce - cs <= kTile) mark_window(P, S, cs, ce, c.lane, stamp);
  }
  const int ntask = ldv(&pc->n_ctask);
  for (int t = gw; t < ntask; t += nw) {
    const int2 tk = S.ctask[t];
    const int ce  = __ldg(P.col_start + tk.x + 1);
    const int e0  = __ldg(P.col_start + tk.x) + tk.y * kTile;
    mark_window(P, S, e0, min(ce, e0 + kTile), c.lane, stamp);
  }
}

// Empties every candidate slot (before a true full round when a previous round left data in them).
__device__ void clear_slots(const DevProblem& P, const DevState& S)
{
  CandSlot e;
  e.lo_key  = kLoEmpty;
  e.up_key  = kUpEmpty;
  e.lo_zero = kZeroEmpty;
  e.up_zero = kZeroEmpty;
  e.pad0 = e.pad1 = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) S.slot[i] = e;
}

__device__ void zero_par(ParCtl* q)
{
  int* w = reinterpret_cast<int*>(q);
  for (int j = 0; j < (int)(sizeof(ParCtl) / sizeof(int)); ++j) w[j] = 0;
}

#ifndef BP_MIN_BLOCKS
#define BP_MIN_BLOCKS 2
#endif
// F2 of a full round as its own launch: the row phase is a latency-bound stream of independent
// warp tasks, so it runs at the occupancy its own register budget allows instead of the
// cooperative engine's (whose allocation is the maximum over every phase).
#ifndef BP_F2_MIN_BLOCKS
#define BP_F2_MIN_BLOCKS 2
#endif
// Shared memory of k_rows_full: its row tasks stage 4 x kFoldVals values (heavy folds) or 4 x 32
// (grouped medium rows) in b0 / b1, so each warp gets a 3 KB region (b0 at 0, b1 at 2 KB) instead
// of a full WarpSmem: 24 KB per block, which lets the SM keep the larger L1 split (the bound
// gathers are L1 hits as often as the L1 is large).
// (TMA bulk copies of the heavy contribution streams were measured in round 2 -- 12% slower on C2:
// two chunks in flight per warp hide less latency than 128 independent register loads, and more
// buffers cost the L1 carveout; removed. profiles/README.md.)
#ifndef BP_ROWS_COMPACT_SMEM
#define BP_ROWS_COMPACT_SMEM 1
#endif
constexpr int kRowsWarpBytes = 3072;
static_assert(offsetof(WarpSmem, b1) == 2048 && 2048 + 128 * 8 <= kRowsWarpBytes, "row-task smem layout");
static_assert(4 * kFoldVals * 8 <= kRowsWarpBytes, "heavy-fold staging buffers");
#ifndef BP_ROWS_SMEM_PAD
#define BP_ROWS_SMEM_PAD 0
#endif
constexpr size_t kRowsSmem =
    BP_ROWS_COMPACT_SMEM ? (size_t)kWarps * kRowsWarpBytes + 16 + BP_ROWS_SMEM_PAD : sizeof(Smem);
// The host enqueues [k_rows_full, k_cand_pieces, k_engine(resume)] speculatively, several rounds
// ahead without waiting: each is a no-op unless the engine handed a full round over (need_full).
__global__ void __launch_bounds__(kThreads, BP_F2_MIN_BLOCKS)
    k_rows_full(DevProblem P, DevState S, Limits lim, int split_sell)
{
  // with split_sell the SELL slices run in k_rows_sell, launched as a programmatic dependent of
  // this grid: its blocks take over SM resources as soon as this grid's blocks retire
  if (split_sell) asm volatile("griddepcontrol.launch_dependents;");
  if (!ldv(&S.ctl->need_full)) return;
  const int rnd         = ldv(&S.ctl->rounds);
  const int par         = rnd & 1;
  const unsigned stamp  = ldv(&S.ctl->stamp_base) + (unsigned)rnd;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  Smem& sm       = *reinterpret_cast<Smem*>(dyn_smem);
  const int warp = threadIdx.x >> 5;
#if BP_ROWS_COMPACT_SMEM
  // compact warp regions: only the first 3 KB of a WarpSmem are used by the full round's row tasks
  WarpSmem& w = *reinterpret_cast<WarpSmem*>(dyn_smem + warp * kRowsWarpBytes);
#else
  WarpSmem& w = sm.w[warp];
#endif
  Ctx c{P, S, lim, sm, w, (int)(threadIdx.x & 31), warp};
  c.touch = ldv(&S.ctl->df_stamp);
  phase_rows(c, &S.ctl->par[par], par, true, true, stamp, false, !split_sell, c.touch);
}

// The SELL slices of a full round (short rows, thread per row) at this kernel's own occupancy:
// they need no shared memory and few registers, so many more warps keep gathers in flight than in
// k_rows_full. Launched with programmatic stream serialization right behind k_rows_full; before
// exiting, every block waits for k_rows_full to complete (griddepcontrol.wait), so this grid's
// completion -- which the following launches are stream-ordered on -- implies that one's.
#ifndef BP_SELL_MIN_BLOCKS
#define BP_SELL_MIN_BLOCKS 3  // 80 registers, 48 B spills (4: 64 registers, 216 B spills, slower)
#endif
__global__ void __launch_bounds__(kThreads, BP_SELL_MIN_BLOCKS)
    k_rows_sell(DevProblem P, DevState S, Limits lim)
{
  const bool on = ldv(&S.ctl->need_full) != 0;
  __shared__ __align__(16) unsigned char no_smem[16];  // sell_slice never touches the warp smem
  Smem& sm       = *reinterpret_cast<Smem*>(no_smem);
  const int warp = threadIdx.x >> 5;
  Ctx c{P, S, lim, sm, sm.w[0], (int)(threadIdx.x & 31), warp};
  if (on) {
    const int par = ldv(&S.ctl->rounds) & 1;
    c.touch       = ldv(&S.ctl->df_stamp);
    phase_sell(c, &S.ctl->par[par], true, c.touch);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // k_rows_full is complete: the candidate pieces of rows above kCandSplit (their activities are
  // published), here instead of in a launch of their own
  if (on) {
    const unsigned stamp = ldv(&S.ctl->stamp_base) + (unsigned)ldv(&S.ctl->rounds);
    const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
    for (int t = gw; t < P.n_cpiece; t += nw) {
      const int2 tk = P.cpiece_task[t];
      long_cand_piece(c, tk.x, tk.y, stamp, c.touch);
    }
  }
}

// Candidate pieces of rows above kCandSplit, after k_rows_full published their activities.
__global__ void __launch_bounds__(kThreads, 1) k_cand_pieces(DevProblem P, DevState S, Limits lim)
{
  if (!ldv(&S.ctl->need_full)) return;
  const unsigned stamp = ldv(&S.ctl->stamp_base) + (unsigned)ldv(&S.ctl->rounds);
  const unsigned ds    = ldv(&S.ctl->df_stamp);
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  Smem& sm       = *reinterpret_cast<Smem*>(dyn_smem);
  const int warp = threadIdx.x >> 5;
  Ctx c{P, S, lim, sm, sm.w[warp], (int)(threadIdx.x & 31), warp};
  c.touch = ds;
  const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  for (int t = gw; t < P.n_cpiece; t += nw) {
    const int2 tk = P.cpiece_task[t];
    long_cand_piece(c, tk.x, tk.y, stamp, ds);
  }
}

__global__ void __launch_bounds__(kThreads, BP_MIN_BLOCKS)
    k_engine(DevProblem P, DevState S, Limits lim, int mode, int full_first, unsigned stamp_base,
             unsigned long long dense_thr, long long* stats, int ext_f2, int resume,
             unsigned long long mark_max, int df_local)
{
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  Smem& sm            = *reinterpret_cast<Smem*>(dyn_smem);
  cg::grid_group grid = cg::this_grid();
  if (threadIdx.x == 0) {
    sm.blk_crossed  = 0;
    sm.blk_any_rows = 0;
    sm.blk_colnnz   = 0;
    sm.blk_reach    = 0;
    sm.blk_hreach   = 0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  Ctx c{P, S, lim, sm, sm.w[warp], (int)(threadIdx.x & 31), warp};

  if (mode == MODE_ACTIVITY) {
    const bool full = full_first != 0;
    phase_rows(c, &S.ctl->par[1], 1, full, false, stamp_base);
    return;
  }
  if (mode == MODE_TIGHTEN) {
    phase_tighten(c, &S.ctl->par[1], 1, full_first != 0);
    return;
  }

  // slot state of the previous launch / call (read by every thread before any lead write: the
  // lead writes it only after a grid barrier of this launch)
  int slot_state = ldv(S.slot_state);
  if (resume) {  // nothing handed over: the engine already finished (speculative launch)
    if (!ldv(&S.ctl->need_full)) return;
    grid.sync();  // every block has read need_full before it is cleared
    if (blockIdx.x == 0 && threadIdx.x == 0) S.ctl->need_full = 0;
  }
  const unsigned long long t0 = resume ? ldv(&S.ctl->t0) : globaltimer();
  const bool timed            = isfinite(lim.time_limit);
  const bool lead             = blockIdx.x == 0 && threadIdx.x == 0;
  bool full                   = true;  // round 1 is always a full sweep (propagation.hpp:442)
  bool any_change             = false;
  bool fixpoint               = false;
  int status = BP_STATUS_UNSET, crossed_out = 0;
  int rounds = 0;
  bool resumed = false;  // first iteration after k_rows_full ran this round's F2
  unsigned df_next = 0;  // dirty stamp marked for the next round (0: the next full round is a true one)
  if (resume) {
    rounds     = ldv(&S.ctl->rounds);
    any_change = ldv(&S.ctl->any_change) != 0;
    resumed    = true;
  } else {
    if (lead) {
      S.ctl->t0         = t0;
      S.ctl->stamp_base = stamp_base;
    }
    if (slot_state == 1) slot_state = 2;  // valid for the previous call's bounds only
  }
  if (!resume && full_first == 2) {
    // frontier start from a certified fixpoint: rows(changed) / vars(rows) of the staged list
    ParCtl* p0 = &S.ctl->par[0];
    ParCtl* p1 = &S.ctl->par[1];
    const unsigned long long dense2 = dense_thr == ~0ull ? ~0ull : 2 * dense_thr;
    phase_expand_rows(c, p0, p1, 1, stamp_base, dense2);
    grid.sync();
    const unsigned long long rw0 = ldv(&p1->roww);
    if (rw0 <= dense2) {
      phase_expand_vars(c, p0, p1, 1, stamp_base, dense2 == ~0ull ? ~0ull : dense2 - rw0);
      grid.sync();
    }
    full = dense_thr != ~0ull && ldv(&p1->roww) + ldv(&p1->colw) > 2 * dense_thr;
    if (ldv(&p1->n_drow_all) == 0) {  // nothing to revisit: the fixpoint stands
      full     = false;
      rounds   = lim.max_rounds;  // skip the loop; result = Unchanged after one round below
      fixpoint = true;
    }
  }
  if (rounds == lim.max_rounds && fixpoint) {
    rounds = 1;  // the reference's first (full) round finds no change
  } else {
  while (rounds < lim.max_rounds || resumed) {
    if (!resumed) ++rounds;
    const int ppar       = rounds & 1, qpar = ppar ^ 1;
    ParCtl* pc           = &S.ctl->par[ppar];
    ParCtl* qc           = &S.ctl->par[qpar];
    long long* st        = stats ? stats + (long long)(rounds - 1) * kStatCols : nullptr;
    const bool fr        = full || !lim.incremental;
    const unsigned stamp = stamp_base + (unsigned)rounds;
    // A full round right after a full / dirty-filtered one whose changed vars' rows were marked is
    // dirty-filtered: only the marked rows are recomputed and republish; any other
    // full round is a true one and starts from empty candidate slots.
    // (ds = 0 with valid slots: every row is recomputed and republishes into the persistent slots --
    // equally exact; chosen when marking would cost more than it saves)
    unsigned ds = 0;
    if (fr && !resumed) {
      ds = slot_state == 1 ? df_next : 0u;
      if (slot_state == 2) {
        clear_slots(P, S);
        grid.sync();
        slot_state = 0;
      }
    }
    df_next = 0;
    // the dirty-filter stamp of this round's row phase (handed to k_rows_full before a resume)
    const unsigned rds = resumed ? ldv(&S.ctl->df_stamp) : ds;
    if (!fr) {  // a frontier round reads records it does not recompute: no stale heavy row
      const bool rf = ldv(&S.ctl->stale) != 0;
      if (rf) {
        grid.sync();  // every block has read the flag
        if (lead) S.ctl->stale = 0;
        phase_refresh(c, stamp);
        grid.sync();
      }
    }
    if (resumed) {
      resumed = false;  // this round's F2 (fused rows + candidates) ran in k_rows_full
    } else if (fr && ext_f2 &&
               !(ds != 0 && ldv(&S.ctl->df_cnt[1]) + ldv(&S.ctl->df_cnt[2]) +
                                    min(ldv(&S.ctl->df_cnt[0]), (ldv(&S.ctl->df_cnt[3]) + 31) / 32) <=
                                df_local)) {
      // hand the full round's row phase to k_rows_full; the host relaunches us with resume=1
      // (a dirty-filtered round with at most df_local row tasks runs here: its launches and the
      // relaunch would cost more than the occupancy they buy)
      if (lead) {
        if (st) st[10] = (long long)(globaltimer() - t0);
        S.ctl->rounds     = rounds;
        S.ctl->any_change = any_change ? 1 : 0;
        S.ctl->df_stamp   = ds;
        *S.slot_state     = slot_state;
        S.ctl->need_full  = 1;
      }
      return;
    } else {
      if (st && lead) st[10] = (long long)(globaltimer() - t0);
      c.touch = fr ? ds : 0u;
      phase_rows(c, pc, ppar, fr, fr, stamp, true, true, ds);
      c.touch = 0;
      grid.sync();
    }
    if (st && lead) st[6] = (long long)(globaltimer() - t0);
    if (lead) {
      zero_par(qc);  // safe: every block has finished reading the previous round's counters
      for (int j = 0; j < kMultiCursors; ++j) S.ctl->mcur[(qpar * kMultiCursors + j) * 32] = 0;
      // the dirty lists the marks below append to (this round's row phase has consumed them)
      S.ctl->df_cnt[0] = S.ctl->df_cnt[1] = S.ctl->df_cnt[2] = S.ctl->df_cnt[3] = 0;
      if (timed && (double)(globaltimer() - t0) * 1e-9 >= lim.time_limit) pc->stop = 1;
    }
    if (fr && rds != 0) phase_finalize(c, pc, S.touched, ldv(&S.ctl->n_touch));
    else if (fr) phase_finalize(c, pc);
    else phase_tighten(c, pc, ppar, false);
    grid.sync();
    if (lead) S.ctl->n_touch = 0;  // (read by every block before the barrier above)
    slot_state   = fr ? 1 : (slot_state == 0 ? 0 : 2);  // a frontier round leaves the slots stale
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
    if (nc == 0) {
      fixpoint = true;
      break;
    }
    any_change = true;
    if (!ldv(&pc->any_rows)) {  // dirty_rows.empty() (propagation.hpp:481)
      fixpoint = true;
      break;
    }
    if (rounds >= lim.max_rounds) break;
    if (ldv(&pc->stop)) break;       // time limit (propagation.hpp:439)
    // the next frontier would span the matrix: even the upper bound of its work (Σ reach of the
    // changed vars, duplicates counted) is checked against 4x the full-round threshold, so a
    // "full" prediction is only taken when the frontier is certainly large or nearly so
    // the next round is a full one: with valid slots, mark the rows of this round's changed vars
    // (complete even when a frontier expansion below stopped early) and filter by them
    auto go_full = [&]() {
      if (slot_state == 1 && ldv(&pc->colnnz) <= mark_max) {
        phase_mark_rows(c, pc, stamp);  // marks + dirty lists (appended)
        grid.sync();                    // complete before the row phase reads them
        if (st && lead) st[8] = st[9] = st[11] = (long long)(globaltimer() - t0);
        df_next = stamp;
      }
      full = true;
    };
    // with valid slots a dirty-filtered round (the dirty rows only, no CSC pass, no expansion) is
    // never more work than the frontier round it replaces
    if (!lim.incremental || (slot_state == 1 && dense_thr != ~0ull) || ldv(&pc->colnnz) > dense_thr ||
        (dense_thr != ~0ull &&
         ldv(&pc->reach) + min(ldv(&pc->hreach), P.h_reach) > 4 * dense_thr)) {
      go_full();
      continue;
    }
    // both expansions stop early once the next round is known to be a full round
    phase_expand_rows(c, pc, qc, qpar, stamp, dense_thr);
    grid.sync();
    if (st && lead) st[8] = st[9] = (long long)(globaltimer() - t0);
    if (ldv(&qc->roww) > dense_thr) {
      go_full();
      continue;
    }
    phase_expand_vars(c, pc, qc, qpar, stamp,
                      dense_thr == ~0ull ? ~0ull : 2 * dense_thr - ldv(&qc->roww));
    grid.sync();
    if (st && lead) st[9] = (long long)(globaltimer() - t0);
    // a frontier round costs ~ its gathers (row nnz + col nnz); a fused full round ~ N = 4 dense_thr
    // gathers but with far better memory-level parallelism
    full = dense_thr != ~0ull && ldv(&qc->roww) + ldv(&qc->colw) > 2 * dense_thr;
    if (full) go_full();
  }
  }
  {  // the call leaves exact records: refresh the heavy rows a lazy round left stale
    const bool rf = ldv(&S.ctl->stale) != 0;
    if (rf) {
      grid.sync();
      if (lead) S.ctl->stale = 0;
      phase_refresh(c, stamp_base + (unsigned)rounds);
      grid.sync();
    }
  }
  if (lead) {
    if (status == BP_STATUS_UNSET) status = any_change ? BP_STATUS_TIGHTENED : BP_STATUS_UNCHANGED;
    S.ctl->status     = status;
    S.ctl->rounds     = rounds;
    S.ctl->crossed    = crossed_out;
    S.ctl->any_change = any_change ? 1 : 0;
    S.ctl->fixpoint   = fixpoint ? 1 : 0;
    *S.slot_state     = slot_state;
  }
}

}  // namespace

// ------------------------------------------------------------------ host side

DevProblem Problem::dev() const
{
  DevProblem d;
  d.n           = n;
  d.m           = m;
  d.nnz         = nnz;
  d.row_start   = row_start.p;
  d.row_col     = row_col.p;
  d.row_val     = row_val.p;
  d.row_ci      = row_ci.p;
  d.col_start   = col_start.p;
  d.col_row     = col_row.p;
  d.col_val     = col_val.p;
  d.cons        = cons.p;
  d.is_int      = is_int.p;
  d.n_srow      = n_srow;
  d.n_srtile    = n_srtile;
  d.n_srow_long = n_srow_long;
  d.srow        = srow.p;
  d.sell_pos    = sell_pos.p;
  d.sr_ptr      = sr_ptr.p;
  d.sr_ci       = sr_ci.p;
  d.sr_val      = sr_val.p;
  d.sr_own      = sr_own.p;
  d.sr_tile     = sr_tile.p;
  d.long_off    = long_off.p;
  d.hpiece      = hpiece.p;
  d.n_piece     = n_piece;
  d.piece_task  = piece_task.p;
  d.n_fold      = n_fold;
  d.n_fold_heavy = n_fold_heavy;
  d.fold_task   = fold_task.p;
  d.n_cpiece    = n_cpiece;
  d.cpiece_task = cpiece_task.p;
  d.seg_base    = seg_base.p;
  d.n_scol      = n_scol;
  d.n_sctile    = n_sctile;
  d.scol        = scol.p;
  d.sc_ptr      = sc_ptr.p;
  d.sc_row      = sc_row.p;
  d.sc_val      = sc_val.p;
  d.sc_own      = sc_own.p;
  d.sc_tile     = sc_tile.p;
  d.n_mcol      = n_mcol;
  d.reach       = reach.p;
  d.h_reach     = h_reach;
  d.mcol        = mcol.p;
  d.col_mark    = col_mark.p;
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

Packed pack_short(int count, const int* start, const int* idx, const double* val,
                  const uint8_t* int_flag, int max_len, int tile_entries)
{
  Packed pk;
  pk.ptr.push_back(0);
  for (int k = 0; k < count; ++k) {
    const int L = start[k + 1] - start[k];
    if (L > max_len) continue;
    pk.ids.push_back(k);
    for (int e = start[k]; e < start[k + 1]; ++e) {
      pk.idx.push_back(int_flag && int_flag[idx[e]] ? (idx[e] | kIntBit) : idx[e]);
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
    while (q < ns && q - r < 32 && pk.ptr[q + 1] - base <= tile_entries) {
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
  {
    std::vector<int> ci(N);
    for (long long e = 0; e < N; ++e)
      ci[e] = is_integer[row_col[e]] ? (row_col[e] | kIntBit) : row_col[e];
    P.row_ci.upload(ci);
  }
  P.col_start.upload(col_start, n + 1);
  P.col_row.upload(col_row_in, N);
  P.col_val.upload(col_val_in, N);
  std::vector<double2> cons(m);
  for (int k = 0; k < m; ++k) cons[k] = make_double2(cons_lower[k], cons_upper[k]);
  P.cons.upload(cons);
  P.is_int.upload(is_integer, n);

  // Short rows / columns: packed tiles.
  std::vector<int> srow_h;  // SELL slice lane -> row (host copy for the task map)
  {
    // Rows with nnz <= kPackNnz as SELL-32 slices: rows sorted by length (descending, stable), 32
    // per slice, each slice padded to its longest row, entries column-interleaved so lane i reads
    // entry j of its row at base + 32 j + i (coalesced). Any grouping is exact: every row is
    // summed by one thread in its own order, and candidate publication is order-independent.
    std::vector<int> srows;
    for (int k = 0; k < m; ++k)
      if (row_start[k + 1] - row_start[k] <= kPackNnz) srows.push_back(k);
    std::stable_sort(srows.begin(), srows.end(), [&](int a, int b) {
      return row_start[a + 1] - row_start[a] > row_start[b + 1] - row_start[b];
    });
    const int nsl = ((int)srows.size() + 31) / 32;
    std::vector<int> sbase(nsl + 1, 0), srow(32 * (size_t)nsl, -1);
    long long tot = 0;
    for (int sl = 0; sl < nsl; ++sl) {
      sbase[sl]      = (int)tot;
      const int Lmax = row_start[srows[32 * sl] + 1] - row_start[srows[32 * sl]];
      tot += 32ll * Lmax;
      if (tot > 0x7FFFFFFFll) throw std::runtime_error("SELL slices exceed int32 offsets");
    }
    sbase[nsl] = (int)tot;
    std::vector<int> sci((size_t)tot, -1);
    std::vector<double> sval((size_t)tot, 0.0);
    for (int sl = 0; sl < nsl; ++sl)
      for (int i = 0; i < 32 && 32 * sl + i < (int)srows.size(); ++i) {
        const int k           = srows[32 * sl + i];
        srow[32 * (size_t)sl + i] = k;
        for (int e = row_start[k], j = 0; e < row_start[k + 1]; ++e, ++j) {
          const size_t q = (size_t)sbase[sl] + 32 * (size_t)j + i;
          sci[q]         = is_integer[row_col[e]] ? (row_col[e] | kIntBit) : row_col[e];
          sval[q]        = row_val[e];
        }
      }
    P.n_srow   = (int)srows.size();
    P.n_srtile = nsl;
    P.n_srow_long = 0;  // slices whose longest row exceeds kShortNnz (fetched one at a time)
    while (P.n_srow_long < nsl && sbase[P.n_srow_long + 1] - sbase[P.n_srow_long] > 32 * kShortNnz)
      ++P.n_srow_long;
    P.srow.upload(srow);
    std::vector<int> spos(std::max(m, 1), -1);
    for (size_t q = 0; q < srow.size(); ++q)
      if (srow[q] >= 0) spos[srow[q]] = (int)q;
    P.sell_pos.upload(spos);
    srow_h = srow;
    P.sr_ci.upload(sci);
    P.sr_val.upload(sval);
    P.sr_tile.upload(sbase);
    Packed c   = pack_short(n, col_start, col_row_in, col_val_in, nullptr, kShortNnz, kTile);
    P.n_scol   = (int)c.ids.size();
    P.n_sctile = (int)c.tile.size() - 1;
    P.scol.upload(c.ids);
    P.sc_ptr.upload(c.ptr);
    P.sc_row.upload(c.idx);
    P.sc_val.upload(c.val);
    P.sc_own.upload(c.own);
    P.sc_tile.upload(c.tile);
  }
  // Long rows: gather pieces, fold tasks per 16384-segment (longest first: the fold is a
  // sequential chain), candidate pieces for rows above kCandSplit.
  // Full-round fold tasks (rows > kPackNnz, per 16384-segment, longest segments first: the fold
  // is a sequential chain) and candidate pieces of rows above kCandSplit; frontier rounds fold
  // every dirty row > kShortNnz (capacity nf_cap).
  std::vector<int> seg_base(m, -1), order;
  int slot = 0;
  long long nf_front = 0;
  for (int k = 0; k < m; ++k) {
    const int L = row_start[k + 1] - row_start[k];
    if (L <= kShortNnz) continue;
    const int ns = (L + kSumSegment - 1) / kSumSegment;
    nf_front += ns;
    if (ns > 1) {
      seg_base[k] = slot;
      slot += ns;
    }
    if (L > kPackNnz) order.push_back(k);
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return row_start[a + 1] - row_start[a] > row_start[b + 1] - row_start[b];
  });
  std::vector<int2> cpiece, piece;
  std::vector<std::pair<int, int2>> folds;
  std::vector<int> long_off(m, -1), hpiece(m, -1);
  long long goff = 0;
  for (int k : order) {
    const int L = row_start[k + 1] - row_start[k];
    if (L > kCandSplit)
      for (int p = 0; p * kPiece < L; ++p) cpiece.push_back(make_int2(k, p));
    if (L > kHeavyFold) {
      long_off[k] = (int)goff;
      goff += ((L + kTile - 1) / kTile) * (long long)kTile;
      if (goff > 0x7FFFFFFFll) throw std::runtime_error("heavy-row entries exceed int32 offsets");
      hpiece[k] = (int)piece.size();
      for (int p = 0; p * kPiece < L; ++p) piece.push_back(make_int2(k, p));
    }
    for (int s = 0; s * kSumSegment < L; ++s)
      folds.push_back({std::min(L - s * kSumSegment, kSumSegment), make_int2(k, s)});
  }
  // heavy-row segments first (longest first), then the medium rows (longest first): medium rows
  // are folded four per warp (group_fold), so neighbours in the list have similar lengths
  auto heavy_row = [&](int k) { return row_start[k + 1] - row_start[k] > kHeavyFold; };
  std::stable_sort(folds.begin(), folds.end(), [&](const auto& a, const auto& b) {
    const bool ha = heavy_row(a.second.x), hb = heavy_row(b.second.x);
    if (ha != hb) return ha;
    return a.first > b.first;
  });
  std::vector<int2> fold(folds.size());
  P.n_fold_heavy = 0;
  for (size_t j = 0; j < folds.size(); ++j) {
    fold[j] = folds[j].second;
    if (heavy_row(fold[j].x)) P.n_fold_heavy++;
  }
  P.n_long_entries = goff;
  P.n_piece        = (int)piece.size();
  P.long_off.upload(long_off);
  P.hpiece.upload(hpiece);
  P.h_hpiece = hpiece;
  {
    // per CSC entry: the row task holding it, for the marks of dirty-filtered rounds -- the SELL
    // slice (0 .. n_srtile), the group of four medium rows (n_srtile + (fold index - n_fold_heavy) / 4,
    // as phase_rows fetches them) or, for heavy rows, -(piece + 2). CSC positions follow the same
    // stable transpose as the CSC itself.
    std::vector<int> row_task(m, -1);
    for (size_t q = 0; q < srow_h.size(); ++q)
      if (srow_h[q] >= 0) row_task[srow_h[q]] = (int)(q / 32);
    for (size_t j = P.n_fold_heavy; j < fold.size(); ++j)
      row_task[fold[j].x] = P.n_srtile + (int)((j - P.n_fold_heavy) / 4);
    std::vector<int> cmk((size_t)N, 0), cur(col_start, col_start + n);
    for (int k = 0; k < m; ++k)
      for (int e = row_start[k]; e < row_start[k + 1]; ++e) {
        const int d = cur[row_col[e]]++;
        cmk[d]      = hpiece[k] >= 0 ? -(hpiece[k] + (e - row_start[k]) / kPiece) - 2 : row_task[k];
        if (cmk[d] == -1) throw std::runtime_error("row without a full-round task");
      }
    P.col_mark.upload(cmk);
    P.n_task = P.n_srtile + (int)((fold.size() - P.n_fold_heavy + 3) / 4);
  }
  P.piece_task.upload(piece);
  P.n_fold         = (int)fold.size();
  P.n_cpiece       = (int)cpiece.size();
  P.n_part         = slot;
  P.fold_task.upload(fold);
  P.cpiece_task.upload(cpiece);
  P.seg_base.upload(seg_base);
  // reach[i] = Σ_{k in col i} (len(k) + Σ_{j in row k} collen(j)): an upper bound of the frontier
  // work (row + column incidences) a change of var i can cause in the next round.
  // Rows longer than kHeavyFold are shared by many variables: their part is kept separately
  // (reach[2i+1]) and capped, over all changed vars together, by their total h_reach.
  {
    std::vector<unsigned long long> rowcol(m, 0);
    unsigned long long htot = 0;
    for (int k = 0; k < m; ++k) {
      unsigned long long acc = (unsigned long long)(row_start[k + 1] - row_start[k]);
      for (int e = row_start[k]; e < row_start[k + 1]; ++e)
        acc += (unsigned long long)(col_start[row_col[e] + 1] - col_start[row_col[e]]);
      rowcol[k] = acc;
      if (row_start[k + 1] - row_start[k] > kHeavyFold) htot += acc;
    }
    std::vector<unsigned long long> rc(2 * (size_t)n, 0);
    for (int i = 0; i < n; ++i)
      for (int e = col_start[i]; e < col_start[i + 1]; ++e) {
        const int k = col_row_in[e];
        rc[2 * i + (row_start[k + 1] - row_start[k] > kHeavyFold ? 1 : 0)] += rowcol[k];
      }
    P.reach.upload(rc);
    P.h_reach = htot;
  }
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
  P.gbuf.alloc((size_t)std::max(P.n_long_entries, 1ll));
  P.pcnt.alloc((size_t)std::max(P.n_piece, 1));
  P.pagg.alloc((size_t)std::max(P.n_piece, 1));
  P.sfold.alloc((size_t)std::max(P.n_piece, 1));
  BP_CUDA(cudaMemset(P.sfold.p, 0, sizeof(unsigned) * P.sfold.n));
  P.cinfo.alloc((size_t)std::max(P.n_long_entries / kTile, 1ll));
  P.pstamp.alloc((size_t)std::max(P.n_piece, 1));
  P.piece_dirty.alloc((size_t)std::max(P.n_piece, 1));
  BP_CUDA(cudaMemset(P.piece_dirty.p, 0, sizeof(unsigned) * std::max(P.n_piece, 1)));
  P.task_stamp.alloc((size_t)std::max(P.n_task, 1));
  BP_CUDA(cudaMemset(P.task_stamp.p, 0, sizeof(unsigned) * std::max(P.n_task, 1)));
  P.ckpt.alloc((size_t)std::max(P.n_piece, 1));
  BP_CUDA(cudaMemset(P.pstamp.p, 0, sizeof(unsigned) * std::max(P.n_piece, 1)));
  P.slot.alloc(nn);
  {
    std::vector<CandSlot> empty(nn);
    for (auto& s : empty) {
      s.lo_key  = kLoEmpty;
      s.up_key  = kUpEmpty;
      s.lo_zero = kZeroEmpty;
      s.up_zero = kZeroEmpty;
      s.pad0 = s.pad1 = 0;
    }
    BP_CUDA(cudaMemcpy(P.slot.p, empty.data(), sizeof(CandSlot) * nn, cudaMemcpyHostToDevice));
  }
  P.ready.alloc(mm);
  BP_CUDA(cudaMemset(P.ready.p, 0, sizeof(unsigned) * mm));
  P.rquiet.alloc(mm);
  BP_CUDA(cudaMemset(P.rquiet.p, 0, mm));
  P.seg_part.alloc(std::max(slot, 1));
  P.seg_done.alloc(mm);
  BP_CUDA(cudaMemset(P.seg_done.p, 0, sizeof(int) * mm));
  P.row_stamp.alloc(mm);
  P.var_stamp.alloc(nn);
  BP_CUDA(cudaMemset(P.row_stamp.p, 0, sizeof(unsigned) * mm));
  BP_CUDA(cudaMemset(P.var_stamp.p, 0, sizeof(unsigned) * nn));
  // int lists per parity: drow_s (m), dvar_s, dvar_m (n each); changed (n)
  P.lists_i.alloc(2 * (mm + 2 * nn) + nn);
  // int2 lists per parity: dpiece, dfold (all long-row tasks), xtask (N/256 + m)
  const size_t np_cap = (size_t)std::max(P.n_piece, 1);  // dirty heavy rows' contribution pieces
  const size_t nf_cap = (size_t)std::max(nf_front, 1ll);
  const size_t nx_cap = (size_t)(N / kTile) + mm + 1;
  P.lists_i2.alloc(2 * (np_cap + nf_cap + nx_cap) + (size_t)(N / kTile) + nn + 1);
  P.ctl.alloc(1);
  BP_CUDA(cudaMemset(P.ctl.p, 0, sizeof(Ctl)));
  DevState& S = P.st;
  S.bounds    = P.bounds.p;
  S.rec       = P.rec.p;
  S.aux       = P.aux.p;
  S.gmin      = reinterpret_cast<double*>(P.gbuf.p);
  S.gmax      = S.gmin + std::max(P.n_long_entries, 1ll);
  S.pcnt      = P.pcnt.p;
  S.pagg      = P.pagg.p;
  S.sfold     = P.sfold.p;
  S.slot      = P.slot.p;
  P.slot_state.alloc(1);
  BP_CUDA(cudaMemset(P.slot_state.p, 0, sizeof(int)));  // the slots start empty
  S.slot_state = P.slot_state.p;
  S.ready     = P.ready.p;
  S.rquiet    = P.rquiet.p;
  S.cinfo     = P.cinfo.p;
  S.pstamp    = P.pstamp.p;
  S.piece_dirty = P.piece_dirty.p;
  S.task_stamp  = P.task_stamp.p;
  P.row_flag.alloc(mm);
  BP_CUDA(cudaMemset(P.row_flag.p, 0, mm));
  S.row_flag = P.row_flag.p;
  S.n_task      = P.n_task;
  P.df_lists.alloc((size_t)std::max(P.n_task + P.n_piece, 1));
  S.df_slice = P.df_lists.p;
  S.df_group = P.df_lists.p + P.n_srtile;
  S.df_piece = P.df_lists.p + P.n_task;
  P.df_rows.alloc((size_t)std::max(m, 1));
  S.df_rows = P.df_rows.p;
  P.vtouch.alloc((size_t)std::max(n, 1));
  BP_CUDA(cudaMemset(P.vtouch.p, 0, sizeof(unsigned) * P.vtouch.n));
  S.vtouch = P.vtouch.p;
  P.touched.alloc((size_t)std::max(n, 1));
  S.touched = P.touched.p;
  P.sell_stamp.alloc((size_t)std::max(m, 1));
  BP_CUDA(cudaMemset(P.sell_stamp.p, 0, sizeof(unsigned) * P.sell_stamp.n));
  S.sell_stamp = P.sell_stamp.p;
  S.ckpt      = P.ckpt.p;
  S.seg_part  = P.seg_part.p;
  S.seg_done  = P.seg_done.p;
  S.row_stamp = P.row_stamp.p;
  S.var_stamp = P.var_stamp.p;
  int* pi     = P.lists_i.p;
  int2* pi2   = P.lists_i2.p;
  for (int q = 0; q < 2; ++q) {
    S.drow_s[q] = pi;
    pi += mm;
    S.dvar_s[q] = pi;
    pi += nn;
    S.dvar_m[q] = pi;
    pi += nn;
    S.dpiece[q] = pi2;
    pi2 += np_cap;
    S.dfold[q] = pi2;
    pi2 += nf_cap;
    S.xtask[q] = pi2;
    pi2 += nx_cap;
  }
  S.changed = pi;
  S.ctask   = pi2;  // sum over vars of ceil(col nnz / kTile) <= N / kTile + n
  S.ctl     = P.ctl.p;
  S.dbg     = nullptr;
  if (getenv("BP_DEBUG")) {
    P.dbg.alloc(24);
    BP_CUDA(cudaMemset(P.dbg.p, 0, 24 * sizeof(unsigned long long)));
    S.dbg = P.dbg.p;
  }

  int dev_sms = 0, per_sm = 0;
  BP_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, P.device));
  BP_CUDA(cudaFuncSetAttribute(k_engine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sizeof(Smem)));
  BP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_engine, kThreads, sizeof(Smem)));
  if (per_sm < 1) throw cuda_error("engine kernel cannot be resident (occupancy 0)");
  P.grid_blocks = dev_sms * std::min(per_sm, 4);
  // small problems get a grid sized to their work (>= one block per 8192 nonzeros): cheaper grid
  // barriers, and independent instances on their own streams can run side by side (a cooperative
  // grid only launches when all its blocks fit)
  static const int grid_div = getenv("BP_GRID_NNZ") ? atoi(getenv("BP_GRID_NNZ")) : 8192;
  if (grid_div > 0)
    P.grid_blocks = (int)std::max<long long>(std::min<long long>(P.grid_blocks, 16),
                                             std::min<long long>(P.grid_blocks, (P.nnz + grid_div - 1) / grid_div));
  int per_sm2   = 0;
  BP_CUDA(cudaFuncSetAttribute(k_rows_full, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sizeof(Smem)));
  BP_CUDA(cudaFuncSetAttribute(k_cand_pieces, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sizeof(Smem)));
  BP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_rows_full, kThreads, kRowsSmem));
  static const int f2_per_sm = getenv("BP_F2_PER_SM") ? atoi(getenv("BP_F2_PER_SM")) : 0;
  if (f2_per_sm > 0) per_sm2 = std::min(per_sm2, f2_per_sm);
  P.f2_blocks = dev_sms * std::max(per_sm2, 1);
  int per_sm3   = 0;
  BP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, k_rows_sell, kThreads, 0));
  P.sell_blocks = dev_sms * std::max(per_sm3, 1);
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
  int ff       = (mode == MODE_PROPAGATE && (flags & ENGINE_START_FRONTIER)) ? 2 : (full ? 1 : 0);
  // stamps: one value per round, never reused until wrap-around (then the stamp arrays reset)
  if (P.stamp_base > 0xF0000000u - (unsigned)std::max(lim.max_rounds, 1) - 2) {
    BP_CUDA(cudaMemsetAsync(P.row_stamp.p, 0, sizeof(unsigned) * P.row_stamp.n, s));
    BP_CUDA(cudaMemsetAsync(P.sell_stamp.p, 0, sizeof(unsigned) * P.sell_stamp.n, s));
    BP_CUDA(cudaMemsetAsync(P.vtouch.p, 0, sizeof(unsigned) * P.vtouch.n, s));
    BP_CUDA(cudaMemsetAsync(P.var_stamp.p, 0, sizeof(unsigned) * P.var_stamp.n, s));
    BP_CUDA(cudaMemsetAsync(P.ready.p, 0, sizeof(unsigned) * P.ready.n, s));
    BP_CUDA(cudaMemsetAsync(P.pstamp.p, 0, sizeof(unsigned) * P.pstamp.n, s));
    BP_CUDA(cudaMemsetAsync(P.sfold.p, 0, sizeof(unsigned) * P.sfold.n, s));
    BP_CUDA(cudaMemsetAsync(P.piece_dirty.p, 0, sizeof(unsigned) * P.piece_dirty.n, s));
    BP_CUDA(cudaMemsetAsync(P.task_stamp.p, 0, sizeof(unsigned) * P.task_stamp.n, s));
    P.stamp_base = 1;
  }
  unsigned sb = P.stamp_base;
  P.stamp_base += (unsigned)std::max(lim.max_rounds, 1) + 1;
  // a round is evaluated as a full sweep when its frontier (dirty-row nnz + dirty-column nnz)
  // exceeds kFullPct % of nnz: a fused full round costs about as much as a frontier round over
  // ~40% of the matrix (frontier work per entry is the CSC gather, ~2.5x a full round's)
  static const int full_pct = getenv("BP_FULL_PCT") ? atoi(getenv("BP_FULL_PCT")) : 35;
  unsigned long long dense_thr =
      (flags & ENGINE_FORCE_FRONTIER) ? ~0ull : (unsigned long long)(P.nnz * full_pct / 200);
  long long* stp = d_stats;
  static const bool no_ext = getenv("BP_NO_EXT_F2") != nullptr;
  // small problems keep the row phase inside the engine: the hand-off's host round trip would
  // cost more than the occupancy it buys
  static const long long ext_min = getenv("BP_EXT_MIN_NNZ") ? atoll(getenv("BP_EXT_MIN_NNZ")) : 2000000;
  int ext        = (mode == MODE_PROPAGATE && !no_ext && P.nnz >= ext_min) ? 1 : 0;
  int resume     = 0;
  // SELL slices in k_rows_sell at their own occupancy (24 warps / SM at 80 registers, vs 16 in
  // k_rows_full), a programmatic dependent of k_rows_full. Round 1 measured it slower (9.45 -> 11.0
  // ms, 64 registers with spills, next to the heavy chains); with lazy heavy rows and 3 blocks / SM
  // it is 1-3% faster on C2 (tools/gpu_ab.sh: 6.98 -> 6.76, 6.93 -> 6.86 ms). BP_SPLIT_SELL=0: off.
  static const int split_env = getenv("BP_SPLIT_SELL") ? atoi(getenv("BP_SPLIT_SELL")) : 1;
  const int split_sell       = split_env && P.n_srtile > 0 ? 1 : 0;
  // dirty-filtered rounds when the changed vars' columns hold at most BP_DF_MARK_PCT % of the nnz:
  // beyond that the marks and lists cost more than the rows they spare (C2, tools/gpu_ab.sh:
  // 1 % 8.72, 2 % 8.77, 3 % 8.83, 5 % 8.94, 8 % 9.06, 15 % 9.24 ms per propagate; at the end of the
  // round: 0.5 % 5.52, 0.75 % 5.62, 1 % 5.53, 1.5 % 5.55, 2 % 5.57, 3 % 5.68)
  static const double mark_pct = getenv("BP_DF_MARK_PCT") ? atof(getenv("BP_DF_MARK_PCT")) : 1.0;
  unsigned long long mark_max = (unsigned long long)((double)P.nnz * mark_pct / 100.0);
  // dirty-filtered rounds with at most this many row tasks run inside the engine (BP_DF_LOCAL;
  // C2: 0 -> 5.63, 1000 -> 5.74, 3000 -> 5.57, 10000 -> 5.60 ms)
  static const int df_local_env = getenv("BP_DF_LOCAL") ? atoi(getenv("BP_DF_LOCAL")) : 3000;
  int df_local = df_local_env;
  void* args[]   = {&d, &st, &l, &md, &ff, &sb, &dense_thr, &stp, &ext, &resume, &mark_max, &df_local};
  BP_CUDA(cudaEventRecord(P.ev0, s));
  BP_CUDA(cudaLaunchCooperativeKernel((void*)k_engine, P.grid_blocks, kThreads, args, sizeof(Smem), s));
  ++g_kernel_launches;
  // full rounds: the row phase runs in k_rows_full, then the engine resumes. Batches of such
  // round trips are enqueued without waiting (no-ops past the engine's end); the host only reads
  // need_full between batches (1, 2, 4, 8 rounds).
  for (int batch = 1; ext; batch = std::min(2 * batch, 8)) {
    resume = 1;
    for (int b = 0; b < batch; ++b) {
      k_rows_full<<<P.f2_blocks, kThreads, kRowsSmem, s>>>(d, st, l, split_sell);
      if (split_sell) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id                                         = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.gridDim                                      = dim3(P.sell_blocks);
        cfg.blockDim                                     = dim3(kThreads);
        cfg.dynamicSmemBytes                             = 0;
        cfg.stream                                       = s;
        cfg.attrs                                        = at;
        cfg.numAttrs                                     = 1;
        BP_CUDA(cudaLaunchKernelEx(&cfg, k_rows_sell, d, st, l));
        ++g_kernel_launches;
      }
      if (P.n_cpiece && !split_sell)  // (with split SELL they run at the end of k_rows_sell)
        k_cand_pieces<<<std::min(P.f2_blocks, (P.n_cpiece + kWarps - 1) / kWarps), kThreads,
                        sizeof(Smem), s>>>(d, st, l);
      BP_CUDA(cudaGetLastError());
      BP_CUDA(cudaLaunchCooperativeKernel((void*)k_engine, P.grid_blocks, kThreads, args, sizeof(Smem), s));
      g_kernel_launches += P.n_cpiece && !split_sell ? 3 : 2;
    }
    int h = 0;
    BP_CUDA(cudaMemcpyAsync(&h, &P.st.ctl->need_full, sizeof(int), cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaStreamSynchronize(s));
    if (!h) break;
  }
  BP_CUDA(cudaEventRecord(P.ev1, s));
  RunResult r{0, 0, 0, 0};
  if (mode == MODE_PROPAGATE) {
    int h[5];
    BP_CUDA(cudaMemcpyAsync(h, &P.st.ctl->status, sizeof(h), cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaStreamSynchronize(s));
    r.status   = h[0];
    r.rounds   = h[1];
    r.crossed  = h[2];
    r.fixpoint = h[4];
  } else {
    BP_CUDA(cudaStreamSynchronize(s));
  }
  if (P.st.dbg) {
    unsigned long long h[24];
    BP_CUDA(cudaMemcpy(h, P.st.dbg, sizeof(h), cudaMemcpyDeviceToHost));
    const char* nm[5] = {"heavy_fold", "sell_slice", "cand_piece", "heavy_stream", "group_fold"};
    for (int q = 0; q < 5; ++q)
      fprintf(stderr, "[bp dbg] %-10s n=%llu avg=%.1f us max=%.1f us total=%.1f warp-ms\n", nm[q],
              h[3 * q + 2], h[3 * q + 2] ? h[3 * q] / 1965.0 / h[3 * q + 2] : 0.0,
              h[3 * q + 1] / 1965.0, h[3 * q] / 1965.0 / 1e3);
    fprintf(stderr, "[bp dbg] sell rows %llu, past the row gate %llu, pass-2 entries %llu, past the entry gate %llu\n",
            h[16], h[17], h[18], h[19]);
    BP_CUDA(cudaMemset(P.st.dbg, 0, sizeof(h)));
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
  std::vector<int2> pc, fd;
  for (int j = 0; j < nrows; ++j) {
    const int k = rows[j];
    const int L = P.h_row_start[k + 1] - P.h_row_start[k];
    if (L <= kShortNnz) {
      sr.push_back(k);
    } else {
      for (int q = 0; q * kSumSegment < L; ++q) fd.push_back(make_int2(k, q));
      if (L > kHeavyFold) {
        const int p0 = P.h_hpiece[k];
        for (int q = 0; q * kPiece < L; ++q) pc.push_back(make_int2(p0 + q, 0));
      }
    }
  }
  DevState& S = P.st;
  if (!sr.empty())
    BP_CUDA(cudaMemcpyAsync(S.drow_s[1], sr.data(), sr.size() * 4, cudaMemcpyHostToDevice, s));
  if (!pc.empty())
    BP_CUDA(cudaMemcpyAsync(S.dpiece[1], pc.data(), pc.size() * 8, cudaMemcpyHostToDevice, s));
  if (!fd.empty())
    BP_CUDA(cudaMemcpyAsync(S.dfold[1], fd.data(), fd.size() * 8, cudaMemcpyHostToDevice, s));
  int cnt[4] = {(int)sr.size(), (int)pc.size(), (int)fd.size(), nrows};
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

void stage_changed(Problem& P, const int* vars, int nvars, cudaStream_t s)
{
  std::vector<int2> ct;
  for (int j = 0; j < nvars; ++j) {
    const int i = vars[j];
    const int L = P.h_col_start[i + 1] - P.h_col_start[i];
    if (L > kTile)
      for (int q = 0; q * kTile < L; ++q) ct.push_back(make_int2(i, q));
  }
  DevState& S = P.st;
  if (nvars)
    BP_CUDA(cudaMemcpyAsync(S.changed, vars, sizeof(int) * nvars, cudaMemcpyHostToDevice, s));
  if (!ct.empty())
    BP_CUDA(cudaMemcpyAsync(S.ctask, ct.data(), ct.size() * 8, cudaMemcpyHostToDevice, s));
  const int nc = nvars, nt = (int)ct.size();
  BP_CUDA(cudaMemcpyAsync(&S.ctl->par[0].n_changed, &nc, sizeof(int), cudaMemcpyHostToDevice, s));
  BP_CUDA(cudaMemcpyAsync(&S.ctl->par[0].n_ctask, &nt, sizeof(int), cudaMemcpyHostToDevice, s));
  BP_CUDA(cudaStreamSynchronize(s));
}

}  // namespace bp
