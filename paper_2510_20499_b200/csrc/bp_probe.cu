// Batched double probing (probing cache) for sm_100a.
//
// Reference: probing.hpp:194-238 (probe_branch / probe_variable) and :243-281 (build_cache).
// Every branch of every candidate is an independent `propagate` from the root bounds with one
// variable narrowed. Instead of one O(n) bounds copy per branch (probing.hpp:201), each warp runs
// one branch against *overlays* in shared memory over the shared, read-only root state:
//   bounds overlay    var -> (lo, up)     for the variables this branch tightened
//   activity overlay  row -> activity     for the rows this branch recomputed
// Everything not in an overlay is read from the root (bounds, and the root's row activities).
//
// Exactness: a branch starts from the frontier rows(v) instead of a full first round. That is
// bit-identical to the reference only when the root is a certified fixpoint (its own full round
// changes nothing) — SURVEY §8a A12 lemma; the host certifies it with the engine and otherwise
// runs every branch through the full engine (bp_problem's propagate) instead. Inside a branch
// the rounds are the reference's: Jacobi tightening of the dirty vars (all reads before any
// write), activities in fixed 16384-entry segments, std::min/max folds in CSC order, the
// thresholds of counts_as_change, the 64-round cap.
// Branches whose frontier exceeds the overlay capacities are flagged and re-run on the engine.
#include <algorithm>
#include <cmath>

#include "bp_engine.cuh"
#include "bp_probe.cuh"

namespace bp {

namespace {

constexpr unsigned FULL  = 0xffffffffu;
#ifndef PB_WARPS_V
#define PB_WARPS_V 4
#endif
constexpr int PB_WARPS   = PB_WARPS_V;  // warps per block
#ifndef PB_CLAIM
#define PB_CLAIM 1  // C3 kernel: 1 -> 25.17 ms, 4 -> 25.69, 16 -> 26.37 (claims are not the bound)
#endif
constexpr int PB_BCAP    = 128;   // bounds overlay slots (power of 2)
constexpr int PB_ACAP    = 128;   // activity overlay slots (power of 2)
#ifndef PB_RCAP_V
#define PB_RCAP_V 256
#endif
constexpr int PB_RCAP    = PB_RCAP_V;   // dirty rows per round
#ifndef PB_VCAP_V
#define PB_VCAP_V 512
#endif
constexpr int PB_VCAP    = PB_VCAP_V;   // dirty vars per round
#ifndef PB_SCAP_V
#define PB_SCAP_V 1024
#endif
constexpr int PB_SCAP    = PB_SCAP_V;  // dedup hash set (power of 2)
constexpr int PB_CCAP    = 128;   // changed vars per round
#ifndef PB_LANEROW_V
#define PB_LANEROW_V 64
#endif
constexpr int PB_LANEROW = PB_LANEROW_V;  // rows / columns up to this length are handled by one lane
constexpr int PB_LONGROW = 4096;  // a dirty row longer than this sends the branch to the engine

struct PWarp {
  int bkey[PB_BCAP];  // var + 1, 0 = empty
  double2 bval[PB_BCAP];
  int akey[PB_ACAP];  // row + 1
  double amn[PB_ACAP], amx[PB_ACAP];
  int ainf[PB_ACAP][2];
  int drow[PB_RCAP];
  int dvar[PB_VCAP];
  int set[PB_SCAP];
  int cvar[PB_CCAP];
  double2 cval[PB_CCAP];
  double stage[64];
  int off[33], st[32];  // flattened entry windows: exclusive offsets / first entry of 32 items
  int n_drow, n_dvar, n_chg, crossed, overflow;
};

struct PSmem {
  PWarp w[PB_WARPS];
};

__device__ __forceinline__ unsigned hsh(int x) { return (unsigned)x * 2654435761u; }

struct PCtx {
  const DevProblem& P;
  const ProbeRoot& R;
  const Limits& lim;
  PWarp& w;
  int lane;
};

// Overlay slot of var v, or -1 (then the root value applies).
__device__ __forceinline__ int bfind(PCtx& c, int v)
{
  unsigned s = hsh(v) & (PB_BCAP - 1);
  for (int probe = 0; probe < PB_BCAP; ++probe) {
    const int k = c.w.bkey[s];
    if (k == v + 1) return (int)s;
    if (k == 0) break;
    s = (s + 1) & (PB_BCAP - 1);
  }
  return -1;
}

// Overlay slot of row k's activity, or -1 (then the root record applies).
__device__ __forceinline__ int afind(PCtx& c, int k)
{
  unsigned s = hsh(k) & (PB_ACAP - 1);
  for (int probe = 0; probe < PB_ACAP; ++probe) {
    const int key = c.w.akey[s];
    if (key == k + 1) return (int)s;
    if (key == 0) break;
    s = (s + 1) & (PB_ACAP - 1);
  }
  return -1;
}

__device__ __forceinline__ double2 bget(PCtx& c, int v)
{
  unsigned s = hsh(v) & (PB_BCAP - 1);
  for (int probe = 0; probe < PB_BCAP; ++probe) {
    const int k = c.w.bkey[s];
    if (k == v + 1) return c.w.bval[s];
    if (k == 0) break;
    s = (s + 1) & (PB_BCAP - 1);
  }
  return c.R.bounds[v];
}

// Insert / update by a single lane per key (distinct keys across lanes). false on overflow.
__device__ __forceinline__ bool bset(PCtx& c, int v, double2 b)
{
  unsigned s = hsh(v) & (PB_BCAP - 1);
  for (int probe = 0; probe < PB_BCAP / 2; ++probe) {  // keep the load factor <= 1/2
    const int k = atomicCAS(&c.w.bkey[s], 0, v + 1);
    if (k == 0 || k == v + 1) {
      c.w.bval[s] = b;
      return true;
    }
    s = (s + 1) & (PB_BCAP - 1);
  }
  return false;
}

__device__ __forceinline__ void aget(PCtx& c, int k, double& mnf, int& nmn, double& mxf, int& nmx,
                                     double& g, double& h)
{
  unsigned s = hsh(k) & (PB_ACAP - 1);
  for (int probe = 0; probe < PB_ACAP; ++probe) {
    const int key = c.w.akey[s];
    if (key == k + 1) {
      mnf = c.w.amn[s];
      mxf = c.w.amx[s];
      nmn = c.w.ainf[s][0];
      nmx = c.w.ainf[s][1];
      const double2 cb = __ldg(&c.P.cons[k]);
      g = cb.y;
      h = cb.x;
      return;
    }
    if (key == 0) break;
    s = (s + 1) & (PB_ACAP - 1);
  }
  const RowRec r = ld_rec(c.R.rec + k);
  decode_rec(r, c.R.aux, k, mnf, nmn, mxf, nmx);
  g = r.g;
  h = r.h;
}

__device__ __forceinline__ bool aset(PCtx& c, int k, double mnf, int nmn, double mxf, int nmx)
{
  unsigned s = hsh(k) & (PB_ACAP - 1);
  for (int probe = 0; probe < PB_ACAP / 2; ++probe) {
    const int key = atomicCAS(&c.w.akey[s], 0, k + 1);
    if (key == 0 || key == k + 1) {
      c.w.amn[s]     = mnf;
      c.w.amx[s]     = mxf;
      c.w.ainf[s][0] = nmn;
      c.w.ainf[s][1] = nmx;
      return true;
    }
    s = (s + 1) & (PB_ACAP - 1);
  }
  return false;
}

// Dedup set: returns true if x was newly inserted.
__device__ __forceinline__ bool set_insert(PWarp& w, int x, bool& full)
{
  unsigned s = hsh(x) & (PB_SCAP - 1);
  for (int probe = 0; probe < PB_SCAP / 2; ++probe) {
    const int k = atomicCAS(&w.set[s], 0, x + 1);
    if (k == 0) return true;
    if (k == x + 1) return false;
    s = (s + 1) & (PB_SCAP - 1);
  }
  full = true;
  return false;
}

__device__ __forceinline__ void set_clear(PWarp& w, int lane)
{
  for (int j = lane; j < PB_SCAP; j += 32) w.set[j] = 0;
  __syncwarp();
}

// Activity of one row of <= PB_LANEROW entries (a single 16384-entry segment) in reference order,
// four entries' index loads and bound gathers in flight at a time.
#ifndef PB_U_V
#define PB_U_V 3
#endif
constexpr int PB_U = PB_U_V;
__device__ void row_act_lane(PCtx& c, int k, double& smn, int& imn, double& smx, int& imx)
{
  const int rs = __ldg(c.P.row_start + k), re = __ldg(c.P.row_start + k + 1);
  double pmn = 0.0, pmx = 0.0;
  imn = imx = 0;
  for (int e0 = rs; e0 < re; e0 += PB_U) {
    int col[PB_U];
    double a[PB_U];
    double2 b[PB_U];
#pragma unroll
    for (int u = 0; u < PB_U; ++u) {
      col[u] = e0 + u < re ? __ldg(c.P.row_col + e0 + u) : -1;
      a[u]   = e0 + u < re ? __ldg(c.P.row_val + e0 + u) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PB_U; ++u) {
      const int sl = col[u] >= 0 ? bfind(c, col[u]) : -1;
      b[u]         = sl >= 0 ? c.w.bval[sl] : (col[u] >= 0 ? c.R.bounds[col[u]] : make_double2(0.0, 0.0));
    }
#pragma unroll
    for (int u = 0; u < PB_U; ++u) {
      if (col[u] < 0) break;
      double cm, cx;
      int i1, i2;
      contrib(a[u], b[u].x, b[u].y, cm, cx, i1, i2);
      pmn = __dadd_rn(pmn, cm);
      pmx = __dadd_rn(pmx, cx);
      imn += i1;
      imx += i2;
    }
  }
  smn = __dadd_rn(0.0, pmn);  // the segment total onto the row total (propagation.hpp:182-188)
  smx = __dadd_rn(0.0, pmx);
}

// Same for a long row, warp-cooperatively (lanes gather, lanes 0/1 fold).
__device__ void row_act_warp(PCtx& c, int k, double& smn, int& imn, double& smx, int& imx)
{
  const int rs = __ldg(c.P.row_start + k), L = __ldg(c.P.row_start + k + 1) - rs;
  double tot = 0.0, part = 0.0;
  int cmn = 0, cmx = 0;
  for (int base = 0; base < L; base += 32) {
    if (base > 0 && (base % kSumSegment) == 0) {
      tot  = __dadd_rn(tot, part);
      part = 0.0;
    }
    const int j = base + c.lane;
    double cm = 0.0, cx = 0.0;
    if (j < L) {
      const double2 b = bget(c, __ldg(c.P.row_col + rs + j));
      int i1, i2;
      contrib(__ldg(c.P.row_val + rs + j), b.x, b.y, cm, cx, i1, i2);
      cmn += i1;
      cmx += i2;
    }
    c.w.stage[c.lane]      = cm;
    c.w.stage[32 + c.lane] = cx;
    __syncwarp();
    if (c.lane < 2) {
      const int cnt = min(32, L - base);
      for (int q = 0; q < cnt; ++q) part = __dadd_rn(part, c.w.stage[32 * c.lane + q]);
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

// Candidate fold of variable i over its column (lane-sequential, CSC order), four entries' row
// records in flight at a time.
__device__ void col_fold_lane(PCtx& c, int i, double lo, double up, bool integer, double& nl,
                              double& nu)
{
  nl = lo;
  nu = up;
  const int cs = __ldg(c.P.col_start + i), ce = __ldg(c.P.col_start + i + 1);
  for (int e0 = cs; e0 < ce; e0 += PB_U) {
    int k[PB_U], sl[PB_U];
    double a[PB_U];
    RowRec r[PB_U];
#pragma unroll
    for (int u = 0; u < PB_U; ++u) {
      k[u] = e0 + u < ce ? __ldg(c.P.col_row + e0 + u) : -1;
      a[u] = e0 + u < ce ? __ldg(c.P.col_val + e0 + u) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PB_U; ++u) {
      sl[u] = k[u] >= 0 ? afind(c, k[u]) : -1;
      if (k[u] >= 0) r[u] = ld_rec(c.R.rec + k[u]);  // g / h, and the root activity if no overlay
    }
#pragma unroll
    for (int u = 0; u < PB_U; ++u) {
      if (k[u] < 0) break;
      double mnf, mxf, cl, cu;
      int nmn, nmx;
      if (sl[u] >= 0) {
        mnf = c.w.amn[sl[u]];
        mxf = c.w.amx[sl[u]];
        nmn = c.w.ainf[sl[u]][0];
        nmx = c.w.ainf[sl[u]][1];
      } else {
        decode_rec(r[u], c.R.aux, k[u], mnf, nmn, mxf, nmx);
      }
      cand_explicit(lo, up, integer, a[u], mnf, nmn, mxf, nmx, r[u].g, r[u].h, cl, cu);
      if (cu < nu) nu = cu;
      if (nl < cl) nl = cl;
    }
  }
}

// Warp-cooperative version: lexicographic (value, CSC position) reduction.
__device__ void col_fold_warp(PCtx& c, int i, double lo, double up, bool integer, double& nl,
                              double& nu)
{
  const int cs = __ldg(c.P.col_start + i), ce = __ldg(c.P.col_start + i + 1);
  Fold f{lo, -1, up, -1};
  for (int e = cs + c.lane; e < ce; e += 32) {
    const int k = __ldg(c.P.col_row + e);
    double mnf, mxf, g, h, cl, cu;
    int nmn, nmx;
    aget(c, k, mnf, nmn, mxf, nmx, g, h);
    cand_explicit(lo, up, integer, __ldg(c.P.col_val + e), mnf, nmn, mxf, nmx, g, h, cl, cu);
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

// propagation.hpp:354-369 on explicit values; returns 1/0/-1 and the bounds to keep.
__device__ __forceinline__ int decide(double lo, double up, double nl, double nu, bool integer,
                                      const Limits& lim, double2& out)
{
  double2 b = make_double2(lo, up);
  const int r = finish_var(&b, lo, up, nl, nu, integer, lim);
  out = b;
  return r;
}

__device__ __forceinline__ int warp_incl_scan_p(int v, int lane)
{
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Calls f(e) for every entry e of the ranges [start[it], start[it + 1]) of items[0..cnt), the
// (item, entry) pairs flattened across the warp 32 items at a time: two dependent loads per
// window instead of two per item.
template <class F>
__device__ __forceinline__ void for_each_entry(PCtx& c, const int* items, int cnt, const int* start,
                                               F f)
{
  const int lane = c.lane;
  for (int w0 = 0; w0 < cnt; w0 += 32) {
    const int j = w0 + lane;
    int s0 = 0, len = 0;
    if (j < cnt) {
      const int it = items[j];
      s0  = __ldg(start + it);
      len = __ldg(start + it + 1) - s0;
    }
    const int incl  = warp_incl_scan_p(len, lane);
    const int total = __shfl_sync(FULL, incl, 31);
    c.w.off[lane]   = incl - len;
    c.w.st[lane]    = s0;
    if (lane == 0) c.w.off[32] = total;
    __syncwarp();
    for (int f0 = lane; f0 < total; f0 += 32) {
      int o = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1)
        if (c.w.off[o + step] <= f0) o += step;
      f(c.w.st[o] + (f0 - c.w.off[o]));
    }
    __syncwarp();
  }
}

// One probe branch (probing.hpp:194-219 + propagate) on this warp. Returns 0 feasible,
// 1 infeasible, 2 overflow (caller re-runs on the full engine).
__device__ __forceinline__ int probe_branch(PCtx& c, int v, double blo, double bup, unsigned long long (&wk)[5])
{
  PWarp& w = c.w;
  const int lane = c.lane;
  for (int j = lane; j < PB_BCAP; j += 32) w.bkey[j] = 0;
  for (int j = lane; j < PB_ACAP; j += 32) w.akey[j] = 0;
  if (lane == 0) {
    w.n_drow = w.n_dvar = w.n_chg = w.crossed = w.overflow = 0;
  }
  __syncwarp();
  const double2 rb = c.R.bounds[v];
  const double2 nb = make_double2(smax(rb.x, blo), smin(rb.y, bup));
  if (nb.x > nb.y) return 1;
  if (lane == 0) bset(c, v, nb);
  // the initial "changed" set is {v}
  if (lane == 0) {
    w.cvar[0] = v;
    w.n_chg   = 1;
  }
  __syncwarp();
  int rounds = 0;
  while (true) {
    // ---- frontier: rows(changed) -> drow, vars(drow) -> dvar
    set_clear(w, lane);
    bool full = false;
    if (lane == 0) w.n_drow = 0;
    __syncwarp();
    for_each_entry(c, w.cvar, w.n_chg, c.P.col_start, [&](int e) {
      const int k = __ldg(c.P.col_row + e);
      if (set_insert(w, k, full)) {
        const int pos = atomicAdd(&w.n_drow, 1);
        if (pos < PB_RCAP) w.drow[pos] = k;
        // its vars alone would exceed the overlays: overflow now instead of after the work
        if (__ldg(c.P.row_start + k + 1) - __ldg(c.P.row_start + k) > PB_LONGROW) full = true;
      }
    });
    __syncwarp();
    if (__any_sync(FULL, full) || w.n_drow > PB_RCAP) return 2;
    const int nr = w.n_drow;
    if (nr == 0) return 0;  // dirty_rows.empty(): done (propagation.hpp:481)
    if (rounds >= c.lim.max_rounds) return 0;
    set_clear(w, lane);
    if (lane == 0) w.n_dvar = 0;
    __syncwarp();
    for_each_entry(c, w.drow, nr, c.P.row_start, [&](int e) {
      const int i = __ldg(c.P.row_col + e);
      if (set_insert(w, i, full)) {
        const int pos = atomicAdd(&w.n_dvar, 1);
        if (pos < PB_VCAP) w.dvar[pos] = i;
      }
    });
    __syncwarp();
    if (__any_sync(FULL, full) || w.n_dvar > PB_VCAP) return 2;
    ++rounds;
    {  // work of this round (R, A, V, B): lane-strided lengths, reduced to lane 0
      unsigned long long a = 0, bsum = 0;
      for (int j = lane; j < nr; j += 32) a += __ldg(c.P.row_start + w.drow[j] + 1) - __ldg(c.P.row_start + w.drow[j]);
      for (int j = lane; j < w.n_dvar; j += 32) bsum += __ldg(c.P.col_start + w.dvar[j] + 1) - __ldg(c.P.col_start + w.dvar[j]);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(FULL, a, o);
        bsum += __shfl_xor_sync(FULL, bsum, o);
      }
      wk[0] += nr;
      wk[1] += a;
      wk[2] += w.n_dvar;
      wk[3] += bsum;
    }
    // ---- activities of the dirty rows
    // short rows one per lane; the long ones of each 32-row window warp-cooperatively
    bool ovf = false;
    for (int w0 = 0; w0 < nr; w0 += 32) {
      const int j  = w0 + lane;
      const int k  = j < nr ? w.drow[j] : -1;
      const bool lng = k >= 0 && __ldg(c.P.row_start + k + 1) - __ldg(c.P.row_start + k) > PB_LANEROW;
      if (k >= 0 && !lng) {
        double smn, smx;
        int imn, imx;
        row_act_lane(c, k, smn, imn, smx, imx);
        if (!aset(c, k, smn, imn, smx, imx)) ovf = true;
      }
      for (unsigned m = __ballot_sync(FULL, lng); m; m &= m - 1) {
        const int kk = __shfl_sync(FULL, k, __ffs(m) - 1);
        double smn, smx;
        int imn, imx;
        row_act_warp(c, kk, smn, imn, smx, imx);
        if (lane == 0 && !aset(c, kk, smn, imn, smx, imx)) ovf = true;
      }
    }
    __syncwarp();
    if (__any_sync(FULL, ovf)) return 2;
    // ---- Jacobi tightening of the dirty vars (all reads before any write)
    const int nv = w.n_dvar;
    if (lane == 0) w.n_chg = 0;
    __syncwarp();
    int crossed = 0;
    auto record = [&](int i, int r, const double2& out) {
      if (r < 0) crossed++;
      if (r > 0) {
        const int pos = atomicAdd(&w.n_chg, 1);
        if (pos < PB_CCAP) {
          w.cvar[pos] = i;
          w.cval[pos] = out;
        }
      }
    };
    // short columns one per lane; the long ones of each 32-var window warp-cooperatively
    for (int w0 = 0; w0 < nv; w0 += 32) {
      const int j = w0 + lane;
      const int i = j < nv ? w.dvar[j] : -1;
      const bool lng = i >= 0 && __ldg(c.P.col_start + i + 1) - __ldg(c.P.col_start + i) > PB_LANEROW;
      if (i >= 0 && !lng) {
        const double2 b    = bget(c, i);
        const bool integer = __ldg(c.P.is_int + i) != 0;
        double nl, nu;
        col_fold_lane(c, i, b.x, b.y, integer, nl, nu);
        double2 out;
        record(i, decide(b.x, b.y, nl, nu, integer, c.lim, out), out);
      }
      for (unsigned m = __ballot_sync(FULL, lng); m; m &= m - 1) {
        const int ii       = __shfl_sync(FULL, i, __ffs(m) - 1);
        const double2 b    = bget(c, ii);
        const bool integer = __ldg(c.P.is_int + ii) != 0;
        double nl, nu;
        col_fold_warp(c, ii, b.x, b.y, integer, nl, nu);
        if (lane == 0) {
          double2 out;
          record(ii, decide(b.x, b.y, nl, nu, integer, c.lim, out), out);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int o = 16; o; o >>= 1) crossed += __shfl_xor_sync(FULL, crossed, o);
    if (crossed > 0) return 1;        // propagation.hpp:448-452
    const int nc = w.n_chg;
    wk[4] += nc;
    if (nc > PB_CCAP) return 2;
    if (nc == 0) return 0;            // fixpoint (propagation.hpp:453)
    bool bovf = false;
    for (int j = lane; j < nc; j += 32)
      if (!bset(c, w.cvar[j], w.cval[j])) bovf = true;
    __syncwarp();
    if (__any_sync(FULL, bovf)) return 2;
    if (rounds >= c.lim.max_rounds) return 0;
  }
}

__global__ void __launch_bounds__(PB_WARPS * 32, 1)
    k_probe(DevProblem P, ProbeRoot R, ProbeBatch B, Limits lim)
{
  extern __shared__ __align__(16) unsigned char dyn[];
  PSmem& sm      = *reinterpret_cast<PSmem*>(dyn);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PCtx c{P, R, lim, sm.w[warp], lane};
  unsigned long long wk[5] = {0, 0, 0, 0, 0};  // warp-uniform work counters
  for (;;) {  // PB_CLAIM branches per claim of the shared cursor
    int t0 = 0;
    if (lane == 0) t0 = atomicAdd(B.cursor, PB_CLAIM);
    t0 = __shfl_sync(FULL, t0, 0);
    if (t0 >= B.n_task) break;
    const int t1 = min(t0 + PB_CLAIM, B.n_task);
    for (int t = t0; t < t1; ++t) {
    const int v      = B.var[t];
    unsigned long long bw[5] = {0, 0, 0, 0, 0};
    const int status = probe_branch(c, v, B.lo[t], B.up[t], bw);
    if (status != 2)  // overflowing branches are counted by the kernel that reruns them
      for (int q = 0; q < 5; ++q) wk[q] += bw[q];
    // deltas: overlay entries differing from the root, ascending by var (probing.hpp:213-217)
    PWarp& w = c.w;
    int cnt  = 0;
    if (status == 0) {
      for (int j = lane; j < PB_BCAP; j += 32) {
        const int key = w.bkey[j];
        bool d        = false;
        if (key) {
          const double2 b = w.bval[j], r = R.bounds[key - 1];
          d = (b.x != r.x) || (b.y != r.y);
        }
        cnt += d;
        if (!d) w.bkey[j] = 0;  // keep only the deltas in the table
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
    }
    __syncwarp();
    long long base = 0;
    if (lane == 0) {
      if (cnt) base = (long long)atomicAdd(B.pool_cursor, (unsigned long long)cnt);
      B.status[t] = status;
      B.dcount[t] = cnt;
      B.doff[t]   = base;
    }
    base = __shfl_sync(FULL, base, 0);
    if (status == 0 && cnt) {
      if (base + cnt > B.pool_cap) {
        if (lane == 0) B.status[t] = 3;  // pool exhausted: host grows it and retries
      } else {
        for (int j = lane; j < PB_BCAP; j += 32) {
          const int key = w.bkey[j];
          if (!key) continue;
          int rank = 0;  // position among the deltas by ascending var
          for (int q = 0; q < PB_BCAP; ++q) {
            const int o = w.bkey[q];
            rank += (o != 0 && o < key);
          }
          B.pvar[base + rank] = key - 1;
          B.plo[base + rank]  = w.bval[j].x;
          B.pup[base + rank]  = w.bval[j].y;
        }
      }
    }
    __syncwarp();
    }
  }
  if (lane == 0 && B.work)
    for (int q = 0; q < 5; ++q)
      if (wk[q]) atomicAdd(B.work + q, wk[q]);
}

}  // namespace

void probe_launch(Problem& Pr, const ProbeRoot& R, ProbeBatch& B, const Limits& lim, cudaStream_t s)
{
  // the attribute is per device (problems may live on several GPUs): set it on every launch's
  // device, next to the occupancy query (a cheap driver call)
  BP_CUDA(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PSmem)));
  int dev_sms = 0, per_sm = 0;
  BP_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, Pr.device));
  BP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_probe, PB_WARPS * 32, sizeof(PSmem)));
  const int blocks = dev_sms * std::max(per_sm, 1);
  k_probe<<<blocks, PB_WARPS * 32, sizeof(PSmem), s>>>(Pr.dev(), R, B, lim);
  BP_CUDA(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace bp
