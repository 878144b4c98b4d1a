// PDHG sparse matrix-vector products (lp.hpp:74-102) and the PDHG inner iteration (lp.hpp:315-340)
// on the device, bit-identical to the reference.
//
// spmv_rows: out[k] = sum over the row's entries of a * x[col], summed like the reference: within
// each 16384-entry segment left to right from 0.0 (`part += a * x`, separately rounded product, no
// FMA), segment partials added in order onto 0.0 (`total += part`). spmv_cols is the same over the
// CSC. Rows (columns) of <= kLpLane entries sit in SELL-32 slices (thread per item, coalesced
// index / value loads, four entries' gathers in flight); longer ones are split into 16384-entry
// segments, one warp per segment: the lanes gather 256 products into shared memory while lane 0
// runs the sequential sum over the previous 256 (double buffered), then the segment partials are
// combined in order.
//
// The PDHG iteration adds one elementwise kernel after each product: the dual step
// (y = v - sigma * clamp(v / sigma, row bounds), v = y + sigma * A x_bar) and the primal step
// (x_next = clamp(x - tau (c + A'y)), x_bar = 2 x_next - x) fused with the running sums
// x_sum += x, y_sum += y -- each vector is read and written once per half-step.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bp.h"
#include "bp_capi_internal.h"
#include "bp_engine.cuh"

namespace bp {
namespace {

constexpr int kLpLane    = 64;      // rows / columns up to this length: one thread each
constexpr int kLpSeg     = 16384;   // problem.hpp:274 kSumSegment
#ifndef LP_CHUNK
#define LP_CHUNK 512
#endif
#ifndef LP_SELL_U
#define LP_SELL_U 4
#endif
constexpr int kLpChunk   = LP_CHUNK;  // products staged per warp step
constexpr int kLpSellU   = LP_SELL_U; // SELL entries in flight per lane
constexpr int kLpThreads = 256;

__device__ __forceinline__ double lp_clamp(double v, double lo, double hi)
{
  return v < lo ? lo : (v > hi ? hi : v);  // common.hpp clamp: std::max(lo, std::min(v, hi))
}

// Short rows / columns in SELL-32 slices (sorted by length, 32 per slice, entry j of lane i at
// base + 32 j + i): thread per item, coalesced index / value loads, four entries' gathers in
// flight, the sequential single-segment sum in registers.
__global__ void k_spmv_sell(int nslice, const int* sbase, const int* sitem, const int* sidx,
                            const double* sval, const double* x, double* out)
{
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int sl = gw; sl < nslice; sl += nw) {
    const int b0 = __ldg(sbase + sl), Lm = (__ldg(sbase + sl + 1) - b0) >> 5;
    const int it = __ldg(sitem + 32 * sl + lane);
    const int* ip    = sidx + b0 + lane;
    const double* vp = sval + b0 + lane;
    double part = 0.0;
    for (int j = 0; j < Lm; j += kLpSellU) {
      int c[kLpSellU];
      double a[kLpSellU], xv[kLpSellU];
#pragma unroll
      for (int u = 0; u < kLpSellU; ++u) {
        c[u] = j + u < Lm ? __ldg(ip + 32 * (j + u)) : -1;
        a[u] = j + u < Lm ? __ldg(vp + 32 * (j + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kLpSellU; ++u) xv[u] = c[u] >= 0 ? x[c[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < kLpSellU; ++u)
        if (c[u] >= 0) part = __dadd_rn(part, __dmul_rn(a[u], xv[u]));  // padding follows the row
    }
    if (it >= 0) out[it] = __dadd_rn(0.0, part);
  }
}

// Sequential left-to-right sum of src[0..cnt) onto acc with the next eight shared-memory values
// loaded while the current eight are added (the chain runs at the DADD latency, not the load's).
__device__ __forceinline__ double lp_fold_seq(const double* src, int cnt, double acc)
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

// One 16384-entry segment of a long row / column per warp: partial sum into seg_out[task]. The
// products of chunk j + 1 are loaded into registers while lane 0 runs the sequential sum over
// chunk j from shared memory, then staged (the loads overlap the DADD chain).
__global__ void __launch_bounds__(kLpThreads)
    k_spmv_segments(const int* start, const int* idx, const double* val, const double* x,
                    const int2* tasks, const int* slot, int ntask, double* seg_out)
{
  __shared__ __align__(16) double buf[kLpThreads / 32][kLpChunk];
  constexpr int PL = kLpChunk / 32;  // products per lane per chunk
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * (kLpThreads / 32) + wib, nw = gridDim.x * (kLpThreads / 32);
  for (int t = gw; t < ntask; t += nw) {
    const int2 tk = tasks[t];  // (item, segment), longest first
    const int s0  = __ldg(start + tk.x) + tk.y * kLpSeg;
    const int s1  = min(__ldg(start + tk.x + 1), s0 + kLpSeg);
    double part   = 0.0;
    double pr[PL];
    auto load = [&](int b0) {
#pragma unroll
      for (int h = 0; h < PL; ++h) {
        const int e = b0 + h * 32 + lane;
        pr[h]       = e < s1 ? __dmul_rn(__ldg(val + e), x[__ldg(idx + e)]) : 0.0;
      }
    };
    load(s0);
    for (int b0 = s0; b0 < s1; b0 += kLpChunk) {
#pragma unroll
      for (int h = 0; h < PL; ++h) buf[wib][h * 32 + lane] = pr[h];
      __syncwarp();
      load(b0 + kLpChunk);  // in flight during the fold below
      if (lane == 0) part = lp_fold_seq(buf[wib], min(kLpChunk, s1 - b0), part);
      __syncwarp();
    }
    if (lane == 0) seg_out[slot[t]] = part;
  }
}

// total = ((0.0 + p0) + p1) + ... over each long item's segments, in order.
__global__ void k_spmv_combine(const int* long_items, const int* seg_first, int nlong,
                               const double* seg_out, double* out)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nlong; j += gridDim.x * blockDim.x) {
    double total = 0.0;
    for (int q = seg_first[j]; q < seg_first[j + 1]; ++q) total = __dadd_rn(total, seg_out[q]);
    out[long_items[j]] = total;
  }
}

// lp.hpp:319-323: y = v - sigma * clamp(v / sigma, lo, up), v = y + sigma * ax.
__global__ void k_pdhg_dual(int m, const double* ax, const double* lo, const double* up, double sigma,
                            double* y)
{
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
    const double v    = __dadd_rn(y[k], __dmul_rn(sigma, ax[k]));
    const double proj = lp_clamp(__ddiv_rn(v, sigma), lo[k], up[k]);
    y[k]              = __dsub_rn(v, __dmul_rn(sigma, proj));
  }
}

// lp.hpp:327-339: x_next = clamp(x - tau (c + aty)), x_bar = 2 x_next - x, x = x_next, then the
// running sums x_sum += x, y_sum += y.
__global__ void k_pdhg_primal(int n, int m, const double* aty, const double* c, const double* lo,
                              const double* up, double tau, double* x, double* x_bar, double* x_sum,
                              const double* y, double* y_sum)
{
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v  = __dsub_rn(x[i], __dmul_rn(tau, __dadd_rn(c[i], aty[i])));
    const double xn = lp_clamp(v, lo[i], up[i]);
    x_bar[i]        = __dsub_rn(__dmul_rn(2.0, xn), x[i]);
    x[i]            = xn;
    x_sum[i]        = __dadd_rn(x_sum[i], xn);
  }
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride)
    y_sum[k] = __dadd_rn(y_sum[k], y[k]);
}

// ---- KKT scoring (lp.hpp:134-200) ------------------------------------------------------------
// The maxima are order-independent (exact); the two objective sums are compensated: each thread
// and block accumulates a double-double (TwoSum), blocks are combined in a fixed order, so the
// result is the exact sum rounded once -- the reference's Neumaier sum agrees with it to a few ulps.
struct DD {
  double hi, lo;
};
__device__ __forceinline__ void dd_add(DD& a, double x)
{
  const double s = __dadd_rn(a.hi, x);
  const double bb = __dsub_rn(s, a.hi);
  const double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(x, bb));
  a.hi = s;
  a.lo = __dadd_rn(a.lo, err);
}
__device__ __forceinline__ void dd_merge(DD& a, const DD& b)
{
  dd_add(a, b.hi);
  a.lo = __dadd_rn(a.lo, b.lo);
}
__device__ __forceinline__ void max_u64(unsigned long long* p, double v)  // v >= +0.0
{
  atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

constexpr int kKktThreads = 256;
// stats: [0] primal_res, [1] rhs_scale, [2] obj_scale, [3] x_norm, [4] dual_res (u64 bit patterns)
__global__ void __launch_bounds__(kKktThreads)
    k_kkt(int n, int m, const double* x, const double* y, const double* ax, const double* aty,
          const double* obj, const double* rlo, const double* rup, const double* vlo,
          const double* vup, unsigned long long* stats, DD* part)
{
  __shared__ DD sp[kKktThreads], sd[kKktThreads];
  double pres = 0.0, rsc = 0.0, osc = 0.0, xn = 0.0, dres = 0.0;
  DD po{0.0, 0.0}, dobj{0.0, 0.0};
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int k = tid; k < m; k += nt) {  // lp.hpp:143-155
    double v = 0.0;
    if (isfinite(rup[k])) {
      const double d = __dsub_rn(ax[k], rup[k]);
      v              = (v < d) ? d : v;
      rsc            = fmax(rsc, fabs(rup[k]));
    }
    if (isfinite(rlo[k])) {
      const double d = __dsub_rn(rlo[k], ax[k]);
      v              = (v < d) ? d : v;
      rsc            = fmax(rsc, fabs(rlo[k]));
    }
    pres = fmax(pres, v);
    const double yk = y[k];  // lp.hpp:181-196
    if (yk > 0.0) {
      if (isfinite(rup[k])) dd_add(dobj, __dmul_rn(-yk, rup[k]));
      else dres = fmax(dres, yk);
    } else if (yk < 0.0) {
      if (isfinite(rlo[k])) dd_add(dobj, __dmul_rn(-yk, rlo[k]));
      else dres = fmax(dres, -yk);
    }
  }
  for (int i = tid; i < n; i += nt) {  // lp.hpp:157-176
    dd_add(po, __dmul_rn(obj[i], x[i]));
    osc = fmax(osc, fabs(obj[i]));
    xn  = fmax(xn, fabs(x[i]));
    const double r = __dadd_rn(obj[i], aty[i]);
    double viol = 0.0, term = 0.0;
    if (r > 0.0) {
      if (isfinite(vlo[i])) term = __dmul_rn(r, vlo[i]);
      else viol = r;
    } else if (r < 0.0) {
      if (isfinite(vup[i])) term = __dmul_rn(r, vup[i]);
      else viol = -r;
    }
    dres = fmax(dres, viol);
    dd_add(dobj, term);
  }
  // maxima of non-negative values (+0.0 at least): bit patterns order like the values
  max_u64(stats + 0, pres);
  max_u64(stats + 1, rsc);
  max_u64(stats + 2, osc);
  max_u64(stats + 3, xn);
  max_u64(stats + 4, dres);
  sp[threadIdx.x] = po;
  sd[threadIdx.x] = dobj;
  __syncthreads();
  if (threadIdx.x == 0) {  // fixed-order block combine
    DD a = sp[0], b = sd[0];
    for (int t = 1; t < blockDim.x; ++t) {
      dd_merge(a, sp[t]);
      dd_merge(b, sd[t]);
    }
    part[2 * blockIdx.x]     = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void k_kkt_final(int nblocks, const DD* part, double* sums)
{
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  DD a = part[0], b = part[1];
  for (int q = 1; q < nblocks; ++q) {
    dd_merge(a, part[2 * q]);
    dd_merge(b, part[2 * q + 1]);
  }
  sums[0] = __dadd_rn(a.hi, a.lo);
  sums[1] = __dadd_rn(b.hi, b.lo);
}

inline int nblk(long long n) { return (int)std::max(1ll, std::min(148ll * 16, (n + 255) / 256)); }

}  // namespace

// One matrix view (CSR or CSC) partitioned into short items and long-item segments.
struct LpView {
  int n_item = 0;
  DBuf<int> start, idx;
  DBuf<double> val;
  DBuf<int> long_items, seg_first;
  DBuf<int> sl_base, sl_item, sl_idx;
  DBuf<double> sl_val;
  int n_slice = 0;
  DBuf<int2> tasks;
  DBuf<int> task_slot;
  DBuf<double> seg_out;
  int n_long = 0, n_task = 0;

  void build(int n, const int* h_start, const int* h_idx, const double* h_val)
  {
    n_item = n;
    const long long nnz = h_start[n];
    start.upload(h_start, n + 1);
    idx.upload(h_idx, nnz);
    val.upload(h_val, nnz);
    std::vector<int> sh, lg, sf{0};
    std::vector<int2> tk;
    for (int i = 0; i < n; ++i) {
      const int L = h_start[i + 1] - h_start[i];
      if (L <= kLpLane) {
        sh.push_back(i);
      } else {
        lg.push_back(i);
        for (int q = 0; q * kLpSeg < L; ++q) tk.push_back(make_int2(i, q));
        sf.push_back((int)tk.size());  // segment outputs of item lg[j]: seg_out[sf[j] .. sf[j+1])
      }
    }
    // SELL-32 slices of the short items, longest first
    {
      std::vector<int> ord(sh);
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
        return h_start[a + 1] - h_start[a] > h_start[b + 1] - h_start[b];
      });
      std::vector<int> base{0}, item, sidx;
      std::vector<double> sval;
      for (size_t s0 = 0; s0 < ord.size(); s0 += 32) {
        const size_t cnt = std::min<size_t>(32, ord.size() - s0);
        const int Lm     = h_start[ord[s0] + 1] - h_start[ord[s0]];
        const size_t off = sidx.size();
        sidx.resize(off + 32 * (size_t)Lm, -1);
        sval.resize(off + 32 * (size_t)Lm, 0.0);
        for (size_t i = 0; i < 32; ++i) {
          item.push_back(i < cnt ? ord[s0 + i] : -1);
          if (i >= cnt) continue;
          const int it = ord[s0 + i];
          for (int e = h_start[it], j = 0; e < h_start[it + 1]; ++e, ++j) {
            sidx[off + 32 * (size_t)j + i] = h_idx[e];
            sval[off + 32 * (size_t)j + i] = h_val[e];
          }
        }
        base.push_back((int)sidx.size());
      }
      n_slice = (int)(base.size() - 1);
      sl_base.upload(base);
      sl_item.upload(item);
      sl_idx.upload(sidx);
      sl_val.upload(sval);
    }
    n_long  = (int)lg.size();
    n_task  = (int)tk.size();
    // launch order: longest segments first (the sequential sums are the critical path)
    std::vector<int> ord(tk.size());
    for (size_t t = 0; t < tk.size(); ++t) ord[t] = (int)t;
    auto seglen = [&](const int2& q) {
      return std::min(h_start[q.x + 1] - h_start[q.x] - q.y * kLpSeg, kLpSeg);
    };
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return seglen(tk[a]) > seglen(tk[b]); });
    std::vector<int2> tks(tk.size());
    for (size_t t = 0; t < tk.size(); ++t) tks[t] = tk[ord[t]];
    task_slot.upload(ord);
    long_items.upload(lg);
    seg_first.upload(sf);
    tasks.upload(tks);
    seg_out.alloc(std::max(n_task, 1));
  }

  void spmv(const double* x, double* out, cudaStream_t s)
  {
    if (n_slice)
      k_spmv_sell<<<nblk(32ll * n_slice), 256, 0, s>>>(n_slice, sl_base.p, sl_item.p, sl_idx.p,
                                                       sl_val.p, x, out);
    if (n_task) {
      k_spmv_segments<<<std::min(148 * 8, (n_task + kLpThreads / 32 - 1) / (kLpThreads / 32)), kLpThreads,
                        0, s>>>(start.p, idx.p, val.p, x, tasks.p, task_slot.p, n_task, seg_out.p);
      k_spmv_combine<<<nblk(n_long), 256, 0, s>>>(long_items.p, seg_first.p, n_long, seg_out.p, out);
    }
    BP_CUDA(cudaGetLastError());
    g_kernel_launches += (n_slice ? 1 : 0) + (n_task ? 2 : 0);
  }
};

}  // namespace bp

struct bp_lp {
  int device = 0;
  int n = 0, m = 0;
  bp::LpView rows, cols;
  bp::DBuf<double> obj, rlo, rup, vlo, vup;
  bp::DBuf<double> x, y, xbar, xsum, ysum, ax, aty, vin, vout;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  double last_ms = 0.0;
};

namespace {

template <class F>
int lguard(F&& f)
{
  try {
    f();
    return BP_OK;
  } catch (const std::invalid_argument& e) {
    bp_set_last_error(e.what());
    return BP_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    bp_set_last_error(e.what());
    return BP_ERR_OUT_OF_RANGE;
  } catch (const bp::cuda_error& e) {
    bp_set_last_error(e.what());
    return BP_ERR_CUDA;
  } catch (const std::exception& e) {
    bp_set_last_error(e.what());
    return BP_ERR_RUNTIME;
  }
}

void need(bool c, const char* msg)
{
  if (!c) throw std::invalid_argument(msg);
}

}  // namespace

extern "C" {

int bp_lp_create(const bp_lp_desc* d, int32_t device, bp_lp** out)
{
  return lguard([&] {
    need(d && out, "null argument");
    need(d->n_vars >= 0 && d->n_rows >= 0, "negative dimension");
    need(d->row_start && d->col_start, "missing CSR / CSC offsets");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw bp::cuda_error("no CUDA device available (the engine has no CPU fallback)");
    need(device >= 0 && device < ndev, "device index out of range");
    BP_CUDA(cudaSetDevice(device));
    auto L    = std::make_unique<bp_lp>();
    L->device = device;
    L->n      = d->n_vars;
    L->m      = d->n_rows;
    L->rows.build(d->n_rows, d->row_start, d->row_col, d->row_val);
    L->cols.build(d->n_vars, d->col_start, d->col_row, d->col_val);
    const int n = L->n, m = L->m;
    if (d->obj) L->obj.upload(d->obj, n);
    if (d->row_lower) L->rlo.upload(d->row_lower, m);
    if (d->row_upper) L->rup.upload(d->row_upper, m);
    if (d->var_lower) L->vlo.upload(d->var_lower, n);
    if (d->var_upper) L->vup.upload(d->var_upper, n);
    for (auto* b : {&L->x, &L->xbar, &L->xsum, &L->aty}) b->alloc(std::max(n, 1));
    for (auto* b : {&L->y, &L->ysum, &L->ax}) b->alloc(std::max(m, 1));
    L->vin.alloc(std::max(std::max(n, m), 1));
    L->vout.alloc(std::max(std::max(n, m), 1));
    BP_CUDA(cudaStreamCreateWithFlags(&L->s, cudaStreamNonBlocking));
    BP_CUDA(cudaEventCreate(&L->e0));
    BP_CUDA(cudaEventCreate(&L->e1));
    *out = L.release();
  });
}

int bp_lp_destroy(bp_lp* L)
{
  return lguard([&] {
    if (!L) return;
    cudaSetDevice(L->device);
    if (L->s) cudaStreamDestroy(L->s);
    if (L->e0) cudaEventDestroy(L->e0);
    if (L->e1) cudaEventDestroy(L->e1);
    delete L;
  });
}

int bp_lp_spmv_rows(bp_lp* L, const double* x, double* ax)
{
  return lguard([&] {
    need(L && x && ax, "null argument");
    BP_CUDA(cudaSetDevice(L->device));
    if (L->n) BP_CUDA(cudaMemcpyAsync(L->vin.p, x, sizeof(double) * L->n, cudaMemcpyHostToDevice, L->s));
    BP_CUDA(cudaEventRecord(L->e0, L->s));
    L->rows.spmv(L->vin.p, L->vout.p, L->s);
    BP_CUDA(cudaEventRecord(L->e1, L->s));
    if (L->m) BP_CUDA(cudaMemcpyAsync(ax, L->vout.p, sizeof(double) * L->m, cudaMemcpyDeviceToHost, L->s));
    BP_CUDA(cudaStreamSynchronize(L->s));
    float ms = 0.f;
    BP_CUDA(cudaEventElapsedTime(&ms, L->e0, L->e1));
    L->last_ms = ms;
  });
}

int bp_lp_spmv_cols(bp_lp* L, const double* y, double* aty)
{
  return lguard([&] {
    need(L && y && aty, "null argument");
    BP_CUDA(cudaSetDevice(L->device));
    if (L->m) BP_CUDA(cudaMemcpyAsync(L->vin.p, y, sizeof(double) * L->m, cudaMemcpyHostToDevice, L->s));
    BP_CUDA(cudaEventRecord(L->e0, L->s));
    L->cols.spmv(L->vin.p, L->vout.p, L->s);
    BP_CUDA(cudaEventRecord(L->e1, L->s));
    if (L->n) BP_CUDA(cudaMemcpyAsync(aty, L->vout.p, sizeof(double) * L->n, cudaMemcpyDeviceToHost, L->s));
    BP_CUDA(cudaStreamSynchronize(L->s));
    float ms = 0.f;
    BP_CUDA(cudaEventElapsedTime(&ms, L->e0, L->e1));
    L->last_ms = ms;
  });
}

int bp_lp_pdhg_iterate(bp_lp* L, double* x, double* y, double* x_bar, double* x_sum, double* y_sum,
                       double tau, double sigma, int32_t iters)
{
  return lguard([&] {
    need(L && x && y && x_bar && x_sum && y_sum, "null argument");
    need(iters >= 0, "negative iteration count");
    // empty dimensions upload nothing (null device arrays): only non-empty ones must be present
    need((L->n == 0 || (L->obj.p && L->vlo.p && L->vup.p)) && (L->m == 0 || (L->rlo.p && L->rup.p)),
         "PDHG needs obj and row / variable bounds");
    BP_CUDA(cudaSetDevice(L->device));
    const int n = L->n, m = L->m;
    cudaStream_t s = L->s;
    auto up = [&](bp::DBuf<double>& b, const double* h, int k) {
      if (k) BP_CUDA(cudaMemcpyAsync(b.p, h, sizeof(double) * k, cudaMemcpyHostToDevice, s));
    };
    auto down = [&](double* h, bp::DBuf<double>& b, int k) {
      if (k) BP_CUDA(cudaMemcpyAsync(h, b.p, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    };
    up(L->x, x, n);
    up(L->xbar, x_bar, n);
    up(L->xsum, x_sum, n);
    up(L->y, y, m);
    up(L->ysum, y_sum, m);
    BP_CUDA(cudaEventRecord(L->e0, s));
    for (int it = 0; it < iters; ++it) {
      L->rows.spmv(L->xbar.p, L->ax.p, s);  // lp.hpp:318
      if (m) bp::k_pdhg_dual<<<bp::nblk(m), 256, 0, s>>>(m, L->ax.p, L->rlo.p, L->rup.p, sigma, L->y.p);
      L->cols.spmv(L->y.p, L->aty.p, s);  // lp.hpp:326
      if (n || m)
        bp::k_pdhg_primal<<<bp::nblk(std::max(n, m)), 256, 0, s>>>(n, m, L->aty.p, L->obj.p, L->vlo.p,
                                                                   L->vup.p, tau, L->x.p, L->xbar.p,
                                                                   L->xsum.p, L->y.p, L->ysum.p);
      bp::g_kernel_launches += 2;
    }
    BP_CUDA(cudaGetLastError());
    BP_CUDA(cudaEventRecord(L->e1, s));
    down(x, L->x, n);
    down(x_bar, L->xbar, n);
    down(x_sum, L->xsum, n);
    down(y, L->y, m);
    down(y_sum, L->ysum, m);
    BP_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    BP_CUDA(cudaEventElapsedTime(&ms, L->e0, L->e1));
    L->last_ms = ms;
  });
}

int bp_lp_evaluate_kkt(bp_lp* L, const double* x, const double* y, double* out7)
{
  return lguard([&] {
    need(L && x && y && out7, "null argument");
    need((L->n == 0 || (L->obj.p && L->vlo.p && L->vup.p)) && (L->m == 0 || (L->rlo.p && L->rup.p)),
         "KKT needs obj and bounds");
    BP_CUDA(cudaSetDevice(L->device));
    const int n = L->n, m = L->m;
    cudaStream_t s = L->s;
    if (n) BP_CUDA(cudaMemcpyAsync(L->x.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    if (m) BP_CUDA(cudaMemcpyAsync(L->y.p, y, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    BP_CUDA(cudaEventRecord(L->e0, s));
    L->rows.spmv(L->x.p, L->ax.p, s);  // lp.hpp:139-140
    L->cols.spmv(L->y.p, L->aty.p, s);
    const int nb = std::max(1, std::min(148 * 4, (std::max(n, m) + bp::kKktThreads - 1) / bp::kKktThreads));
    bp::DBuf<unsigned long long> st;
    bp::DBuf<bp::DD> part;
    bp::DBuf<double> sums;
    st.alloc(5);
    part.alloc(2 * nb);
    sums.alloc(2);
    BP_CUDA(cudaMemsetAsync(st.p, 0, 5 * sizeof(unsigned long long), s));
    bp::k_kkt<<<nb, bp::kKktThreads, 0, s>>>(n, m, L->x.p, L->y.p, L->ax.p, L->aty.p, L->obj.p, L->rlo.p,
                                             L->rup.p, L->vlo.p, L->vup.p, st.p, part.p);
    bp::k_kkt_final<<<1, 32, 0, s>>>(nb, part.p, sums.p);
    BP_CUDA(cudaGetLastError());
    bp::g_kernel_launches += 2;
    BP_CUDA(cudaEventRecord(L->e1, s));
    unsigned long long h[5];
    double sm[2];
    BP_CUDA(cudaMemcpyAsync(h, st.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaMemcpyAsync(sm, sums.p, sizeof(sm), cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaStreamSynchronize(s));
    double v[5];
    std::memcpy(v, h, sizeof(v));
    const double primal_res = v[0], rhs_scale = v[1], obj_scale = v[2], x_norm = v[3], dual_res = v[4];
    const double pobj = sm[0], dobj = sm[1];
    // lp.hpp:198-205, on the host in the reference's expression order
    const double gap = std::abs(pobj - dobj) / (1.0 + std::abs(pobj) + std::abs(dobj));
    const double pr  = primal_res / (1.0 + rhs_scale);
    const double dr  = dual_res / (1.0 + obj_scale);
    out7[0] = primal_res;
    out7[1] = dual_res;
    out7[2] = gap;
    out7[3] = pobj;
    out7[4] = dobj;
    out7[5] = x_norm;
    out7[6] = std::max({pr, dr, gap});
    float ms = 0.f;
    BP_CUDA(cudaEventElapsedTime(&ms, L->e0, L->e1));
    L->last_ms = ms;
  });
}

int bp_lp_last_ms(const bp_lp* L, double* ms)
{
  return lguard([&] {
    need(L && ms, "null argument");
    *ms = L->last_ms;
  });
}

}  // extern "C"
