// PDHG sparse matrix-vector products (lp.hpp:74-102) and the PDHG inner iteration (lp.hpp:315-340)
// on the device, bit-identical to the reference.
//
// spmv_rows: out[k] = sum over the row's entries of a * x[col], summed like the reference: within
// each 16384-entry segment left to right from 0.0 (`part += a * x`, separately rounded product, no
// FMA), segment partials added in order onto 0.0 (`total += part`). spmv_cols is the same over the
// CSC. Rows (columns) of <= kLpLane entries are one per thread with four entries' loads and gathers
// in flight; longer ones are split into 16384-entry segments, one warp per segment: the lanes
// gather 256 products into shared memory while lane 0 runs the sequential sum over the previous
// 256 (double buffered), then the segment partials are combined in order by a finalize pass.
//
// The PDHG step kernels fuse the elementwise updates into the SpMV epilogues: the dual update
// (y = v - sigma * clamp(v / sigma, row bounds), v = y + sigma * A x_bar) into spmv_rows, and the
// primal update (x_next = clamp(x - tau (c + A'y)), x_bar = 2 x_next - x) plus the running sums
// x_sum += x, y_sum += y into spmv_cols / its finalize — each vector is read and written once per
// half-step.
#include <algorithm>
#include <cmath>
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
constexpr int kLpChunk   = 256;     // products staged per warp step
constexpr int kLpThreads = 256;

__device__ __forceinline__ double lp_clamp(double v, double lo, double hi)
{
  return v < lo ? lo : (v > hi ? hi : v);  // common.hpp clamp: std::max(lo, std::min(v, hi))
}

// One short row / column per thread (single segment): total = 0.0 + (sequential partial).
__global__ void k_spmv_short(int nitem, const int* start, const int* idx, const double* val,
                             const double* x, const int* items, int nshort, double* out)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nshort; j += gridDim.x * blockDim.x) {
    const int it = items[j];
    const int s0 = __ldg(start + it), s1 = __ldg(start + it + 1);
    double part  = 0.0;
    for (int e0 = s0; e0 < s1; e0 += 4) {
      int c[4];
      double a[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = e0 + u < s1 ? __ldg(idx + e0 + u) : -1;
        a[u] = e0 + u < s1 ? __ldg(val + e0 + u) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = c[u] >= 0 ? x[c[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c[u] >= 0) part = __dadd_rn(part, __dmul_rn(a[u], xv[u]));
    }
    out[it] = __dadd_rn(0.0, part);
  }
  (void)nitem;
}

// One 16384-entry segment of a long row / column per warp: partial sum into seg_out[task].
__global__ void __launch_bounds__(kLpThreads)
    k_spmv_segments(const int* start, const int* idx, const double* val, const double* x,
                    const int2* tasks, int ntask, double* seg_out)
{
  __shared__ double buf[kLpThreads / 32][2][kLpChunk];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * (kLpThreads / 32) + wib, nw = gridDim.x * (kLpThreads / 32);
  for (int t = gw; t < ntask; t += nw) {
    const int2 tk = tasks[t];  // (item, segment)
    const int s0  = __ldg(start + tk.x) + tk.y * kLpSeg;
    const int s1  = min(__ldg(start + tk.x + 1), s0 + kLpSeg);
    double part   = 0.0;
    int cur       = 0;
    int prev_n    = 0;
    for (int b0 = s0; b0 < s1 + kLpChunk; b0 += kLpChunk) {
      // stage the products of chunk b0 (if any) while lane 0 folds the previous chunk
      const int n = max(0, min(kLpChunk, s1 - b0));
#pragma unroll
      for (int h = 0; h < kLpChunk / 32; ++h) {
        const int e = b0 + h * 32 + lane;
        if (h * 32 + lane < n) buf[wib][cur][h * 32 + lane] = __dmul_rn(__ldg(val + e), x[__ldg(idx + e)]);
      }
      if (lane == 0)
        for (int q = 0; q < prev_n; ++q) part = __dadd_rn(part, buf[wib][cur ^ 1][q]);
      __syncwarp();
      prev_n = n;
      cur ^= 1;
    }
    if (lane == 0) seg_out[t] = part;
    __syncwarp();
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

inline int nblk(long long n) { return (int)std::max(1ll, std::min(148ll * 16, (n + 255) / 256)); }

}  // namespace

// One matrix view (CSR or CSC) partitioned into short items and long-item segments.
struct LpView {
  int n_item = 0;
  DBuf<int> start, idx;
  DBuf<double> val;
  DBuf<int> short_items, long_items, seg_first;
  DBuf<int2> tasks;
  DBuf<double> seg_out;
  int n_short = 0, n_long = 0, n_task = 0;

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
        sf.push_back((int)tk.size());
      }
    }
    n_short = (int)sh.size();
    n_long  = (int)lg.size();
    n_task  = (int)tk.size();
    short_items.upload(sh);
    long_items.upload(lg);
    seg_first.upload(sf);
    tasks.upload(tk);
    seg_out.alloc(std::max(n_task, 1));
  }

  void spmv(const double* x, double* out, cudaStream_t s)
  {
    if (n_short)
      k_spmv_short<<<nblk(n_short), 256, 0, s>>>(n_item, start.p, idx.p, val.p, x, short_items.p,
                                                 n_short, out);
    if (n_task) {
      k_spmv_segments<<<std::min(148 * 8, (n_task + kLpThreads / 32 - 1) / (kLpThreads / 32)), kLpThreads,
                        0, s>>>(start.p, idx.p, val.p, x, tasks.p, n_task, seg_out.p);
      k_spmv_combine<<<nblk(n_long), 256, 0, s>>>(long_items.p, seg_first.p, n_long, seg_out.p, out);
    }
    BP_CUDA(cudaGetLastError());
    g_kernel_launches += (n_short ? 1 : 0) + (n_task ? 2 : 0);
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
    need(L->obj.p && L->rlo.p && L->rup.p && L->vlo.p && L->vup.p,
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

int bp_lp_last_ms(const bp_lp* L, double* ms)
{
  return lguard([&] {
    need(L && ms, "null argument");
    *ms = L->last_ms;
  });
}

}  // extern "C"
