// Fix-and-propagate bulk rounding (rounding.hpp:393-558) with device-resident working bounds.
//
// The control flow is the reference's, step for step, on the host (same RNG stream:
// std::mt19937_64 + std::uniform_real_distribution from the same libstdc++, rounding.hpp:127-152;
// the same stable sorts; the same probe-0 preference, forcing, recovery and terminal phases).
// Everything O(n) or O(N) per bulk runs on the GPU:
//   - the working bounds `ws` never leave the device;
//   - compute_activities + implied_slack_sort keys (rounding.hpp:71-115) + a stable radix sort of
//     the unset list (CUB) and its stable compaction (drop_fixed);
//   - both candidate probes (run_probe, rounding.hpp:167-207): warm start merged on the host from
//     the packed cache (sparse), met with `ws` on the device, fixings scattered, then the engine's
//     propagate. When `ws` is a certified fixpoint (its last propagate ended at a fixpoint) the
//     first round starts from the frontier of the changed variables, which turns
//     the reference's O(N) first round into O(frontier);
//   - count_envelope_violations (rounding.hpp:361-383).
// lp_polish (PDHG, rounding.hpp:315-345) is out of scope: the outcome reports `bounds_feasible`
// (the condition under which the reference would polish) and returns the pre-polish point.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <random>
#include <sstream>
#include <string>
#include <stdexcept>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/bp.h"
#include "bp_capi_internal.h"
#include "bp_engine.cuh"
#include "bp_probe.cuh"

namespace bp {

namespace {

constexpr double kFeasTol = 1e-6;  // common.hpp:20

__global__ void k_meet_root(double2* b, const double2* root, int n, int* flags)
{
  int fl = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2 x = b[i], r = root[i];
    const double lo = (x.x < r.x) ? r.x : x.x;  // std::max(b, other)
    const double up = (r.y < x.y) ? r.y : x.y;  // std::min(b, other)
    if (lo != x.x || up != x.y) {
      fl |= 1;
      b[i] = make_double2(lo, up);
    }
    if (lo > up) fl |= 2;
  }
  if (fl) atomicOr(flags, fl);
}

// Meet of listed vars with the given bounds; new values + per-var "changed" written back.
__global__ void k_meet_list(double2* b, const int* var, const double* lo, const double* up, int k,
                            int* changed, int* flags)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    const int i    = var[j];
    const double2 x = b[i];
    const double nl = (x.x < lo[j]) ? lo[j] : x.x;
    const double nu = (up[j] < x.y) ? up[j] : x.y;
    changed[j]      = (nl != x.x || nu != x.y) ? 1 : 0;
    b[i]            = make_double2(nl, nu);
    if (nl > nu) atomicOr(flags, 2);
  }
}

__global__ void k_gather(const double2* b, const int* var, int k, double2* out)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    out[j] = b[var[j]];
}

// The first k vars of the current order and their bounds in one pass (take_first + gather).
__global__ void k_take_gather(const int* order, const double2* b, int k, int* var_out, double2* b_out)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    const int v = order[j];
    var_out[j]  = v;
    b_out[j]    = b[v];
  }
}

__global__ void k_scatter(double2* b, const int* var, const double2* val, int k)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    b[var[j]] = val[j];
}

// rounding.hpp:71-115 keys: S_i = sum over rows of (a / slack)^2 in CSC order, +inf on a
// non-positive slack; returned as order-preserving 64-bit keys (S >= +0.0, never -0.0).
__global__ void k_slack_keys(DevProblem P, const RowRec* rec, const double2* aux, const int* vars,
                             int k, unsigned long long* keys, int* pos)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    const int i  = vars[j];
    double total = 0.0;
    for (int e = P.col_start[i]; e < P.col_start[i + 1]; ++e) {
      const int r    = P.col_row[e];
      const double a = P.col_val[e];
      const RowRec q = rec[r];
      double mnf, mxf;
      int nmn, nmx;
      decode_rec(q, aux, r, mnf, nmn, mxf, nmx);
      if (isfinite(q.g) && nmn == 0) {
        const double slack = __dsub_rn(q.g, mnf);
        if (slack <= 0.0) {
          total = INFINITY;
          break;
        }
        const double s = __ddiv_rn(a, slack);
        total          = __dadd_rn(total, __dmul_rn(s, s));
      }
      if (isfinite(q.h) && nmx == 0) {
        const double slack = __dsub_rn(mxf, q.h);
        if (slack <= 0.0) {
          total = INFINITY;
          break;
        }
        const double s = __ddiv_rn(a, slack);
        total          = __dadd_rn(total, __dmul_rn(s, s));
      }
    }
    keys[j] = okey(total);
    pos[j]  = j;
  }
}

__global__ void k_permute(const int* src, const int* pos, int k, int* dst)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    dst[j] = src[pos[j]];
}

// rounding.hpp:372-381: rows violated by the fixed-value envelope.
__global__ void k_count_violations(DevProblem P, const RowRec* rec, const double2* aux, int* out)
{
  int cnt = 0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.m; k += gridDim.x * blockDim.x) {
    const RowRec q = rec[k];
    double mnf, mxf;
    int nmn, nmx;
    decode_rec(q, aux, k, mnf, nmn, mxf, nmx);
    if (isfinite(q.g) && nmn == 0 && mnf > __dadd_rn(q.g, kFeasTol)) ++cnt;
    else if (isfinite(q.h) && nmx == 0 && mxf < __dsub_rn(q.h, kFeasTol)) ++cnt;
  }
  if (cnt) atomicAdd(out, cnt);
}

// repair's most-violated-row scan (rounding.hpp:249-266), pass 1: the largest violation above
// kFeasTol (positive doubles order like their bit patterns).
__device__ __forceinline__ void row_violations(const RowRec& q, const double2* aux, int k,
                                               double& vu, double& vl)
{
  double mnf, mxf;
  int nmn, nmx;
  decode_rec(q, aux, k, mnf, nmn, mxf, nmx);
  vu = (isfinite(q.g) && nmn == 0) ? __dsub_rn(mnf, q.g) : -INFINITY;
  vl = (isfinite(q.h) && nmx == 0) ? __dsub_rn(q.h, mxf) : -INFINITY;
}

__global__ void k_worst_viol(DevProblem P, const RowRec* rec, const double2* aux,
                             unsigned long long* best)
{
  double w = kFeasTol;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.m; k += gridDim.x * blockDim.x) {
    double vu, vl;
    row_violations(rec[k], aux, k, vu, vl);
    if (vu > w) w = vu;
    if (vl > w) w = vl;
  }
  unsigned long long b = __double_as_longlong(w);
  for (int o = 16; o; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, b, o);
    b = x > b ? x : b;
  }
  if ((threadIdx.x & 31) == 0 && b > (unsigned long long)__double_as_longlong(kFeasTol))
    atomicMax(best, b);
}

// pass 2: the first (row ascending, upper side before lower) candidate attaining it, as 2k + side
// (the reference keeps the earlier candidate on ties: `viol > worst_viol`).
__global__ void k_worst_pos(DevProblem P, const RowRec* rec, const double2* aux,
                            const unsigned long long* best, int* pos)
{
  const unsigned long long b = *best;
  if (b == 0) return;
  const double w = __longlong_as_double((long long)b);
  int first      = INT_MAX;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.m; k += gridDim.x * blockDim.x) {
    double vu, vl;
    row_violations(rec[k], aux, k, vu, vl);
    if (vu == w) {
      first = min(first, 2 * k);
      break;  // later k of this thread are larger
    }
    if (vl == w) {
      first = min(first, 2 * k + 1);
      break;
    }
  }
  for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  if ((threadIdx.x & 31) == 0 && first != INT_MAX) atomicMin(pos, first);
}

struct NotFixed {
  const double2* ws;
  __device__ __forceinline__ bool operator()(const int& v) const { return ws[v].x != ws[v].y; }
};

inline int blocks_for(long long n) { return (int)std::max(1ll, std::min(4096ll, (n + 255) / 256)); }

double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

}  // namespace

// Host-side step timers of the driver (BP_ROUND_PROFILE=1 prints them at the end of a call).
struct StepTimes {
  double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool on = getenv("BP_ROUND_PROFILE") != nullptr;
};
struct StepTimer {
  StepTimes& T;
  int k;
  std::chrono::steady_clock::time_point t0;
  StepTimer(StepTimes& T_, int k_) : T(T_), k(k_), t0(std::chrono::steady_clock::now()) {}
  ~StepTimer()
  {
    T.t[k] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    T.n[k]++;
  }
};

// Persistent per-call device context of the rounding driver.
struct RoundCtx {
  Problem& P;
  const bp_problem_host& H;
  cudaStream_t s;
  DBuf<double2> ws, root, tmp2, orig;
  DBuf<RowRec> ws_rec;   // activity records consistent with ws while ws_cert holds
  DBuf<double2> ws_aux;
  DBuf<int> unset, unset_alt, pos_in, pos_out, sel_count, flags, ivar, jvar, ichg;
  DBuf<unsigned long long> keys_in, keys_out;
  DBuf<double> dlo, dup;
  DBuf<unsigned char> cub_tmp;
  StepTimes* tt = nullptr;
  int n_unset = 0;
  bool ws_infeasible = false;
  bool ws_cert       = false;
  long long bp_calls = 0;
  double dev_ms      = 0.0;
  // BP_ROUND_STATS=1 (with BP_ROUND_PROFILE): per-round work and phase times of every engine call,
  // aggregated by round index (device stats rows, see kStatCols)
  bool stats_on = getenv("BP_ROUND_STATS") != nullptr;
  DBuf<long long> d_stats;
  std::vector<double> st_sum = std::vector<double>(17 * 10, 0.0);
  std::vector<long long> st_rounds = std::vector<long long>(66, 0);

  RoundCtx(Problem& P_, const bp_problem_host& H_) : P(P_), H(H_), s(P_.stream) {}

  Limits limits() const
  {
    Limits l;
    l.max_rounds    = 64;
    l.time_limit    = INFINITY;
    l.abs_threshold = 1e-7;
    l.rel_threshold = 1e-4;
    l.incremental   = 1;
    return l;
  }

  // Pinned staging for the driver's small transfers: uploads are copied into it and sent
  // asynchronously, readbacks land in it and are copied out at the next sync() -- one stream
  // synchronisation per step instead of one per (pageable, hence synchronous) copy.
  char* pin        = nullptr;
  size_t pin_cap   = 0, pin_off = 0;
  struct Pending {
    void* dst;
    const char* src;
    size_t bytes;
  };
  std::vector<Pending> pending;

  ~RoundCtx()
  {
    if (pin) cudaFreeHost(pin);
  }
  char* stage(size_t bytes)
  {
    bytes = (bytes + 15) / 16 * 16;
    if (pin_off + bytes > pin_cap) {
      sync();  // every staged copy has completed: the buffer may be reused / grown
      if (bytes > pin_cap) {
        if (pin) cudaFreeHost(pin);
        pin_cap = std::max<size_t>(bytes, 1 << 22);
        BP_CUDA(cudaMallocHost(&pin, pin_cap));
      }
    }
    char* p = pin + pin_off;
    pin_off += bytes;
    return p;
  }
  void sync()
  {
    BP_CUDA(cudaStreamSynchronize(s));
    for (const auto& q : pending) std::memcpy(q.dst, q.src, q.bytes);
    pending.clear();
    pin_off = 0;
  }
  // device -> host readback delivered to dst at the next sync()
  void get_async(void* dst, const void* dev_src, size_t bytes)
  {
    if (!bytes) return;
    char* st = stage(bytes);
    BP_CUDA(cudaMemcpyAsync(st, dev_src, bytes, cudaMemcpyDeviceToHost, s));
    pending.push_back({dst, st, bytes});
  }

  // Stream-ordered upload through the pinned staging (the engine stream is non-blocking: a plain
  // cudaMemcpy would race with kernels still reading the buffer).
  template <class T>
  void put(DBuf<T>& b, const std::vector<T>& v)
  {
    if (b.n < v.size()) b.alloc(std::max(v.size(), 2 * b.n));
    if (!v.empty()) {
      char* st = stage(sizeof(T) * v.size());
      std::memcpy(st, v.data(), sizeof(T) * v.size());
      BP_CUDA(cudaMemcpyAsync(b.p, st, sizeof(T) * v.size(), cudaMemcpyHostToDevice, s));
    }
  }
  template <class T>
  void reserve(DBuf<T>& b, size_t k)
  {
    if (b.n < k) b.alloc(std::max(k, 2 * b.n));
  }

  std::vector<double2> gather(const DBuf<double2>& b, const std::vector<int>& vars)
  {
    std::vector<double2> out(vars.size());
    if (vars.empty()) return out;
    put(ivar, vars);
    reserve(tmp2, vars.size());
    k_gather<<<blocks_for(vars.size()), 256, 0, s>>>(b.p, ivar.p, (int)vars.size(), tmp2.p);
    BP_CUDA(cudaMemcpyAsync(out.data(), tmp2.p, sizeof(double2) * vars.size(), cudaMemcpyDeviceToHost, s));
    sync();
    return out;
  }

  void scatter(double2* b, const std::vector<int>& vars, const std::vector<double2>& vals)
  {
    if (vars.empty()) return;
    put(ivar, vars);
    put(tmp2, vals);
    k_scatter<<<blocks_for(vars.size()), 256, 0, s>>>(b, ivar.p, tmp2.p, (int)vars.size());
  }

  // Commit: the engine's result becomes the working state by swapping buffers (no 16n / 48m-byte
  // copies): ws <- P.st.bounds, and while certified the activity records with it.
  void adopt_engine_state(bool cert)
  {
    std::swap(ws.p, P.bounds.p);
    std::swap(ws.n, P.bounds.n);
    P.st.bounds = P.bounds.p;
    if (cert && P.m) {
      reserve(ws_rec, (size_t)std::max(P.m, 1));
      reserve(ws_aux, (size_t)std::max(P.m, 1));
      std::swap(ws_rec.p, P.rec.p);
      std::swap(ws_rec.n, P.rec.n);
      std::swap(ws_aux.p, P.aux.p);
      std::swap(ws_aux.n, P.aux.n);
      P.st.rec = P.rec.p;
      P.st.aux = P.aux.p;
    }
  }

  // After a propagate that ended at a fixpoint, P.st.rec / aux describe its final bounds for
  // every row; keep them as the certified state's activities.
  void snapshot_ws_activities()
  {
    reserve(ws_rec, (size_t)std::max(P.m, 1));
    reserve(ws_aux, (size_t)std::max(P.m, 1));
    if (P.m) {
      BP_CUDA(cudaMemcpyAsync(ws_rec.p, P.st.rec, sizeof(RowRec) * P.m, cudaMemcpyDeviceToDevice, s));
      BP_CUDA(cudaMemcpyAsync(ws_aux.p, P.st.aux, sizeof(double2) * P.m, cudaMemcpyDeviceToDevice, s));
    }
  }

  RunResult propagate_engine(bool start_frontier, const std::vector<int>& changed)
  {
    BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(Ctl), s));
    int flags = 0;
    if (start_frontier) {
      // a frontier round reads the activities of rows it does not recompute: they must be the
      // certified state's, whatever the previous engine call left behind
      if (P.m) {
        BP_CUDA(cudaMemcpyAsync(P.st.rec, ws_rec.p, sizeof(RowRec) * P.m, cudaMemcpyDeviceToDevice, s));
        BP_CUDA(cudaMemcpyAsync(P.st.aux, ws_aux.p, sizeof(double2) * P.m, cudaMemcpyDeviceToDevice, s));
      }
      stage_changed(P, changed.data(), (int)changed.size(), s);
      flags = ENGINE_START_FRONTIER;
    }
    long long* stp = nullptr;
    if (stats_on) {
      reserve(d_stats, 64 * kStatCols);
      BP_CUDA(cudaMemsetAsync(d_stats.p, 0, sizeof(long long) * 64 * kStatCols, s));
      stp = d_stats.p;
    }
    const RunResult r = run_engine(P, MODE_PROPAGATE, true, limits(), s, flags, stp);
    if (stats_on) {
      std::vector<long long> h(64 * kStatCols);
      BP_CUDA(cudaMemcpy(h.data(), d_stats.p, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost));
      st_rounds[std::min(r.rounds, 65)]++;
      long long prev = 0;
      for (int q = 0; q < std::min(r.rounds, 64); ++q) {
        const long long* row = h.data() + q * kStatCols;
        const int b = std::min(q, 16);
        double* o = st_sum.data() + b * 10;
        // calls reaching this round, full rounds, |R|, A, |V|, B, then us: gather, activity,
        // tightening, expansion (rows + vars)
        o[0] += 1; o[1] += row[0]; o[2] += row[1]; o[3] += row[2]; o[4] += row[3]; o[5] += row[4];
        o[6] += (row[10] - prev) * 1e-3;
        o[7] += (row[6] - row[10]) * 1e-3;
        o[8] += (row[7] - row[6]) * 1e-3;
        o[9] += (row[9] - row[7]) * 1e-3;
        prev = row[9];
      }
    }
    bp_calls++;
    dev_ms += P.last_kernel_ms;
    return r;
  }

  // compute_activities(p, b, nullptr, acts) of bounds `b` (device) into P.st.rec / aux.
  void activities(const double2* b)
  {
    BP_CUDA(cudaMemcpyAsync(P.st.bounds, b, sizeof(double2) * P.n, cudaMemcpyDeviceToDevice, s));
    BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(Ctl), s));
    run_engine(P, MODE_ACTIVITY, true, limits(), s);
    dev_ms += P.last_kernel_ms;
  }

  // implied_slack_sort of the unset list, in place (stable).
  void slack_sort()
  {
    // compute_activities(p, ws) (rounding.hpp:427): a certified ws already has them -- the
    // records its last propagate ended with (no bound changed in that round), kept in ws_rec
    const RowRec* rec  = P.st.rec;
    const double2* aux = P.st.aux;
    if (ws_cert && P.m && ws_rec.n >= (size_t)P.m) {
      rec = ws_rec.p;
      aux = ws_aux.p;
    } else {
      activities(ws.p);
    }
    const int k = n_unset;
    k_slack_keys<<<blocks_for(k), 256, 0, s>>>(P.dev(), rec, aux, unset.p, k, keys_in.p, pos_in.p);
    // stable LSD radix sort of (key, position): std::stable_sort's order (rounding.hpp:81-104).
    // (An incremental variant -- merging the vars whose key did not change with the re-sorted
    // rest -- measured slower on C4: nearly every key changes every bulk.)
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, keys_in.p, keys_out.p, pos_in.p, pos_out.p, k, 0,
                                    64, s);
    if (need > cub_tmp.n) cub_tmp.alloc(need);
    size_t have = cub_tmp.n;
    cub::DeviceRadixSort::SortPairs(cub_tmp.p, have, keys_in.p, keys_out.p, pos_in.p, pos_out.p, k,
                                    0, 64, s);
    k_permute<<<blocks_for(k), 256, 0, s>>>(unset.p, pos_out.p, k, unset_alt.p);
    std::swap(unset.p, unset_alt.p);
    std::swap(unset.n, unset_alt.n);
  }

  // unset.erase(remove_if(ws.fixed(v))) (stable).
  void drop_fixed()
  {
    size_t need = 0;
    NotFixed pred{ws.p};
    cub::DeviceSelect::If(nullptr, need, unset.p, unset_alt.p, sel_count.p, n_unset, pred, s);
    if (need > cub_tmp.n) cub_tmp.alloc(need);
    size_t have = cub_tmp.n;
    cub::DeviceSelect::If(cub_tmp.p, have, unset.p, unset_alt.p, sel_count.p, n_unset, pred, s);
    std::swap(unset.p, unset_alt.p);
    std::swap(unset.n, unset_alt.n);
    get_async(&n_unset, sel_count.p, sizeof(int));
    sync();
  }

  // take_first(k) + gather(ws, ...) with one kernel and one synchronisation.
  std::vector<int> take_gather(int k, std::vector<double2>& tb)
  {
    std::vector<int> t(k);
    tb.resize(k);
    if (k) {
      reserve(ivar, k);
      reserve(tmp2, k);
      k_take_gather<<<blocks_for(k), 256, 0, s>>>(unset.p, ws.p, k, ivar.p, tmp2.p);
      get_async(t.data(), ivar.p, sizeof(int) * k);
      get_async(tb.data(), tmp2.p, sizeof(double2) * k);
      sync();
    }
    return t;
  }

  std::vector<int> take_first(int k)
  {
    std::vector<int> t(k);
    if (k) BP_CUDA(cudaMemcpyAsync(t.data(), unset.p, sizeof(int) * k, cudaMemcpyDeviceToHost, s));
    sync();
    return t;
  }

  struct Probe {
    int infeas_count = 0;
    bool infeasible  = false;
    bool cert        = false;
    std::vector<int> evicted;
    std::vector<std::pair<int, double>> fixed;
  };

  // rounding.hpp:167-207 with the result bounds left in P.st.bounds.
  Probe run_probe(const std::vector<int>& vars, const std::vector<double>& values,
                  const HostCache* cache)
  {
    Probe out;
    BP_CUDA(cudaMemcpyAsync(P.st.bounds, ws.p, sizeof(double2) * P.n, cudaMemcpyDeviceToDevice, s));
    bool inf          = ws_infeasible;
    bool root_changed = false;
    std::vector<int> changed, dv_keep, ch;
    int fl = 0;
    auto t_ws = std::chrono::steady_clock::now();
    if (cache) {
      // warm start on the host (sparse deltas over the cache root), meet on the device
      std::vector<int> conflicts, dv;
      std::vector<double> dl, du;
      bp::warm_start_sparse(*cache, vars.data(), values.data(), (int)vars.size(), dv, dl, du,
                            conflicts, out.evicted);
      reserve(flags, 1);
      BP_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), s));
      k_meet_root<<<blocks_for(P.n), 256, 0, s>>>(P.st.bounds, root.p, P.n, flags.p);
      if (!dv.empty()) {
        put(ivar, dv);
        put(dlo, dl);
        put(dup, du);
        reserve(ichg, dv.size());
        k_meet_list<<<blocks_for(dv.size()), 256, 0, s>>>(P.st.bounds, ivar.p, dlo.p, dup.p,
                                                          (int)dv.size(), ichg.p, flags.p);
      }
      get_async(&fl, flags.p, sizeof(int));
      ch.resize(dv.size());
      get_async(ch.data(), ichg.p, sizeof(int) * dv.size());
      dv_keep = std::move(dv);
    }
    // fixings (rounding.hpp:186-195) need the post-meet bounds of the bulk vars: gathered in the
    // same stream step and read back with the meet's flags -- one synchronisation
    std::vector<double2> cur(vars.size());
    if (!vars.empty()) {
      put(jvar, vars);
      reserve(tmp2, vars.size());
      k_gather<<<blocks_for(vars.size()), 256, 0, s>>>(P.st.bounds, jvar.p, (int)vars.size(), tmp2.p);
      get_async(cur.data(), tmp2.p, sizeof(double2) * vars.size());
    }
    sync();
    if (cache) {
      root_changed = (fl & 1) != 0;
      if (fl & 2) inf = true;
      for (size_t j = 0; j < dv_keep.size(); ++j)
        if (ch[j]) changed.push_back(dv_keep[j]);
    }
    if (tt) {
      tt->t[4] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_ws).count();
      tt->n[4]++;
    }
    auto t_fx = std::chrono::steady_clock::now();
    const std::unordered_set<int> evm(out.evicted.begin(), out.evicted.end());
    int crossings = inf ? 1 : 0;
    std::vector<int> fv;
    std::vector<double2> fb;
    // repeated vars: later assignments see earlier fixings (the var's current bounds)
    std::unordered_map<int, int> slot_of;  // var -> index in fv
    slot_of.reserve(2 * vars.size());
    for (size_t j = 0; j < vars.size(); ++j) {
      const int v = vars[j];
      if (!evm.empty() && evm.count(v)) continue;
      const auto it   = slot_of.find(v);
      const double2 b = it == slot_of.end() ? cur[j] : fb[it->second];
      const double val = values[j];
      if (val < b.x - 1e-9 || val > b.y + 1e-9) {
        ++crossings;
        continue;
      }
      if (b.x != val || b.y != val) changed.push_back(v);
      if (it == slot_of.end()) {
        slot_of.emplace(v, (int)fv.size());
        fv.push_back(v);
        fb.push_back(make_double2(val, val));
      } else {
        fb[it->second] = make_double2(val, val);  // the last fixing of v wins
      }
      out.fixed.push_back({v, val});
    }
    scatter(P.st.bounds, fv, fb);  // applied even when crossing, as in the reference's out.bounds
    if (crossings > 0) {
      out.infeasible   = true;
      out.infeas_count = crossings;
      return out;
    }
    std::sort(changed.begin(), changed.end());
    changed.erase(std::unique(changed.begin(), changed.end()), changed.end());
    const bool frontier = ws_cert && !root_changed;
    if (tt) {
      tt->t[5] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_fx).count();
      tt->n[5]++;
    }
    auto t_en         = std::chrono::steady_clock::now();
    const RunResult r = propagate_engine(frontier, changed);
    if (tt) {
      tt->t[6] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_en).count();
      tt->n[6]++;
    }
    if (r.status == BP_STATUS_INFEASIBLE) {
      out.infeasible   = true;
      out.infeas_count = std::max(1, r.crossed);
    }
    out.cert = r.fixpoint != 0;
    return out;
  }

  // repair (rounding.hpp:234-311): shifts fixed values one variable per violated row until
  // propagation from the original bounds succeeds. Per shift: original bounds + fixings built on
  // the device, full activity sweep, most-violated-row scan (k_worst_viol / k_worst_pos), then the
  // shift chosen on the host from that one row. On success the repaired bounds are left in
  // P.st.bounds and *rr holds the propagate's result (its exit reason certifies the state).
  template <class Expired>
  bool repair(std::vector<std::pair<int, double>>& fixed, const double2* d_orig, Expired expired,
              int shift_cap, RunResult* rr)
  {
    const int n = P.n;
    std::vector<int> fixed_pos(n, -1);
    for (size_t j = 0; j < fixed.size(); ++j) fixed_pos[fixed[j].first] = (int)j;
    // b.fix in list order: the last fixing of a var wins, so scatter one value per var
    std::vector<int> fv;
    std::vector<double2> fb;
    std::vector<int> slot(n, -1);
    for (const auto& [v, val] : fixed) {
      if (slot[v] < 0) {
        slot[v] = (int)fv.size();
        fv.push_back(v);
        fb.push_back(make_double2(val, val));
      } else {
        fb[slot[v]] = make_double2(val, val);
      }
    }
    DBuf<int> dfv;
    DBuf<double2> dfb;
    if (!fv.empty()) {
      dfv.alloc(fv.size());
      dfb.alloc(fv.size());
      BP_CUDA(cudaMemcpyAsync(dfv.p, fv.data(), sizeof(int) * fv.size(), cudaMemcpyHostToDevice, s));
      BP_CUDA(cudaMemcpyAsync(dfb.p, fb.data(), sizeof(double2) * fv.size(), cudaMemcpyHostToDevice, s));
    }
    DBuf<unsigned long long> best;
    DBuf<int> bpos;
    best.alloc(1);
    bpos.alloc(1);
    for (int iter = 0; iter < shift_cap; ++iter) {
      if (expired()) return false;
      if (n) BP_CUDA(cudaMemcpyAsync(P.st.bounds, d_orig, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
      if (!fv.empty())
        k_scatter<<<blocks_for(fv.size()), 256, 0, s>>>(P.st.bounds, dfv.p, dfb.p, (int)fv.size());
      BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(Ctl), s));
      run_engine(P, MODE_ACTIVITY, true, limits(), s);
      dev_ms += P.last_kernel_ms;
      BP_CUDA(cudaMemsetAsync(best.p, 0, sizeof(unsigned long long), s));
      BP_CUDA(cudaMemsetAsync(bpos.p, 0x7f, sizeof(int), s));
      k_worst_viol<<<blocks_for(P.m), 256, 0, s>>>(P.dev(), P.st.rec, P.st.aux, best.p);
      k_worst_pos<<<blocks_for(P.m), 256, 0, s>>>(P.dev(), P.st.rec, P.st.aux, best.p, bpos.p);
      unsigned long long hb = 0;
      int hpos              = 0;
      BP_CUDA(cudaMemcpyAsync(&hb, best.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaMemcpyAsync(&hpos, bpos.p, sizeof(hpos), cudaMemcpyDeviceToHost, s));
      sync();
      if (hb == 0) {  // no violated row: propagate from the fixed-value state (rounding.hpp:268-274)
        BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(Ctl), s));
        *rr = run_engine(P, MODE_PROPAGATE, true, limits(), s);
        bp_calls++;
        dev_ms += P.last_kernel_ms;
        return rr->status != BP_STATUS_INFEASIBLE;
      }
      double worst_viol;
      std::memcpy(&worst_viol, &hb, sizeof(double));
      const int row         = hpos >> 1;
      const bool upper_side = (hpos & 1) == 0;
      // smallest in-bounds shift of one fixed variable that restores the row (rounding.hpp:276-306)
      int best_var    = -1;
      double best_val = 0.0;
      for (int e = P.h_row_start[row]; e < P.h_row_start[row + 1]; ++e) {
        const int v = H.row_col[e];
        if (fixed_pos[v] < 0) continue;
        const double a_kv = H.row_val[e];
        const double cur  = fixed[fixed_pos[v]].second;
        double delta      = worst_viol / std::abs(a_kv);
        if (H.is_integer[v]) delta = std::ceil(delta - 1e-9);
        double cand;
        if (upper_side) cand = (a_kv > 0.0) ? cur - delta : cur + delta;
        else cand = (a_kv > 0.0) ? cur + delta : cur - delta;
        if (cand < H.var_lower[v] - 1e-9 || cand > H.var_upper[v] + 1e-9) continue;
        if (best_var < 0 || std::abs(cand - cur) < std::abs(best_val - fixed[fixed_pos[best_var]].second)) {
          best_var = v;
          best_val = cand;
        }
      }
      if (best_var < 0) return false;
      fixed[fixed_pos[best_var]].second = best_val;
      const double2 nb                  = make_double2(best_val, best_val);
      fb[slot[best_var]]                = nb;
      BP_CUDA(cudaMemcpyAsync(dfb.p + slot[best_var], &fb[slot[best_var]], sizeof(double2),
                              cudaMemcpyHostToDevice, s));
    }
    sync();
    return false;
  }

  // rounding.hpp:361-383
  int count_envelope_violations(const std::vector<int>& vars, const std::vector<double>& values)
  {
    BP_CUDA(cudaMemcpyAsync(P.st.bounds, ws.p, sizeof(double2) * P.n, cudaMemcpyDeviceToDevice, s));
    std::vector<double2> vals(vars.size());
    for (size_t j = 0; j < vars.size(); ++j) {
      const int v     = vars[j];
      const double lo = std::max(H.var_lower[v], std::min(values[j], H.var_upper[v]));
      vals[j]         = make_double2(lo, lo);
    }
    // repeated vars: the last fixing wins, as in the sequential loop
    scatter(P.st.bounds, vars, vals);
    BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(Ctl), s));
    run_engine(P, MODE_ACTIVITY, true, limits(), s);
    dev_ms += P.last_kernel_ms;
    reserve(flags, 1);
    BP_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), s));
    k_count_violations<<<blocks_for(P.m), 256, 0, s>>>(P.dev(), P.st.rec, P.st.aux, flags.p);
    int h = 0;
    BP_CUDA(cudaMemcpyAsync(&h, flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync();
    return h;
  }
};

// rounding.hpp:35-65
std::vector<int> initial_sort(const bp_problem_host& H, const double* values, int n)
{
  struct Item {
    int var, cls;
    double frac;
  };
  std::vector<Item> items;
  for (int i = 0; i < n; ++i) {
    if (!H.is_integer[i]) continue;
    const double w = H.var_upper[i] - H.var_lower[i];
    const int cls  = (w == 1.0) ? 0 : (w == 2.0 ? 1 : 2);
    const double v = values[i];
    items.push_back({i, cls, std::abs(v - std::round(v))});
  }
  std::stable_sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
    if (a.cls != b.cls) return a.cls < b.cls;
    return a.frac < b.frac;
  });
  std::vector<int> o;
  for (const auto& it : items) o.push_back(it.var);
  return o;
}

// rounding.hpp:119-123
int get_bulk_size(int remaining, bool recovery, int tail)
{
  if (recovery || remaining <= tail) return 1;
  return (int)std::lround(std::sqrt(double(remaining)));
}

// rounding.hpp:127-152 (host RNG; identical stream to the reference)
void candidate_values(const double* sv, const std::vector<int>& vars,
                      const std::vector<double2>& bounds, std::mt19937_64& rng, double band,
                      std::vector<double>& v0, std::vector<double>& v1)
{
  v0.clear();
  v1.clear();
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  for (size_t j = 0; j < vars.size(); ++j) {
    const double v  = sv[vars[j]];
    const double fl = std::floor(v);
    const double f  = v - fl;
    double d0, d1;
    if (std::abs(f - 0.5) >= band) {
      d0 = d1 = std::round(v);
    } else {
      d0 = fl + (unit(rng) < f ? 1.0 : 0.0);
      d1 = fl + (unit(rng) < f ? 1.0 : 0.0);
    }
    const double lo = std::ceil(bounds[j].x - 1e-9);
    const double hi = std::floor(bounds[j].y + 1e-9);
    v0.push_back(clampd(d0, lo, hi));
    v1.push_back(clampd(d1, lo, hi));
  }
}

}  // namespace bp

extern "C" void bp_rounding_config_default(bp_rounding_config* c)
{
  c->random_band        = 0.25;
  c->single_var_tail    = 36;
  c->repair_enabled     = 0;
  c->repair_attempt_cap = 16;
  c->repair_shift_cap   = 64;
}

namespace {

// propagation_round with the caller's generator (consumed exactly like the reference's Rng&).
int round_impl(bp_problem* p, const double* start_values, const bp_cache* cache,
               std::mt19937_64& rng, double deadline_sec, const bp_rounding_config* cfg_in,
               double* out_values, bp_rounding_outcome* out)
{
  try {
    if (!p || !start_values || !out_values || !out) throw std::invalid_argument("null argument");
    bp_rounding_config cfg;
    bp_rounding_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    if (cfg.repair_enabled && (cfg.repair_attempt_cap < 0 || cfg.repair_shift_cap < 0))
      throw std::invalid_argument("negative repair cap");
    bp::Problem& P                 = bp_problem_impl(p);
    const bp_problem_host& H       = bp_problem_hostdata(p);
    const bp::HostCache* hc        = cache ? bp_cache_host(cache) : nullptr;
    std::lock_guard<std::mutex> lk(P.mu);
    BP_CUDA(cudaSetDevice(P.device));
    const int n = P.n;
    const auto t0 = std::chrono::steady_clock::now();
    auto expired  = [&] {
      if (!(deadline_sec > 0.0)) return false;
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() >= deadline_sec;
    };
    bp::RoundCtx X(P, H);
    bp::StepTimes TT;
    X.tt = &TT;
    std::vector<double> orig(2 * (size_t)n);
    bp_problem_root(p, orig.data());
    X.ws.upload(reinterpret_cast<const double2*>(orig.data()), n);
    X.root.alloc(std::max(n, 1));
    if (hc) BP_CUDA(cudaMemcpy(X.root.p, hc->root.data(), sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
    // is the original-bounds state a certified fixpoint? (one full round changes nothing)
    {
      BP_CUDA(cudaMemcpyAsync(P.st.bounds, X.ws.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, X.s));
      BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(bp::Ctl), X.s));
      bp::Limits one   = X.limits();
      one.max_rounds   = 1;
      const auto r     = bp::run_engine(P, bp::MODE_PROPAGATE, true, one, X.s);
      X.ws_cert        = r.status == bp::BP_STATUS_UNCHANGED;
      if (X.ws_cert) X.snapshot_ws_activities();
    }
    // unset = initial_sort minus fixed (rounding.hpp:400-404)
    std::vector<int> unset0;
    for (int v : bp::initial_sort(H, start_values, n))
      if (orig[2 * v] != orig[2 * v + 1]) unset0.push_back(v);
    X.n_unset = (int)unset0.size();
    const size_t cap = std::max<size_t>(unset0.size(), 1);
    X.unset.upload(unset0.data(), unset0.size());
    if (X.unset.n < cap) X.unset.alloc(cap);
    X.unset_alt.alloc(cap);
    X.pos_in.alloc(cap);
    X.pos_out.alloc(cap);
    X.keys_in.alloc(cap);
    X.keys_out.alloc(cap);
    X.sel_count.alloc(1);
    std::vector<std::pair<int, double>> committed;
    bool recovery = false, force = false;
    bp_rounding_outcome o;
    std::memset(&o, 0, sizeof(o));
    std::vector<double> pv0, pv1;
    // measurement knob (bench.py's like-for-like rate against the reference's first K bulks):
    // BP_ROUND_MAX_BULKS=K stops after K committed bulks, reported as a timeout
    const char* mb_env     = std::getenv("BP_ROUND_MAX_BULKS");
    const long long max_bk = mb_env ? std::atoll(mb_env) : 0;
    while (X.n_unset > 0) {
      if (expired() || (max_bk > 0 && o.bulks_committed >= max_bk)) {
        o.timed_out = 1;
        break;
      }
      const int bulk = bp::get_bulk_size(X.n_unset, recovery && !force, cfg.single_var_tail);
      if (!force) {
        if (bulk > 1) {
          bp::StepTimer st(TT, 0);
          X.slack_sort();
        }
        std::vector<int> take;
        std::vector<double2> tb;
        {
          bp::StepTimer st(TT, 1);
          take = X.take_gather(bulk, tb);
          bp::candidate_values(start_values, take, tb, rng, cfg.random_band, pv0, pv1);
        }
        bp::RoundCtx::Probe pr0;
        {
          bp::StepTimer st(TT, 2);
          pr0 = X.run_probe(take, pv0, hc);
        }
        int sel    = -1;
        bp::RoundCtx::Probe pr1;
        if (pr0.infeas_count == 0) {
          sel = 0;
        } else {
          bp::StepTimer st(TT, 2);
          pr1 = X.run_probe(take, pv1, hc);
          if (pr1.infeas_count == 0) sel = 1;
        }
        if (sel >= 0) {
          auto& pr = sel == 0 ? pr0 : pr1;
          if (!pr.fixed.empty()) {  // commit (rounding.hpp:436-443)
            bp::StepTimer st(TT, 3);
            X.adopt_engine_state(pr.cert);
            X.ws_infeasible = false;
            X.ws_cert       = pr.cert;
            for (const auto& fv : pr.fixed) committed.push_back(fv);
            X.drop_fixed();
            recovery = false;
            o.bulks_committed++;
            continue;
          }
          // every bulk var evicted: apply the cache's forced branches (rounding.hpp:447-478)
          bool narrowed = false;
          for (int v : pr.evicted) {
            const int e = (hc && v < hc->n) ? hc->entry_of[v] : -1;
            if (e < 0) continue;
            const double2 b = X.gather(X.ws, {v})[0];
            double lo = b.x, up = b.y;
            if (hc->e_force[2 * e] && up > hc->e_branch[4 * e + 1]) {
              up       = std::min(up, hc->e_branch[4 * e + 1]);
              narrowed = true;
            } else if (hc->e_force[2 * e + 1] && lo < hc->e_branch[4 * e + 2]) {
              lo       = std::max(lo, hc->e_branch[4 * e + 2]);
              narrowed = true;
            }
            X.scatter(X.ws.p, {v}, {make_double2(lo, up)});
            X.ws_cert = false;
            if (lo > up) {
              o.rounding_infeasible = 1;
              force                 = true;
              break;
            }
          }
          if (narrowed && !force) {
            BP_CUDA(cudaMemcpyAsync(P.st.bounds, X.ws.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, X.s));
            const auto r = X.propagate_engine(false, {});
            BP_CUDA(cudaMemcpyAsync(X.ws.p, P.st.bounds, sizeof(double2) * n, cudaMemcpyDeviceToDevice, X.s));
            X.ws_cert = r.fixpoint != 0;
            if (X.ws_cert) X.snapshot_ws_activities();
            if (r.status == bp::BP_STATUS_INFEASIBLE) {
              X.ws_infeasible       = true;
              o.rounding_infeasible = 1;
              force                 = true;
            }
            X.drop_fixed();
            continue;
          }
          if (!force) {
            o.rounding_infeasible = 1;
            force                 = true;
          }
          continue;
        }
        if (!recovery && !o.rounding_infeasible) {
          recovery = true;  // backtrack, single-variable mode (rounding.hpp:480-483)
          continue;
        }
        o.rounding_infeasible = 1;
        const int v      = take[0];
        const double val = bp::clampd(pv0[0], H.var_lower[v], H.var_upper[v]);
        committed.push_back({v, val});
        X.scatter(X.ws.p, {v}, {make_double2(val, val)});
        X.ws_cert = false;
        X.drop_fixed();
        if (cfg.repair_enabled && o.repair_attempts < cfg.repair_attempt_cap && !expired()) {
          o.repair_attempts++;  // rounding.hpp:492-504
          if (!X.orig.p && n) X.orig.upload(reinterpret_cast<const double2*>(orig.data()), n);
          std::vector<std::pair<int, double>> rep = committed;
          bp::RunResult rr{};
          if (X.repair(rep, X.orig.p, expired, cfg.repair_shift_cap, &rr)) {
            committed = std::move(rep);
            if (n) BP_CUDA(cudaMemcpyAsync(X.ws.p, P.st.bounds, sizeof(double2) * n, cudaMemcpyDeviceToDevice, X.s));
            X.ws_infeasible       = false;  // ws.clear_infeasible()
            X.ws_cert             = rr.fixpoint != 0;
            if (X.ws_cert) X.snapshot_ws_activities();
            o.rounding_infeasible = 0;
            recovery              = false;
            X.drop_fixed();
          } else {
            force = true;
          }
        } else {
          force = true;
        }
        continue;
      }
      // terminal phase (rounding.hpp:511-528)
      const std::vector<int> take = X.take_first(bulk);
      const auto tb               = X.gather(X.ws, take);
      bp::candidate_values(start_values, take, tb, rng, cfg.random_band, pv0, pv1);
      for (size_t j = 0; j < take.size(); ++j) {
        pv0[j] = bp::clampd(pv0[j], H.var_lower[take[j]], H.var_upper[take[j]]);
        pv1[j] = bp::clampd(pv1[j], H.var_lower[take[j]], H.var_upper[take[j]]);
      }
      const int viol0 = X.count_envelope_violations(take, pv0);
      const int viol1 = viol0 == 0 ? 1 : X.count_envelope_violations(take, pv1);
      const auto& pv  = viol1 < viol0 ? pv1 : pv0;
      std::vector<double2> fx(take.size());
      for (size_t j = 0; j < take.size(); ++j) {
        fx[j] = make_double2(pv[j], pv[j]);
        committed.push_back({take[j], pv[j]});
      }
      X.scatter(X.ws.p, take, fx);
      X.ws_cert = false;
      X.drop_fixed();
    }
    // value extraction (rounding.hpp:533-549)
    std::vector<double> wsb(2 * (size_t)n);
    if (n) BP_CUDA(cudaMemcpy(wsb.data(), X.ws.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) {
      const double v = start_values[i];
      if (!H.is_integer[i]) {
        out_values[i] = bp::clampd(v, H.var_lower[i], H.var_upper[i]);
        continue;
      }
      if (wsb[2 * i] == wsb[2 * i + 1]) out_values[i] = wsb[2 * i];
      else out_values[i] = bp::clampd(std::round(v), H.var_lower[i], H.var_upper[i]);
      if (wsb[2 * i] == wsb[2 * i + 1]) o.set_count++;
    }
    if (TT.on) {
      const char* nm[7] = {"slack_sort", "take+gather+draw", "run_probe", "commit",
                           " probe:warm+meet", " probe:fix", " probe:engine"};
      for (int q = 0; q < 7; ++q)
        fprintf(stderr, "[bp round] %-18s n=%lld total=%.3f s avg=%.1f us\n", nm[q], TT.n[q], TT.t[q],
                TT.n[q] ? 1e6 * TT.t[q] / TT.n[q] : 0.0);
      fprintf(stderr, "[bp round] engine device %.3f s over %lld calls\n", X.dev_ms * 1e-3, X.bp_calls);
      if (X.stats_on) {
        fprintf(stderr, "[bp round] engine rounds per call:");
        for (int q = 0; q < 66; ++q)
          if (X.st_rounds[q]) fprintf(stderr, " %d:%lld", q, X.st_rounds[q]);
        fprintf(stderr, "\n[bp round]  rnd  calls  full%%      |R|          A      |V|          B   gath_us    act_us  tight_us    exp_us (means per call reaching the round)\n");
        for (int q = 0; q < 17; ++q) {
          const double* o = X.st_sum.data() + q * 10;
          if (o[0] == 0) continue;
          fprintf(stderr, "[bp round] %3d%s %7.0f %5.1f %9.0f %10.0f %8.0f %10.0f %9.1f %9.1f %9.1f %9.1f\n", q + 1,
                  q == 16 ? "+" : " ", o[0], 100 * o[1] / o[0], o[2] / o[0], o[3] / o[0], o[4] / o[0],
                  o[5] / o[0], o[6] / o[0], o[7] / o[0], o[8] / o[0], o[9] / o[0]);
        }
      }
    }
    o.completed       = X.n_unset == 0;
    o.bounds_feasible = o.completed && !o.rounding_infeasible && !X.ws_infeasible;
    o.bp_calls        = (int32_t)X.bp_calls;
    o.device_ms       = X.dev_ms;
    *out              = o;
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


}  // namespace

extern "C" {

int bp_propagation_round(bp_problem* p, const double* start_values, const bp_cache* cache,
                         uint64_t seed, double deadline_sec, const bp_rounding_config* cfg_in,
                         double* out_values, bp_rounding_outcome* out)
{
  std::mt19937_64 rng(seed);
  return round_impl(p, start_values, cache, rng, deadline_sec, cfg_in, out_values, out);
}

int bp_propagation_round_rng(bp_problem* p, const double* start_values, const bp_cache* cache,
                             char* rng_state, int64_t rng_state_bytes, double deadline_sec,
                             const bp_rounding_config* cfg, double* out_values,
                             bp_rounding_outcome* out)
{
  if (!rng_state || rng_state_bytes <= 0) {
    bp_set_last_error("null rng state");
    return BP_ERR_INVALID_ARGUMENT;
  }
  std::mt19937_64 rng;
  {
    std::istringstream is(std::string(rng_state, strnlen(rng_state, (size_t)rng_state_bytes)));
    is >> rng;
    if (!is) {
      bp_set_last_error("rng state is not a std::mt19937_64 text representation");
      return BP_ERR_INVALID_ARGUMENT;
    }
  }
  const int rc = round_impl(p, start_values, cache, rng, deadline_sec, cfg, out_values, out);
  if (rc != BP_OK) return rc;
  std::ostringstream os;
  os << rng;
  const std::string st = os.str();
  if ((int64_t)st.size() + 1 > rng_state_bytes) {
    bp_set_last_error("rng state buffer too small (BP_RNG_STATE_BYTES)");
    return BP_ERR_INVALID_ARGUMENT;
  }
  std::memcpy(rng_state, st.c_str(), st.size() + 1);
  return BP_OK;
}

int bp_repair(bp_problem* p, const int32_t* fixed_vars, const double* fixed_vals, int32_t nfixed,
              double deadline_sec, const bp_rounding_config* cfg_in, int32_t* repaired,
              double* out_vals, double* out_bounds2n)
{
  try {
    if (!p || !repaired || nfixed < 0 || (nfixed > 0 && (!fixed_vars || !fixed_vals || !out_vals)) ||
        !out_bounds2n)
      throw std::invalid_argument("null argument");
    bp_rounding_config cfg;
    bp_rounding_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    bp::Problem& P           = bp_problem_impl(p);
    const bp_problem_host& H = bp_problem_hostdata(p);
    const int n              = P.n;
    std::vector<std::pair<int, double>> fixed(nfixed);
    for (int j = 0; j < nfixed; ++j) {
      if (fixed_vars[j] < 0 || fixed_vars[j] >= n) throw std::out_of_range("var out of range");
      fixed[j] = {fixed_vars[j], fixed_vals[j]};
    }
    std::lock_guard<std::mutex> lk(P.mu);
    BP_CUDA(cudaSetDevice(P.device));
    const auto t0 = std::chrono::steady_clock::now();
    auto expired  = [&] {
      if (!(deadline_sec > 0.0)) return false;
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() >= deadline_sec;
    };
    bp::RoundCtx X(P, H);
    std::vector<double> orig(2 * (size_t)n);
    bp_problem_root(p, orig.data());
    X.orig.upload(reinterpret_cast<const double2*>(orig.data()), n);
    bp::RunResult rr{};
    const bool ok = X.repair(fixed, X.orig.p, expired, cfg.repair_shift_cap, &rr);
    *repaired     = ok ? 1 : 0;
    if (ok) {
      for (int j = 0; j < nfixed; ++j) out_vals[j] = fixed[j].second;
      if (n)
        BP_CUDA(cudaMemcpyAsync(out_bounds2n, P.st.bounds, sizeof(double2) * n, cudaMemcpyDeviceToHost, X.s));
      X.sync();
    }
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

int bp_parallel_propagate(bp_problem* p, const double* base2n, int32_t base_infeasible,
                          const int32_t* vars, int32_t nvars, const double* v0, const double* v1,
                          const bp_cache* cache, double* out_bounds2n, int32_t* out_infeasible,
                          int32_t* infeas_count, int32_t* evicted, int32_t* n_evicted,
                          int32_t* fixed_vars, double* fixed_vals, int32_t* n_fixed)
{
  try {
    if (!p || !base2n || !out_bounds2n || !out_infeasible || !infeas_count || !n_evicted || !n_fixed ||
        (nvars > 0 && (!vars || !v0 || !v1 || !evicted || !fixed_vars || !fixed_vals)) || nvars < 0)
      throw std::invalid_argument("null argument");
    bp::Problem& P           = bp_problem_impl(p);
    const bp_problem_host& H = bp_problem_hostdata(p);
    const bp::HostCache* hc  = cache ? bp_cache_host(cache) : nullptr;
    const int n              = P.n;
    for (int j = 0; j < nvars; ++j)
      if (vars[j] < 0 || vars[j] >= n) throw std::out_of_range("var out of range");
    if (hc && hc->n != n) throw std::invalid_argument("cache does not belong to this problem");
    std::lock_guard<std::mutex> lk(P.mu);
    BP_CUDA(cudaSetDevice(P.device));
    bp::RoundCtx X(P, H);
    X.ws.upload(reinterpret_cast<const double2*>(base2n), n);
    X.ws_infeasible = base_infeasible != 0;
    X.ws_cert       = false;  // an arbitrary base: every probe runs the reference's full first round
    X.root.alloc(std::max(n, 1));
    if (hc && n) BP_CUDA(cudaMemcpy(X.root.p, hc->root.data(), sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
    const std::vector<int> vv(vars, vars + nvars);
    for (int q = 0; q < 2; ++q) {
      const double* val = q ? v1 : v0;
      const auto pr     = X.run_probe(vv, std::vector<double>(val, val + nvars), hc);
      if (n)
        BP_CUDA(cudaMemcpyAsync(out_bounds2n + 2 * (size_t)n * q, P.st.bounds, sizeof(double2) * n,
                                cudaMemcpyDeviceToHost, X.s));
      X.sync();
      out_infeasible[q] = pr.infeasible ? 1 : 0;
      infeas_count[q]   = pr.infeas_count;
      n_evicted[q]      = (int32_t)pr.evicted.size();
      std::copy(pr.evicted.begin(), pr.evicted.end(), evicted + (size_t)nvars * q);
      n_fixed[q] = (int32_t)pr.fixed.size();
      for (size_t j = 0; j < pr.fixed.size(); ++j) {
        fixed_vars[(size_t)nvars * q + j] = pr.fixed[j].first;
        fixed_vals[(size_t)nvars * q + j] = pr.fixed[j].second;
      }
    }
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

}  // extern "C"
