// Probing cache: host driver of the batched probe kernel, fallback path, priority order,
// warm-start merge, and (de)serialisation for the multi-GPU gather. C-ABI in include/bp.h.
//
// References: probing.hpp:30-60 make_branch_spec, :105-190 prioritize_probe_vars,
// :225-238 probe_variable, :243-281 build_cache, :292-352 assemble_bulk_warm_start.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bp.h"
#include "bp_engine.cuh"
#include "bp_probe.cuh"
#include "bp_capi_internal.h"

namespace bp {

void HostCache::finalize_stats()
{
  n_probed              = (int)e_var.size();
  n_infeasible_branches = 0;
  for (size_t e = 0; e < e_var.size(); ++e)
    n_infeasible_branches += (e_feas[2 * e] ? 0 : 1) + (e_feas[2 * e + 1] ? 0 : 1);
}

namespace {

// probing.hpp:30-60. Returns 0 (no spec) or kind + 1; s = {down lo, down up, up lo, up up}.
int branch_spec(double lo, double up, double* s)
{
  if (lo == up) return 0;
  if (std::isfinite(lo) && std::isfinite(up)) {
    const double mid = std::ceil((lo + up) / 2.0);
    s[0] = lo; s[1] = mid - 1.0; s[2] = mid; s[3] = up;
    return 1;
  }
  if (std::isfinite(lo)) {
    s[0] = lo; s[1] = lo; s[2] = lo + 1.0; s[3] = up;
    return 2;
  }
  if (std::isfinite(up)) {
    s[0] = lo; s[1] = up - 1.0; s[2] = up; s[3] = up;
    return 3;
  }
  return 0;
}


Limits default_limits()
{
  Limits l;
  l.max_rounds    = 64;
  l.time_limit    = INFINITY;
  l.abs_threshold = 1e-7;
  l.rel_threshold = 1e-4;
  l.incremental   = 1;
  return l;
}

// Batched branches' deltas from the kernel's pool (allocation order) into task order: task t's
// deltas go to [scan[t], scan[t] + cnt[t]) (scan = exclusive sum of the counts). One copy to
// the host then yields the cache's delta arrays directly.
__global__ void k_pack_pool(int nt, const int* cnt, const long long* off, const int* scan,
                            const int* pvar, const double* plo, const double* pup, int* ovar,
                            double* olo, double* oup)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const int c = cnt[t];
    const long long o = off[t];
    const int d       = scan[t];
    for (int j = 0; j < c; ++j) {
      ovar[d + j] = pvar[o + j];
      olo[d + j]  = plo[o + j];
      oup[d + j]  = pup[o + j];
    }
  }
}

}  // namespace

// Probes `vars` (both branches each) from `root`; entries follow probe_variable semantics.
// Pinned host staging that only grows (async copies at full PCIe / C2C rate).
struct PinBuf {
  void* p  = nullptr;
  size_t n = 0;
  PinBuf() = default;
  PinBuf(const PinBuf&) = delete;
  PinBuf& operator=(const PinBuf&) = delete;
  ~PinBuf()
  {
    if (p) cudaFreeHost(p);
  }
  template <class T>
  T* get(size_t count)
  {
    const size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
    if (n < bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      n = bytes + bytes / 4;
      BP_CUDA(cudaMallocHost(&p, n));
    }
    return static_cast<T*>(p);
  }
};

template <class T>
void grow(DBuf<T>& b, size_t k)
{
  if (b.n < k) b.alloc(k + k / 4);
}

// Probing scratch of one problem, kept across calls (no cudaMalloc / cudaFree per batch).
struct ProbeWs {
  DBuf<double2> d_root;
  DBuf<int> dvar, dcur, dstat, dcnt, dscan, qvar, pvar;
  DBuf<double> dlo, dup, qlo, qup, plo, pup;
  DBuf<long long> doff;
  DBuf<unsigned long long> dpc, dwork;
  DBuf<unsigned char> dtmp;
  PinBuf h_var, h_lo, h_up, h_st, h_cn, h_qv, h_ql, h_qu, h_root;
  std::vector<int> tv, tslot;  // task lists, reused across calls (no first-touch page faults)
  std::vector<double> tlo, tup;
  DBuf<char> blk;              // dense per-block state of the block-per-branch kernel
  BlockScratch bs;
};

// The block kernel's scratch: as many blocks as one per SM, within a quarter of the free memory
// (and at most 24 GB); zeroed once -- its stamps compare against tags that only grow.
BlockScratch& block_scratch(Problem& P, ProbeWs& W)
{
  if (W.bs.base && W.bs.n == P.n && W.bs.m == P.m) return W.bs;
  int sms = 0;
  BP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device));
  size_t freeb = 0, totb = 0;
  BP_CUDA(cudaMemGetInfo(&freeb, &totb));
  const size_t per = (block_scratch_bytes(P.n, P.m) + 255) / 256 * 256;
  const size_t cap = std::min<size_t>(freeb / 4, 24ull << 30);
  const int nb     = (int)std::max<size_t>(1, std::min<size_t>((size_t)sms, cap / per));
  W.blk.alloc(per * nb);
  BP_CUDA(cudaMemset(W.blk.p, 0, per * nb));
  W.bs.nblocks = nb;
  W.bs.n       = P.n;
  W.bs.m       = P.m;
  W.bs.stride  = per;
  W.bs.base    = W.blk.p;
  for (int b = 0; b < nb; ++b) {  // tags start at 1 (0 = never stamped)
    const unsigned one = 1;
    BP_CUDA(cudaMemcpy(W.bs.for_block(b).tagc, &one, sizeof(one), cudaMemcpyHostToDevice));
  }
  return W.bs;
}

HostCache probe_vars(Problem& P, const std::vector<double>& root, const std::vector<int>& vars,
                     double budget_sec)
{
  const auto t_start = std::chrono::steady_clock::now();
  auto elapsed       = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  BP_CUDA(cudaSetDevice(P.device));
  cudaStream_t s = P.stream;
  const int n    = P.n;
  HostCache C;
  C.n    = n;
  C.root = root;
  C.entry_of.assign(n, -1);
  if (!P.probe_ws) P.probe_ws = std::make_shared<ProbeWs>();
  ProbeWs& W            = *static_cast<ProbeWs*>(P.probe_ws.get());
  DBuf<double2>& d_root = W.d_root;
  grow(d_root, (size_t)std::max(n, 1));
  if (n) {  // through pinned staging (a pageable 16n-byte copy is several times slower)
    double* hr = W.h_root.get<double>(2 * (size_t)n);
    std::memcpy(hr, root.data(), sizeof(double) * 2 * n);
    BP_CUDA(cudaMemcpyAsync(d_root.p, hr, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, s));
  }
  // certification: one full round from the root changes nothing (fixpoint) -> frontier starts
  // are exact. Leaves the root activities in P.st.rec / aux.
  const double t_up = elapsed();
  bool certified = false;
  if (n) {
    BP_CUDA(cudaMemcpyAsync(P.st.bounds, d_root.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
    BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(Ctl), s));
    Limits one       = default_limits();
    one.max_rounds   = 1;
    const RunResult r = run_engine(P, MODE_PROPAGATE, true, one, s);
    certified         = r.status == BP_STATUS_UNCHANGED;
  }
  C.certified = certified;
  const double t_cert = elapsed();

  // tasks: down then up branch of every var with a spec (probing.hpp:228-234)
  std::vector<int>& tv    = W.tv;
  std::vector<int>& tslot = W.tslot;
  std::vector<double>& tlo = W.tlo;
  std::vector<double>& tup = W.tup;
  // (sized up front and filled by index: this loop runs over every candidate on the host)
  const size_t nv = vars.size();
  tv.resize(2 * nv);
  tslot.resize(2 * nv);
  tlo.resize(2 * nv);
  tup.resize(2 * nv);
  C.e_var.resize(nv);
  C.e_kind.assign(nv, 0);
  C.e_feas.assign(2 * nv, 1);
  C.e_force.assign(2 * nv, 0);
  C.e_branch.assign(4 * nv, 0.0);
  int ne_ = 0;
  size_t nt = 0;
  for (int v : vars) {
    if (v < 0 || v >= n) throw std::out_of_range("probe var out of range");
    int e = C.entry_of[v];
    if (e < 0) {
      e             = ne_++;
      C.entry_of[v] = e;
      C.e_var[e]    = v;
    }
    double sp[4];
    const int kind = branch_spec(root[2 * v], root[2 * v + 1], sp);
    if (!kind) continue;  // default entry: no spec (probing.hpp:231)
    C.e_kind[e] = kind - 1;
    for (int q = 0; q < 4; ++q) C.e_branch[4 * e + q] = sp[q];
    for (int side = 0; side < 2; ++side, ++nt) {
      tv[nt]    = v;
      tlo[nt]   = sp[2 * side];
      tup[nt]   = sp[2 * side + 1];
      tslot[nt] = 2 * e + side;
    }
  }
  tv.resize(nt);
  tslot.resize(nt);
  tlo.resize(nt);
  tup.resize(nt);
  C.e_var.resize(ne_);
  C.e_kind.resize(ne_);
  C.e_feas.resize(2 * (size_t)ne_);
  C.e_force.resize(2 * (size_t)ne_);
  C.e_branch.resize(4 * (size_t)ne_);
  static const bool prof = getenv("BP_PROBE_PROFILE") != nullptr;
  const double t_tasks = elapsed();
  const int ne = (int)C.e_var.size();
  // per branch: kernel result (range of the flat host pool) or index of an engine branch
  struct BrRef {
    long long pool_off = -1;
    int pool_cnt       = 0;
    int feasible       = 1;
  };
  std::vector<BrRef> res(2 * (size_t)ne);
  std::vector<int> hp_var;  // batched branches' deltas (flat, by chunk)
  std::vector<double> hp_lo, hp_up;
  std::vector<uint8_t> done(2 * (size_t)ne, 0);
  for (int e = 0; e < ne; ++e) done[2 * e] = done[2 * e + 1] = 1;
  for (int slot : tslot) done[slot] = 0;

  const int ntask = (int)tv.size();
  auto& dvar  = W.dvar;
  auto& dcur  = W.dcur;
  auto& dstat = W.dstat;
  auto& dcnt  = W.dcnt;
  auto& dlo   = W.dlo;
  auto& dup   = W.dup;
  auto& doff  = W.doff;
  auto& dpc   = W.dpc;
  auto& dscan = W.dscan;
  auto& qvar  = W.qvar;
  auto& qlo   = W.qlo;
  auto& qup   = W.qup;
  auto& dtmp  = W.dtmp;
  auto& pvar  = W.pvar;
  auto& plo   = W.plo;
  auto& pup   = W.pup;
  // chunks small enough for the time budget to be honoured between them
  const int chunk = std::isfinite(budget_sec) && budget_sec < 1e6 ? (1 << 14) : (1 << 20);
  grow(pvar, 4ull * std::min(std::max(ntask, 1), chunk) + 4096);
  grow(plo, pvar.n);
  grow(pup, pvar.n);
  long long pool_cap = (long long)std::min(pvar.n, std::min(plo.n, pup.n));
  ProbeRoot R{d_root.p, P.st.rec, P.st.aux};
  // One batch of tasks (indices into tv / tlo / tup) on the warp kernel (block = false) or the
  // block-per-branch kernel (block = true): results into `res` / the flat host pool; the tasks the
  // warp kernel could not hold (overlay overflow) are appended to `overflow`.
  std::vector<int> hidx;
  auto run_batch = [&](const int* tidx, int nt, bool block, int full_first, std::vector<int>& overflow) {
    const double tb0 = elapsed();
    grow(dvar, nt);
    grow(dlo, nt);
    grow(dup, nt);
    grow(dcur, 1);
    grow(dstat, nt);
    grow(dcnt, nt);
    grow(doff, nt);
    grow(dpc, 1);
    {
      int* hv    = W.h_var.get<int>(nt);
      double* hl = W.h_lo.get<double>(nt);
      double* hu = W.h_up.get<double>(nt);
      for (int j = 0; j < nt; ++j) {
        hv[j] = tv[tidx[j]];
        hl[j] = tlo[tidx[j]];
        hu[j] = tup[tidx[j]];
      }
      BP_CUDA(cudaMemcpyAsync(dvar.p, hv, sizeof(int) * nt, cudaMemcpyHostToDevice, s));
      BP_CUDA(cudaMemcpyAsync(dlo.p, hl, sizeof(double) * nt, cudaMemcpyHostToDevice, s));
      BP_CUDA(cudaMemcpyAsync(dup.p, hu, sizeof(double) * nt, cudaMemcpyHostToDevice, s));
    }
    for (;;) {
      BP_CUDA(cudaMemsetAsync(dcur.p, 0, sizeof(int), s));
      BP_CUDA(cudaMemsetAsync(dpc.p, 0, sizeof(unsigned long long), s));
      grow(W.dwork, 5);
      BP_CUDA(cudaMemsetAsync(W.dwork.p, 0, 5 * sizeof(unsigned long long), s));
      ProbeBatch B{nt, dvar.p, dlo.p, dup.p, dcur.p, dstat.p, dcnt.p, doff.p, dpc.p,
                   pool_cap, pvar.p, plo.p, pup.p, W.dwork.p};
      BP_CUDA(cudaEventRecord(P.ev0, s));
      if (block) probe_block_launch(P, R, B, default_limits(), block_scratch(P, W), full_first, s);
      else probe_launch(P, R, B, default_limits(), s);
      BP_CUDA(cudaEventRecord(P.ev1, s));
      unsigned long long used = 0;
      const double tb1 = elapsed();
      BP_CUDA(cudaMemcpyAsync(&used, dpc.p, sizeof(used), cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaStreamSynchronize(s));
      const double tb2 = elapsed();
      float ms = 0.f;
      BP_CUDA(cudaEventElapsedTime(&ms, P.ev0, P.ev1));
      C.probe_ms += ms;
      if ((long long)used > pool_cap) {  // grow the delta pool and rerun the batch
        pool_cap = (long long)used + 4096;
        pvar.alloc(pool_cap);
        plo.alloc(pool_cap);
        pup.alloc(pool_cap);
        continue;
      }
      {
        unsigned long long wkh[5];
        BP_CUDA(cudaMemcpy(wkh, W.dwork.p, sizeof(wkh), cudaMemcpyDeviceToHost));
        for (int q = 0; q < 5; ++q) C.work[q] += wkh[q];
      }
      int* st = W.h_st.get<int>(nt);
      int* cn = W.h_cn.get<int>(nt);
      BP_CUDA(cudaMemcpyAsync(st, dstat.p, sizeof(int) * nt, cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaMemcpyAsync(cn, dcnt.p, sizeof(int) * nt, cudaMemcpyDeviceToHost, s));
      // the batch's deltas in task order (device scan + pack), appended to the flat host pool
      const long long hbase = (long long)hp_var.size();
      int* hqv    = nullptr;
      double* hql = nullptr;
      double* hqu = nullptr;
      if (used) {
        grow(dscan, nt);
        size_t nb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, nb, dcnt.p, dscan.p, nt, s);
        if (nb > dtmp.n) dtmp.alloc(nb);
        nb = dtmp.n;
        cub::DeviceScan::ExclusiveSum(dtmp.p, nb, dcnt.p, dscan.p, nt, s);
        grow(qvar, used);
        grow(qlo, used);
        grow(qup, used);
        k_pack_pool<<<(int)std::min<long long>(4096, (nt + 255) / 256), 256, 0, s>>>(
            nt, dcnt.p, doff.p, dscan.p, pvar.p, plo.p, pup.p, qvar.p, qlo.p, qup.p);
        BP_CUDA(cudaGetLastError());
        hqv = W.h_qv.get<int>(used);
        hql = W.h_ql.get<double>(used);
        hqu = W.h_qu.get<double>(used);
        BP_CUDA(cudaMemcpyAsync(hqv, qvar.p, sizeof(int) * used, cudaMemcpyDeviceToHost, s));
        BP_CUDA(cudaMemcpyAsync(hql, qlo.p, sizeof(double) * used, cudaMemcpyDeviceToHost, s));
        BP_CUDA(cudaMemcpyAsync(hqu, qup.p, sizeof(double) * used, cudaMemcpyDeviceToHost, s));
      }
      BP_CUDA(cudaStreamSynchronize(s));
      if (used) {  // appended from the pinned staging (one copy, no zero-fill of a resize)
        hp_var.insert(hp_var.end(), hqv, hqv + used);
        hp_lo.insert(hp_lo.end(), hql, hql + used);
        hp_up.insert(hp_up.end(), hqu, hqu + used);
      }
      const double tb3 = elapsed();
      if (prof)
        fprintf(stderr, "[bp probe] %s batch of %d: uploads+launch %.2f ms, kernel wait %.2f ms, pack+D2H %.2f ms\n",
                block ? "block" : "warp", nt, 1e3 * (tb1 - tb0), 1e3 * (tb2 - tb1), 1e3 * (tb3 - tb2));
      long long run = hbase;
      for (int j = 0; j < nt; ++j) {
        const int t = tidx[j];
        BrRef& br   = res[tslot[t]];
        if (st[j] == 0) {
          br.feasible    = 1;
          br.pool_off    = run;
          br.pool_cnt    = cn[j];
          run += cn[j];
          done[tslot[t]] = 1;
        } else if (st[j] == 1) {
          br.feasible    = 0;
          done[tslot[t]] = 1;
        } else {
          overflow.push_back(t);
        }
        if (block && st[j] <= 1) C.n_block++;
      }
      return;
    }
  };
  std::vector<int> fallback;  // tasks for the block-per-branch kernel
  if (certified) {
    for (int t0 = 0; t0 < ntask; t0 += chunk) {
      if (t0 > 0 && elapsed() >= budget_sec) break;
      const int nt = std::min(chunk, ntask - t0);
      hidx.resize(nt);
      std::iota(hidx.begin(), hidx.end(), t0);
      run_batch(hidx.data(), nt, false, 0, fallback);
    }
  } else {
    for (int t = 0; t < ntask; ++t) fallback.push_back(t);
  }
  const double t_batch = elapsed();
  // block-per-branch kernel: the warp kernel's overflows (frontier start from the certified root)
  // or every branch of an uncertified root (full first round)
  for (size_t f0 = 0; f0 < fallback.size(); f0 += chunk) {
    if (elapsed() >= budget_sec) break;
    const int nt = (int)std::min<size_t>(chunk, fallback.size() - f0);
    std::vector<int> again;
    run_batch(fallback.data() + f0, nt, true, certified ? 0 : 1, again);
    if (!again.empty()) throw std::runtime_error("block-per-branch probing returned an overflow");
  }
  const double t_fallback = elapsed();
  bool all_done = C.n_fallback == 0 && fallback.empty() && C.n_block == 0;
  for (size_t t = 1; t < tslot.size() && all_done; ++t) all_done = tslot[t] > tslot[t - 1];  // no repeated vars
  for (int e = 0; e < ne && all_done; ++e) all_done = done[2 * e] && done[2 * e + 1];
  if (all_done) {
    // every branch came from the batched kernel: the flat pool is already the cache's delta
    // arrays in entry order (down, up), so only the per-entry tables are filled
    HostCache out;
    out.n          = n;
    out.root       = root;
    out.certified  = certified;
    out.probe_ms   = C.probe_ms;
    out.n_fallback = 0;
    out.n_block    = C.n_block;
    std::copy(C.work, C.work + 5, out.work);
    out.entry_of   = std::move(C.entry_of);
    out.e_var      = std::move(C.e_var);
    out.e_kind     = std::move(C.e_kind);
    out.e_branch   = std::move(C.e_branch);
    out.e_feas.resize(2 * (size_t)ne);
    out.e_force.resize(2 * (size_t)ne);
    out.d_off.resize(2 * (size_t)ne + 1);
    long long o = 0;
    for (int e = 0; e < ne; ++e) {
      const BrRef& dn  = res[2 * e];
      const BrRef& upb = res[2 * e + 1];
      out.e_feas[2 * e]      = (uint8_t)dn.feasible;
      out.e_feas[2 * e + 1]  = (uint8_t)upb.feasible;
      out.e_force[2 * e]     = (uint8_t)(!upb.feasible && dn.feasible);  // forces_down
      out.e_force[2 * e + 1] = (uint8_t)(!dn.feasible && upb.feasible);  // forces_up
      out.d_off[2 * e]       = o;
      o += dn.pool_off >= 0 ? dn.pool_cnt : 0;
      out.d_off[2 * e + 1] = o;
      o += upb.pool_off >= 0 ? upb.pool_cnt : 0;
    }
    out.d_off[2 * (size_t)ne] = o;
    out.d_var = std::move(hp_var);
    out.d_lo  = std::move(hp_lo);
    out.d_up  = std::move(hp_up);
    out.finalize_stats();
    if (prof)
      fprintf(stderr, "[bp probe] setup+cert %.2f ms (upload %.2f, certification %.2f, tasks %.2f), batches %.2f ms (device %.2f ms), assemble %.2f ms\n",
              1e3 * t_tasks, 1e3 * t_up, 1e3 * (t_cert - t_up), 1e3 * (t_tasks - t_cert),
              1e3 * (t_batch - t_tasks), C.probe_ms, 1e3 * (elapsed() - t_fallback));
    return out;
  }
  // assemble (entries whose branches were not both computed within the budget are dropped)
  HostCache out;
  out.n         = n;
  out.root      = root;
  out.certified = certified;
  out.probe_ms  = C.probe_ms;
  out.n_fallback = C.n_fallback;
  out.n_block    = C.n_block;
  std::copy(C.work, C.work + 5, out.work);
  out.entry_of.assign(n, -1);
  out.d_off.reserve(2 * (size_t)ne + 1);
  out.d_off.push_back(0);
  out.e_var.reserve(ne);
  out.e_kind.reserve(ne);
  out.e_branch.reserve(4 * (size_t)ne);
  out.e_feas.reserve(2 * (size_t)ne);
  out.e_force.reserve(2 * (size_t)ne);
  out.d_var.reserve(hp_var.size());
  out.d_lo.reserve(hp_var.size());
  out.d_up.reserve(hp_var.size());
  for (int e = 0; e < ne; ++e) {
    if (!done[2 * e] || !done[2 * e + 1]) continue;
    const int v    = C.e_var[e];
    const int ne2  = (int)out.e_var.size();
    out.entry_of[v] = ne2;
    out.e_var.push_back(v);
    out.e_kind.push_back(C.e_kind[e]);
    for (int q = 0; q < 4; ++q) out.e_branch.push_back(C.e_branch[4 * e + q]);
    const BrRef& dn  = res[2 * e];
    const BrRef& upb = res[2 * e + 1];
    out.e_feas.push_back((uint8_t)dn.feasible);
    out.e_feas.push_back((uint8_t)upb.feasible);
    out.e_force.push_back((uint8_t)(!upb.feasible && dn.feasible));  // forces_down
    out.e_force.push_back((uint8_t)(!dn.feasible && upb.feasible));  // forces_up
    for (const BrRef* b : {&dn, &upb}) {
      if (b->pool_off >= 0) {
        const long long o = b->pool_off, cnt = b->pool_cnt;
        out.d_var.insert(out.d_var.end(), hp_var.begin() + o, hp_var.begin() + o + cnt);
        out.d_lo.insert(out.d_lo.end(), hp_lo.begin() + o, hp_lo.begin() + o + cnt);
        out.d_up.insert(out.d_up.end(), hp_up.begin() + o, hp_up.begin() + o + cnt);
      }
      out.d_off.push_back((long long)out.d_var.size());
    }
  }
  out.finalize_stats();
  if (prof)
    fprintf(stderr, "[bp probe] setup+cert %.2f ms, batches %.2f ms (device %.2f ms), fallback %.2f ms, assemble %.2f ms\n",
            1e3 * t_tasks, 1e3 * (t_batch - t_tasks), C.probe_ms, 1e3 * (t_fallback - t_batch),
            1e3 * (elapsed() - t_fallback));
  return out;
}

__global__ void k_gather_u64(const unsigned long long* src, const int* idx, int k, unsigned long long* dst)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) dst[j] = src[idx[j]];
}
__global__ void k_gather_u32(const unsigned* src, const int* idx, int k, unsigned* dst)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) dst[j] = src[idx[j]];
}
__global__ void k_gather_i32(const int* src, const int* idx, int k, int* dst)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) dst[j] = src[idx[j]];
}

// probing.hpp:105-190 on the device: one warp per integer variable folds its column's keys
// (count, max and min are order-independent here: every folded value is positive, so there are
// no signed-zero ties), then three stable radix passes give the lexicographic stable order.
__global__ void k_prio_keys(DevProblem P, const RowRec* rec, const double2* aux,
                            const double2* bounds, const int* ivar, int k, unsigned* k_viol,
                            unsigned long long* k_maxv, unsigned long long* k_slack, int* vals)
{
  constexpr double kFeasTol = 1e-6;  // common.hpp:20
  const int lane  = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < k; j += warps) {
    const int i  = ivar[j];
    const int e0 = P.col_start[i], e1 = P.col_start[i + 1];
    bool pos = false, neg = false;
    for (int e = e0 + lane; e < e1; e += 32) (P.col_val[e] > 0 ? pos : neg) = true;
    const bool both = __any_sync(0xffffffffu, pos) && __any_sync(0xffffffffu, neg);
    const double2 b = bounds[i];
    const double lo = b.x, up = b.y;
    int viol        = 0;
    double maxv     = 0.0, slk = INFINITY;
    for (int e = e0 + lane; e < e1; e += 32) {
      const int r    = P.col_row[e];
      const double a = P.col_val[e];
      const RowRec q = rec[r];
      double mnf, mxf;
      int nmn, nmx;
      decode_rec(q, aux, r, mnf, nmn, mxf, nmx);
      if (both) {
        const double min_c = a > 0 ? __dmul_rn(a, lo) : __dmul_rn(a, up);
        const double max_c = a > 0 ? __dmul_rn(a, up) : __dmul_rn(a, lo);
        const bool min_inf = a > 0 ? lo == -INFINITY : up == INFINITY;
        const bool max_inf = a > 0 ? up == INFINITY : lo == -INFINITY;
        if (isfinite(q.g) && nmn - (min_inf ? 1 : 0) == 0) {
          const double fm = max_inf ? INFINITY : __dadd_rn(__dsub_rn(mnf, min_inf ? 0.0 : min_c), max_c);
          if (fm > __dadd_rn(q.g, kFeasTol)) {
            ++viol;
            const double d = __dsub_rn(fm, q.g);
            maxv           = (maxv < d) ? d : maxv;
          }
        }
        if (isfinite(q.h) && nmx - (max_inf ? 1 : 0) == 0) {
          const double fx = min_inf ? -INFINITY : __dadd_rn(__dsub_rn(mxf, max_inf ? 0.0 : max_c), min_c);
          if (fx < __dsub_rn(q.h, kFeasTol)) {
            ++viol;
            const double d = __dsub_rn(q.h, fx);
            maxv           = (maxv < d) ? d : maxv;
          }
        }
      }
      if (isfinite(q.g) && nmn == 0) {
        const double sl = __dsub_rn(q.g, mnf);
        if (sl > 0.0) {
          const double u = __ddiv_rn(fabs(a), sl);
          slk            = (u < slk) ? u : slk;
        }
      }
      if (isfinite(q.h) && nmx == 0) {
        const double sl = __dsub_rn(mxf, q.h);
        if (sl > 0.0) {
          const double u = __ddiv_rn(fabs(a), sl);
          slk            = (u < slk) ? u : slk;
        }
      }
    }
    for (int o = 16; o; o >>= 1) {
      viol += __shfl_xor_sync(0xffffffffu, viol, o);
      const double m = __shfl_xor_sync(0xffffffffu, maxv, o);
      const double s = __shfl_xor_sync(0xffffffffu, slk, o);
      maxv           = (maxv < m) ? m : maxv;
      slk            = (s < slk) ? s : slk;
    }
    if (lane == 0) {
      k_viol[j]  = (unsigned)viol;
      k_maxv[j]  = (unsigned long long)__double_as_longlong(maxv);  // >= +0.0: bits order like values
      k_slack[j] = (unsigned long long)__double_as_longlong(slk);   // > 0 or +inf (or +0 on underflow)
      vals[j]    = i;
    }
  }
}

// probing.hpp:292-352 over the flat cache. Returns merged bounds; fills conflicts / evicted.
void warm_start(const HostCache& C, const int* vars, const double* vals, int na,
                std::vector<double>& bounds, std::vector<int>& conflicts, std::vector<int>& evicted)
{
  bounds = C.root;
  conflicts.clear();
  evicted.clear();
  std::vector<int> last_writer(C.n, -1);
  std::vector<uint8_t> ev(C.n, 0);
  struct Undo {
    int var;
    double lo, up;
    int writer;
  };
  std::vector<Undo> undo;
  for (int j = 0; j < na; ++j) {
    const int v = vars[j];
    const int e = (v >= 0 && v < C.n) ? C.entry_of[v] : -1;
    if (e < 0) continue;
    const int side = (vals[j] <= C.e_branch[4 * e + 1]) ? 0 : 1;
    if (!C.e_feas[2 * e + side]) {
      conflicts.push_back(v);
      conflicts.push_back(v);
      if (!ev[v]) {
        ev[v] = 1;
        evicted.push_back(v);
      }
      continue;
    }
    undo.clear();
    bool conflict   = false;
    int conflicting = -1;
    for (long long d = C.d_off[2 * e + side]; d < C.d_off[2 * e + side + 1]; ++d) {
      const int dv    = C.d_var[d];
      const double cl = bounds[2 * dv], cu = bounds[2 * dv + 1];
      const double nl = (cl < C.d_lo[d]) ? C.d_lo[d] : cl;  // std::max(cur, delta)
      const double nu = (C.d_up[d] < cu) ? C.d_up[d] : cu;  // std::min(cur, delta)
      if (nl > nu + 1e-9) {
        conflict    = true;
        conflicting = last_writer[dv] >= 0 ? last_writer[dv] : v;
        break;
      }
      if (nl != cl || nu != cu) {
        undo.push_back({dv, cl, cu, last_writer[dv]});
        bounds[2 * dv]     = nl;
        bounds[2 * dv + 1] = nu;
        last_writer[dv]    = v;
      }
    }
    if (conflict) {
      for (auto it = undo.rbegin(); it != undo.rend(); ++it) {
        bounds[2 * it->var]     = it->lo;
        bounds[2 * it->var + 1] = it->up;
        last_writer[it->var]    = it->writer;
      }
      conflicts.push_back(conflicting);
      conflicts.push_back(v);
      if (!ev[v]) {
        ev[v] = 1;
        evicted.push_back(v);
      }
    }
  }
}

// Sparse form of the same merge: only the variables whose merged bounds differ from the root are
// returned (O(bulk deltas) instead of an O(n) copy of the root per call).
void warm_start_sparse(const HostCache& C, const int* vars, const double* vals, int na,
                       std::vector<int>& dv, std::vector<double>& dl, std::vector<double>& du,
                       std::vector<int>& conflicts, std::vector<int>& evicted)
{
  thread_local std::vector<double> cur;
  thread_local std::vector<int> writer;
  thread_local std::vector<uint8_t> has, ev;
  thread_local std::vector<int> touched;
  if ((int)has.size() != C.n) {
    cur.assign(2 * (size_t)C.n, 0.0);
    writer.assign(C.n, -1);
    has.assign(C.n, 0);
    ev.assign(C.n, 0);
  }
  touched.clear();
  dv.clear();
  dl.clear();
  du.clear();
  conflicts.clear();
  evicted.clear();
  auto touch = [&](int v) {
    if (!has[v]) {
      has[v]         = 1;
      cur[2 * v]     = C.root[2 * v];
      cur[2 * v + 1] = C.root[2 * v + 1];
      touched.push_back(v);
    }
  };
  struct Undo {
    int var;
    double lo, up;
    int writer;
  };
  std::vector<Undo> undo;
  for (int j = 0; j < na; ++j) {
    const int v = vars[j];
    const int e = (v >= 0 && v < C.n) ? C.entry_of[v] : -1;
    if (e < 0) continue;
    const int side = (vals[j] <= C.e_branch[4 * e + 1]) ? 0 : 1;
    if (!C.e_feas[2 * e + side]) {
      conflicts.push_back(v);
      conflicts.push_back(v);
      touch(v);
      if (!ev[v]) {
        ev[v] = 1;
        evicted.push_back(v);
      }
      continue;
    }
    undo.clear();
    bool conflict   = false;
    int conflicting = -1;
    for (long long d = C.d_off[2 * e + side]; d < C.d_off[2 * e + side + 1]; ++d) {
      const int x = C.d_var[d];
      touch(x);
      const double cl = cur[2 * x], cu = cur[2 * x + 1];
      const double nl = (cl < C.d_lo[d]) ? C.d_lo[d] : cl;
      const double nu = (C.d_up[d] < cu) ? C.d_up[d] : cu;
      if (nl > nu + 1e-9) {
        conflict    = true;
        conflicting = writer[x] >= 0 ? writer[x] : v;
        break;
      }
      if (nl != cl || nu != cu) {
        undo.push_back({x, cl, cu, writer[x]});
        cur[2 * x]     = nl;
        cur[2 * x + 1] = nu;
        writer[x]      = v;
      }
    }
    if (conflict) {
      for (auto it = undo.rbegin(); it != undo.rend(); ++it) {
        cur[2 * it->var]     = it->lo;
        cur[2 * it->var + 1] = it->up;
        writer[it->var]      = it->writer;
      }
      conflicts.push_back(conflicting);
      conflicts.push_back(v);
      touch(v);
      if (!ev[v]) {
        ev[v] = 1;
        evicted.push_back(v);
      }
    }
  }
  for (int x : touched) {
    if (cur[2 * x] != C.root[2 * x] || cur[2 * x + 1] != C.root[2 * x + 1]) {
      dv.push_back(x);
      dl.push_back(cur[2 * x]);
      du.push_back(cur[2 * x + 1]);
    }
    has[x]    = 0;
    writer[x] = -1;
    ev[x]     = 0;
  }
}

}  // namespace bp

const bp::HostCache* bp_cache_host(const bp_cache* c);

// ------------------------------------------------------------------ C-ABI

struct bp_cache {
  bp::HostCache c;
};

const bp::HostCache* bp_cache_host(const bp_cache* c) { return &c->c; }
bp_cache* bp_cache_adopt(bp::HostCache&& c)
{
  auto* h = new bp_cache();
  h->c    = std::move(c);
  return h;
}

namespace {

template <class F>
int cguard(F&& f)
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

void need(bool ok, const char* what)
{
  if (!ok) throw std::invalid_argument(what);
}

}  // namespace

extern "C" {

int bp_probe_variables(bp_problem* p, const double* root2n, const int32_t* vars, int32_t nvars,
                       bp_cache** out)
{
  return cguard([&] {
    need(p && out && (nvars == 0 || vars), "null argument");
    bp::Problem& P = bp_problem_impl(p);
    std::lock_guard<std::mutex> lk(P.mu);
    std::vector<double> root(2 * (size_t)P.n);
    if (root2n) std::memcpy(root.data(), root2n, sizeof(double) * root.size());
    else bp_problem_root(p, root.data());
    std::vector<int> v(vars, vars + nvars);
    auto c = std::make_unique<bp_cache>();
    c->c   = bp::probe_vars(P, root, v, INFINITY);
    *out   = c.release();
  });
}

int bp_prioritize_probe_vars(bp_problem* p, int32_t* order, int32_t* n_order)
{
  return cguard([&] {
    need(p && order && n_order, "null argument");
    bp::Problem& P           = bp_problem_impl(p);
    const bp_problem_host& H = bp_problem_hostdata(p);
    std::lock_guard<std::mutex> lk(P.mu);
    BP_CUDA(cudaSetDevice(P.device));
    cudaStream_t s = P.stream;
    std::vector<int> ivar;
    for (int i = 0; i < P.n; ++i)
      if (H.is_integer[i]) ivar.push_back(i);
    const int k = (int)ivar.size();
    *n_order    = k;
    if (k == 0) return;
    // compute_activities of the original bounds (probing.hpp:107-109) into P.st.rec / aux
    std::vector<double> root(2 * (size_t)P.n);
    bp_problem_root(p, root.data());
    BP_CUDA(cudaMemcpyAsync(P.st.bounds, root.data(), sizeof(double) * root.size(), cudaMemcpyHostToDevice, s));
    BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(bp::Ctl), s));
    bp::Limits lim{};
    lim.max_rounds    = 64;
    lim.time_limit    = INFINITY;
    lim.abs_threshold = 1e-7;
    lim.rel_threshold = 1e-4;
    lim.incremental   = 1;
    bp::run_engine(P, bp::MODE_ACTIVITY, true, lim, s);
    bp::DBuf<int> d_ivar, va, vb;
    bp::DBuf<unsigned> kv, kv2;
    bp::DBuf<unsigned long long> km, ks, k64;
    d_ivar.alloc(k);
    va.alloc(k);
    vb.alloc(k);
    kv.alloc(k);
    kv2.alloc(k);
    km.alloc(k);
    ks.alloc(k);
    k64.alloc(k);
    BP_CUDA(cudaMemcpyAsync(d_ivar.p, ivar.data(), sizeof(int) * k, cudaMemcpyHostToDevice, s));
    const int blocks = (int)std::min<long long>(148LL * 16, ((long long)k * 32 + 255) / 256);
    bp::k_prio_keys<<<blocks, 256, 0, s>>>(P.dev(), P.st.rec, P.st.aux, P.st.bounds, d_ivar.p, k,
                                           kv.p, km.p, ks.p, va.p);
    BP_CUDA(cudaGetLastError());
    // stable lexicographic sort (probing.hpp:176-180): least significant key first; each pass
    // carries the var ids and the remaining keys' positions through a permutation.
    bp::DBuf<int> perm, perm2;
    perm.alloc(k);
    perm2.alloc(k);
    bp::DBuf<unsigned char> tmp;
    size_t need_b = 0, have = 0;
    auto grow = [&](size_t nb) {
      if (nb > tmp.n) tmp.alloc(nb);
      have = tmp.n;
    };
    // pass 1: min_unit_slack ascending; values = positions 0..k-1 (va holds var ids by position)
    std::vector<int> iota(k);
    std::iota(iota.begin(), iota.end(), 0);
    bp::DBuf<int> pos0;
    pos0.upload(iota);
    cub::DeviceRadixSort::SortPairs(nullptr, need_b, ks.p, k64.p, pos0.p, perm.p, k, 0, 64, s);
    grow(need_b);
    cub::DeviceRadixSort::SortPairs(tmp.p, have, ks.p, k64.p, pos0.p, perm.p, k, 0, 64, s);
    // pass 2: max_violation descending over the pass-1 order
    bp::k_gather_u64<<<(k + 255) / 256, 256, 0, s>>>(km.p, perm.p, k, ks.p);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, need_b, ks.p, k64.p, perm.p, perm2.p, k, 0, 64, s);
    grow(need_b);
    cub::DeviceRadixSort::SortPairsDescending(tmp.p, have, ks.p, k64.p, perm.p, perm2.p, k, 0, 64, s);
    // pass 3: violated count descending
    bp::k_gather_u32<<<(k + 255) / 256, 256, 0, s>>>(kv.p, perm2.p, k, kv2.p);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, need_b, kv2.p, kv.p, perm2.p, perm.p, k, 0, 32, s);
    grow(need_b);
    cub::DeviceRadixSort::SortPairsDescending(tmp.p, have, kv2.p, kv.p, perm2.p, perm.p, k, 0, 32, s);
    bp::k_gather_i32<<<(k + 255) / 256, 256, 0, s>>>(va.p, perm.p, k, vb.p);
    BP_CUDA(cudaMemcpyAsync(order, vb.p, sizeof(int) * k, cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaStreamSynchronize(s));
  });
}

int bp_build_cache(bp_problem* p, double budget_sec, bp_cache** out)
{
  return cguard([&] {
    need(p && out, "null argument");
    bp::Problem& P = bp_problem_impl(p);
    std::vector<double> root(2 * (size_t)P.n);
    bp_problem_root(p, root.data());
    auto c = std::make_unique<bp_cache>();
    c->c.n    = P.n;
    c->c.root = root;
    c->c.entry_of.assign(P.n, -1);
    c->c.d_off.push_back(0);
    if (budget_sec > 0.0) {  // probing.hpp:248
      std::vector<int> order(P.n);
      int32_t no = 0;
      if (int rc = bp_prioritize_probe_vars(p, order.data(), &no)) throw std::runtime_error(bp_last_error());
      std::vector<int> cand;
      for (int j = 0; j < no; ++j)
        if (root[2 * order[j]] != root[2 * order[j] + 1]) cand.push_back(order[j]);
      std::lock_guard<std::mutex> lk(P.mu);
      c->c = bp::probe_vars(P, root, cand, budget_sec);
    }
    *out = c.release();
  });
}

int bp_cache_block_branches(const bp_cache* c, int32_t* n_block)
{
  return cguard([&] {
    need(c && n_block, "null argument");
    *n_block = c->c.n_block;
  });
}

int bp_cache_work(const bp_cache* c, int64_t* work5)
{
  return cguard([&] {
    need(c && work5, "null argument");
    for (int q = 0; q < 5; ++q) work5[q] = (int64_t)c->c.work[q];
  });
}

int bp_cache_destroy(bp_cache* c)
{
  delete c;
  return BP_OK;
}

int bp_cache_info(const bp_cache* c, int32_t* n_vars, int32_t* n_probed,
                  int32_t* n_infeasible_branches, int64_t* n_deltas, int32_t* n_fallback,
                  int32_t* certified, double* probe_ms)
{
  return cguard([&] {
    need(c, "null cache");
    if (n_vars) *n_vars = c->c.n;
    if (n_probed) *n_probed = c->c.n_probed;
    if (n_infeasible_branches) *n_infeasible_branches = c->c.n_infeasible_branches;
    if (n_deltas) *n_deltas = (int64_t)c->c.d_var.size();
    if (n_fallback) *n_fallback = c->c.n_fallback;
    if (certified) *certified = c->c.certified ? 1 : 0;
    if (probe_ms) *probe_ms = c->c.probe_ms;
  });
}

int bp_cache_entry(const bp_cache* c, int32_t v, int32_t* present, int32_t* hdr7, double* br4)
{
  return cguard([&] {
    need(c && present && hdr7 && br4, "null argument");
    if (v < 0 || v >= c->c.n) throw std::out_of_range("var out of range");
    const int e = c->c.entry_of[v];
    *present    = e >= 0;
    if (e < 0) return;
    hdr7[0] = c->c.e_kind[e];
    hdr7[1] = c->c.e_force[2 * e];
    hdr7[2] = c->c.e_force[2 * e + 1];
    hdr7[3] = c->c.e_feas[2 * e];
    hdr7[4] = c->c.e_feas[2 * e + 1];
    hdr7[5] = (int32_t)(c->c.d_off[2 * e + 1] - c->c.d_off[2 * e]);
    hdr7[6] = (int32_t)(c->c.d_off[2 * e + 2] - c->c.d_off[2 * e + 1]);
    for (int q = 0; q < 4; ++q) br4[q] = c->c.e_branch[4 * e + q];
  });
}

int bp_cache_deltas(const bp_cache* c, int32_t v, int32_t side, int32_t* vars, double* lo,
                    double* up)
{
  return cguard([&] {
    need(c && vars && lo && up && (side == 0 || side == 1), "bad argument");
    if (v < 0 || v >= c->c.n) throw std::out_of_range("var out of range");
    const int e = c->c.entry_of[v];
    if (e < 0) throw std::out_of_range("var has no cache entry");
    for (long long d = c->c.d_off[2 * e + side], j = 0; d < c->c.d_off[2 * e + side + 1]; ++d, ++j) {
      vars[j] = c->c.d_var[d];
      lo[j]   = c->c.d_lo[d];
      up[j]   = c->c.d_up[d];
    }
  });
}

int bp_cache_root(const bp_cache* c, double* root2n)
{
  return cguard([&] {
    need(c && root2n, "null argument");
    std::memcpy(root2n, c->c.root.data(), sizeof(double) * c->c.root.size());
  });
}

int bp_cache_create_empty(int32_t n_vars, const double* root2n, bp_cache** out)
{
  return cguard([&] {
    need(out && n_vars >= 0 && (n_vars == 0 || root2n), "bad argument");
    auto c   = std::make_unique<bp_cache>();
    c->c.n   = n_vars;
    c->c.root.assign(root2n, root2n + 2 * (size_t)n_vars);
    c->c.entry_of.assign(n_vars, -1);
    c->c.d_off.push_back(0);
    *out = c.release();
  });
}

int bp_cache_set_entry(bp_cache* c, int32_t v, const int32_t* hdr5, const double* br4,
                       int32_t n_down, const int32_t* down_vars, const double* down_lo,
                       const double* down_up, int32_t n_up, const int32_t* up_vars,
                       const double* up_lo, const double* up_up)
{
  return cguard([&] {
    need(c && hdr5 && br4 && n_down >= 0 && n_up >= 0, "bad argument");
    need((n_down == 0 || (down_vars && down_lo && down_up)) && (n_up == 0 || (up_vars && up_lo && up_up)),
         "null delta array");
    bp::HostCache& C = c->c;
    if (v < 0 || v >= C.n) throw std::out_of_range("var out of range");
    if (C.entry_of[v] >= 0) throw std::invalid_argument("var already has a cache entry");
    for (int j = 0; j < n_down; ++j)
      if (down_vars[j] < 0 || down_vars[j] >= C.n) throw std::out_of_range("delta var out of range");
    for (int j = 0; j < n_up; ++j)
      if (up_vars[j] < 0 || up_vars[j] >= C.n) throw std::out_of_range("delta var out of range");
    C.entry_of[v] = (int)C.e_var.size();
    C.e_var.push_back(v);
    C.e_kind.push_back(hdr5[0]);
    C.e_force.push_back((uint8_t)(hdr5[1] != 0));
    C.e_force.push_back((uint8_t)(hdr5[2] != 0));
    C.e_feas.push_back((uint8_t)(hdr5[3] != 0));
    C.e_feas.push_back((uint8_t)(hdr5[4] != 0));
    C.e_branch.insert(C.e_branch.end(), br4, br4 + 4);
    C.d_var.insert(C.d_var.end(), down_vars, down_vars + n_down);
    C.d_lo.insert(C.d_lo.end(), down_lo, down_lo + n_down);
    C.d_up.insert(C.d_up.end(), down_up, down_up + n_down);
    C.d_off.push_back((long long)C.d_var.size());
    C.d_var.insert(C.d_var.end(), up_vars, up_vars + n_up);
    C.d_lo.insert(C.d_lo.end(), up_lo, up_lo + n_up);
    C.d_up.insert(C.d_up.end(), up_up, up_up + n_up);
    C.d_off.push_back((long long)C.d_var.size());
    C.n_probed++;  // probing.hpp:274-278, incrementally
    C.n_infeasible_branches += (hdr5[3] ? 0 : 1) + (hdr5[4] ? 0 : 1);
  });
}

// Packed slice: [i64 n_entries, i64 n_deltas, i64 n_fallback, i64 certified]
//   entries: i32 var, i32 kind, u8 feas[2], u8 force[2], f64 branch[4], i64 count[2]
//   deltas:  i32 var[], f64 lo[], f64 up[]
int bp_cache_pack_size(const bp_cache* c, int64_t* bytes)
{
  return cguard([&] {
    need(c && bytes, "null argument");
    const int64_t ne = (int64_t)c->c.e_var.size(), nd = (int64_t)c->c.d_var.size();
    *bytes = 32 + ne * (4 + 4 + 2 + 2 + 32 + 16) + nd * (4 + 8 + 8);
  });
}

int bp_cache_pack(const bp_cache* c, void* buf, int64_t bytes)
{
  return cguard([&] {
    int64_t need_b = 0;
    bp_cache_pack_size(c, &need_b);
    need(buf && bytes >= need_b, "buffer too small");
    char* p  = static_cast<char*>(buf);
    auto put = [&](const void* src, size_t nb) {
      std::memcpy(p, src, nb);
      p += nb;
    };
    const auto& C     = c->c;
    const int64_t hdr[4] = {(int64_t)C.e_var.size(), (int64_t)C.d_var.size(), C.n_fallback,
                            C.certified ? 1 : 0};
    put(hdr, sizeof(hdr));
    for (size_t e = 0; e < C.e_var.size(); ++e) {
      put(&C.e_var[e], 4);
      put(&C.e_kind[e], 4);
      put(&C.e_feas[2 * e], 2);
      put(&C.e_force[2 * e], 2);
      put(&C.e_branch[4 * e], 32);
      const int64_t cnt[2] = {C.d_off[2 * e + 1] - C.d_off[2 * e], C.d_off[2 * e + 2] - C.d_off[2 * e + 1]};
      put(cnt, 16);
    }
    if (!C.d_var.empty()) {
      put(C.d_var.data(), 4 * C.d_var.size());
      put(C.d_lo.data(), 8 * C.d_lo.size());
      put(C.d_up.data(), 8 * C.d_up.size());
    }
  });
}

// Merges a packed slice (from any rank) into `dst`; entries of the same variable are identical
// by determinism, later slices overwrite earlier ones.
int bp_cache_merge_packed(bp_cache* dst, const void* buf, int64_t bytes)
{
  return cguard([&] {
    need(dst && buf && bytes >= 32, "bad argument");
    const char* p = static_cast<const char*>(buf);
    auto get      = [&](void* d, size_t nb) {
      std::memcpy(d, p, nb);
      p += nb;
    };
    int64_t hdr[4];
    get(hdr, sizeof(hdr));
    const int64_t ne = hdr[0], nd = hdr[1];
    // the slice arrives from another rank: validate its header against the buffer before reading
    need(ne >= 0 && nd >= 0 && ne <= (bytes - 32) / 60 && nd <= (bytes - 32) / 20 &&
             bytes >= 32 + ne * 60 + nd * 20,
         "packed cache slice: header does not match the buffer size");
    struct E {
      int var, kind;
      uint8_t feas[2], force[2];
      double br[4];
      int64_t cnt[2];
    };
    std::vector<E> es(ne);
    for (auto& e : es) {
      get(&e.var, 4);
      get(&e.kind, 4);
      get(e.feas, 2);
      get(e.force, 2);
      get(e.br, 32);
      get(e.cnt, 16);
    }
    {
      int64_t tot = 0;
      for (const auto& e : es) {
        need(e.cnt[0] >= 0 && e.cnt[1] >= 0 && e.cnt[0] <= nd && e.cnt[1] <= nd,
             "packed cache slice: negative or oversized delta count");
        tot += e.cnt[0] + e.cnt[1];
      }
      need(tot == nd, "packed cache slice: delta counts do not sum to the delta total");
    }
    std::vector<int> dv(nd);
    std::vector<double> dl(nd), du(nd);
    if (nd) {
      get(dv.data(), 4 * nd);
      get(dl.data(), 8 * nd);
      get(du.data(), 8 * nd);
    }
    // rebuild: existing entries not overwritten + the new ones, in arrival order
    bp::HostCache& C = dst->c;
    bp::HostCache M;
    M.n         = C.n;
    M.root      = C.root;
    M.certified = C.certified || hdr[3];
    M.n_fallback = C.n_fallback + (int)hdr[2];
    M.probe_ms  = C.probe_ms;
    M.entry_of.assign(C.n, -1);
    M.d_off.push_back(0);
    std::vector<uint8_t> over(C.n, 0);
    for (const auto& e : es) {
      if (e.var < 0 || e.var >= C.n) throw std::out_of_range("packed entry var out of range");
      over[e.var] = 1;
    }
    auto add = [&](int var, int kind, const uint8_t* feas, const uint8_t* force, const double* br,
                   const int* v0, const double* l0, const double* u0, int64_t c0, const int* v1,
                   const double* l1, const double* u1, int64_t c1) {
      M.entry_of[var] = (int)M.e_var.size();
      M.e_var.push_back(var);
      M.e_kind.push_back(kind);
      M.e_feas.insert(M.e_feas.end(), feas, feas + 2);
      M.e_force.insert(M.e_force.end(), force, force + 2);
      M.e_branch.insert(M.e_branch.end(), br, br + 4);
      M.d_var.insert(M.d_var.end(), v0, v0 + c0);
      M.d_lo.insert(M.d_lo.end(), l0, l0 + c0);
      M.d_up.insert(M.d_up.end(), u0, u0 + c0);
      M.d_off.push_back((long long)M.d_var.size());
      M.d_var.insert(M.d_var.end(), v1, v1 + c1);
      M.d_lo.insert(M.d_lo.end(), l1, l1 + c1);
      M.d_up.insert(M.d_up.end(), u1, u1 + c1);
      M.d_off.push_back((long long)M.d_var.size());
    };
    for (size_t e = 0; e < C.e_var.size(); ++e) {
      if (over[C.e_var[e]]) continue;
      const long long a = C.d_off[2 * e], b = C.d_off[2 * e + 1], d = C.d_off[2 * e + 2];
      add(C.e_var[e], C.e_kind[e], &C.e_feas[2 * e], &C.e_force[2 * e], &C.e_branch[4 * e],
          C.d_var.data() + a, C.d_lo.data() + a, C.d_up.data() + a, b - a, C.d_var.data() + b,
          C.d_lo.data() + b, C.d_up.data() + b, d - b);
    }
    int64_t off = 0;
    for (const auto& e : es) {
      add(e.var, e.kind, e.feas, e.force, e.br, dv.data() + off, dl.data() + off, du.data() + off,
          e.cnt[0], dv.data() + off + e.cnt[0], dl.data() + off + e.cnt[0],
          du.data() + off + e.cnt[0], e.cnt[1]);
      off += e.cnt[0] + e.cnt[1];
    }
    M.finalize_stats();
    C = std::move(M);
  });
}

int bp_assemble_bulk_warm_start(const bp_cache* c, const int32_t* vars, const double* vals,
                                int32_t n, double* bounds2n, int32_t* conflicts,
                                int32_t* n_conflicts, int32_t* evicted, int32_t* n_evicted)
{
  return cguard([&] {
    need(c && bounds2n && n_conflicts && n_evicted && (n == 0 || (vars && vals)), "null argument");
    std::vector<double> b;
    std::vector<int> cf, ev;
    bp::warm_start(c->c, vars, vals, n, b, cf, ev);
    std::memcpy(bounds2n, b.data(), sizeof(double) * b.size());
    if (conflicts) std::copy(cf.begin(), cf.end(), conflicts);
    *n_conflicts = (int32_t)(cf.size() / 2);
    if (evicted) std::copy(ev.begin(), ev.end(), evicted);
    *n_evicted = (int32_t)ev.size();
  });
}

}  // extern "C"
