// Multi-GPU probing-cache construction from one process (SURVEY §8b `bp_build_cache_multi`, §8e).
//
// Reference: build_cache (probing.hpp:243-281), whose `min(n, threads)` workers pull candidates
// from an atomic cursor (:256-272). Here the workers are GPUs: the priority-ordered candidates are
// interleaved over the devices (device d takes positions d, d + G, ...), every device probes its
// share with the batched kernels against its own replica of the problem, packs its cache slice
// (bp_cache_pack layout) into device memory, and the slices travel to device 0 with NCCL
// point-to-point sends inside one group (ncclSend on each peer, ncclRecv on rank 0 — a gather, not
// an all-gather: only rank 0 needs them). Rank 0 merges them by variable. Entries are
// deterministic per variable, so any partition yields the same cache as one GPU (tested).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 — the one torch already loaded, or the
// system's), so the library has no link-time NCCL dependency; one device needs no NCCL at all.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "bp_capi_internal.h"
#include "bp_engine.cuh"
#include "bp_probe.cuh"

namespace bp {
HostCache probe_vars(Problem& P, const std::vector<double>& root, const std::vector<int>& vars,
                     double budget_sec);
}

namespace {

struct Nccl {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t)                   = nullptr;
  ncclResult_t (*GroupStart)()                              = nullptr;
  ncclResult_t (*GroupEnd)()                                = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t)       = nullptr;
  const char* (*GetErrorString)(ncclResult_t)                                              = nullptr;

  static const Nccl& get()
  {
    static Nccl n = [] {
      Nccl x;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!h) throw std::runtime_error("bp_build_cache_multi: libnccl.so.2 not found");
      auto sym = [&](const char* s) {
        void* f = dlsym(h, s);
        if (!f) throw std::runtime_error(std::string("bp_build_cache_multi: NCCL symbol missing: ") + s);
        return f;
      };
      x.CommInitAll    = reinterpret_cast<decltype(x.CommInitAll)>(sym("ncclCommInitAll"));
      x.CommDestroy    = reinterpret_cast<decltype(x.CommDestroy)>(sym("ncclCommDestroy"));
      x.GroupStart     = reinterpret_cast<decltype(x.GroupStart)>(sym("ncclGroupStart"));
      x.GroupEnd       = reinterpret_cast<decltype(x.GroupEnd)>(sym("ncclGroupEnd"));
      x.Send           = reinterpret_cast<decltype(x.Send)>(sym("ncclSend"));
      x.Recv           = reinterpret_cast<decltype(x.Recv)>(sym("ncclRecv"));
      x.GetErrorString = reinterpret_cast<decltype(x.GetErrorString)>(sym("ncclGetErrorString"));
      return x;
    }();
    return n;
  }
};

void nccl_check(ncclResult_t r, const char* what)
{
  if (r != ncclSuccess)
    throw bp::cuda_error(std::string(what) + ": " + Nccl::get().GetErrorString(r));
}

struct DevBytes {
  int device = 0;
  void* p    = nullptr;
  ~DevBytes()
  {
    if (p) {
      cudaSetDevice(device);
      cudaFree(p);
    }
  }
};

template <class F>
int mguard(F&& f)
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

int bp_build_cache_multi(bp_problem* const* probs, int32_t nprob, double budget_sec,
                         const int32_t* vars, int32_t nvars, bp_cache** out,
                         double* probe_ms_per_device)
{
  return mguard([&] {
    need(probs && nprob >= 1 && out && (nvars <= 0 || vars), "null argument");
    std::vector<bp::Problem*> Ps(nprob);
    std::vector<int> devs(nprob);
    for (int d = 0; d < nprob; ++d) {
      need(probs[d] != nullptr, "null problem handle");
      Ps[d]   = &bp_problem_impl(probs[d]);
      devs[d] = Ps[d]->device;
      need(Ps[d]->n == Ps[0]->n && Ps[d]->m == Ps[0]->m && Ps[d]->nnz == Ps[0]->nnz,
           "problem replicas differ in shape");
      for (int e = 0; e < d; ++e) need(devs[e] != devs[d], "two replicas on one device");
    }
    const int n = Ps[0]->n;
    std::vector<double> root(2 * (size_t)n);
    bp_problem_root(probs[0], root.data());
    // candidates: the caller's list, or build_cache's (priority order minus root-fixed vars)
    std::vector<int> cand;
    const bool explicit_vars = nvars >= 0 && vars;
    if (explicit_vars) {
      cand.assign(vars, vars + nvars);
    } else if (budget_sec > 0.0) {
      std::vector<int> order(std::max(n, 1));
      int32_t no = 0;
      if (bp_prioritize_probe_vars(probs[0], order.data(), &no) != BP_OK)
        throw std::runtime_error(bp_last_error());
      for (int j = 0; j < no; ++j)
        if (root[2 * order[j]] != root[2 * order[j] + 1]) cand.push_back(order[j]);
    }
    // one host thread per device: probe the strided share, pack it into device memory
    std::vector<std::vector<char>> packed(nprob);
    std::vector<DevBytes> dbuf(nprob);
    std::vector<double> probe_ms(nprob, 0.0);
    std::vector<std::string> err(nprob);
    std::vector<std::thread> th;
    for (int d = 0; d < nprob; ++d)
      th.emplace_back([&, d] {
        try {
          std::vector<int> mine;
          for (size_t j = d; j < cand.size(); j += nprob) mine.push_back(cand[j]);
          bp::Problem& P = *Ps[d];
          std::lock_guard<std::mutex> lk(P.mu);
          std::unique_ptr<bp_cache, int (*)(bp_cache*)> c(
              bp_cache_adopt(bp::probe_vars(P, root, mine, explicit_vars ? INFINITY : budget_sec)),
              bp_cache_destroy);
          probe_ms[d]  = bp_cache_host(c.get())->probe_ms;
          int64_t bytes = 0;
          if (bp_cache_pack_size(c.get(), &bytes) != BP_OK) throw std::runtime_error(bp_last_error());
          packed[d].resize((size_t)bytes);
          if (bp_cache_pack(c.get(), packed[d].data(), bytes) != BP_OK) throw std::runtime_error(bp_last_error());
          BP_CUDA(cudaSetDevice(devs[d]));
          dbuf[d].device = devs[d];
          BP_CUDA(cudaMalloc(&dbuf[d].p, std::max<size_t>(packed[d].size(), 1)));
          BP_CUDA(cudaMemcpy(dbuf[d].p, packed[d].data(), packed[d].size(), cudaMemcpyHostToDevice));
        } catch (const std::exception& e) {
          err[d] = e.what();
        }
      });
    for (auto& t : th) t.join();
    for (int d = 0; d < nprob; ++d)
      if (!err[d].empty()) throw std::runtime_error("device " + std::to_string(devs[d]) + ": " + err[d]);
    if (probe_ms_per_device)
      for (int d = 0; d < nprob; ++d) probe_ms_per_device[d] = probe_ms[d];
    // gather the slices to rank 0 (device devs[0]) over NCCL
    std::vector<DevBytes> rbuf(nprob);
    if (nprob > 1) {
      const Nccl& N = Nccl::get();
      std::vector<ncclComm_t> comms(nprob);
      nccl_check(N.CommInitAll(comms.data(), nprob, devs.data()), "ncclCommInitAll");
      std::vector<cudaStream_t> st(nprob);
      for (int d = 0; d < nprob; ++d) {
        BP_CUDA(cudaSetDevice(devs[d]));
        BP_CUDA(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
        if (d > 0) {
          BP_CUDA(cudaSetDevice(devs[0]));
          rbuf[d].device = devs[0];
          BP_CUDA(cudaMalloc(&rbuf[d].p, std::max<size_t>(packed[d].size(), 1)));
        }
      }
      nccl_check(N.GroupStart(), "ncclGroupStart");
      for (int d = 1; d < nprob; ++d) {
        if (packed[d].empty()) continue;
        nccl_check(N.Send(dbuf[d].p, packed[d].size(), ncclUint8, 0, comms[d], st[d]), "ncclSend");
        nccl_check(N.Recv(rbuf[d].p, packed[d].size(), ncclUint8, d, comms[0], st[0]), "ncclRecv");
      }
      nccl_check(N.GroupEnd(), "ncclGroupEnd");
      for (int d = 0; d < nprob; ++d) {
        BP_CUDA(cudaSetDevice(devs[d]));
        BP_CUDA(cudaStreamSynchronize(st[d]));
      }
      BP_CUDA(cudaSetDevice(devs[0]));
      for (int d = 1; d < nprob; ++d)  // rank 0 reads the gathered slices
        if (!packed[d].empty())
          BP_CUDA(cudaMemcpy(packed[d].data(), rbuf[d].p, packed[d].size(), cudaMemcpyDeviceToHost));
      for (int d = 0; d < nprob; ++d) {
        cudaSetDevice(devs[d]);
        cudaStreamDestroy(st[d]);
        N.CommDestroy(comms[d]);
      }
    }
    // rank-0 merge by variable
    bp_cache* merged = nullptr;
    if (bp_cache_create_empty(n, root.data(), &merged) != BP_OK) throw std::runtime_error(bp_last_error());
    std::unique_ptr<bp_cache, int (*)(bp_cache*)> guard(merged, bp_cache_destroy);
    for (int d = 0; d < nprob; ++d)
      if (bp_cache_merge_packed(merged, packed[d].data(), (int64_t)packed[d].size()) != BP_OK)
        throw std::runtime_error(bp_last_error());
    *out = guard.release();
  });
}

}  // extern "C"
