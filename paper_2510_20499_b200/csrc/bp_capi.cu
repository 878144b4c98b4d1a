// extern "C" boundary (include/bp.h). Marshals plain host arrays to the device engine and maps
// C++ exceptions onto the reference's error taxonomy (std::invalid_argument / out_of_range /
// runtime_error, problem.hpp:166-180).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bp.h"
#include "bp_engine.cuh"
#include "bp_capi_internal.h"

namespace {

thread_local std::string g_last_error;

template <class F>
int guard(F&& f)
{
  try {
    f();
    g_last_error.clear();
    return BP_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return BP_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return BP_ERR_OUT_OF_RANGE;
  } catch (const bp::cuda_error& e) {
    g_last_error = e.what();
    return BP_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BP_ERR_RUNTIME;
  } catch (...) {
    g_last_error = "unknown error";
    return BP_ERR_RUNTIME;
  }
}

void need(bool ok, const char* what)
{
  if (!ok) throw std::invalid_argument(what);
}

bp::Limits to_limits(const bp_limits* l)
{
  bp_limits d;
  bp_limits_default(&d);
  if (!l) l = &d;
  bp::Limits o;
  o.max_rounds    = l->max_rounds;
  o.time_limit    = l->time_limit;
  o.abs_threshold = l->abs_threshold;
  o.rel_threshold = l->rel_threshold;
  o.incremental   = l->incremental;
  return o;
}

void decode_activities(bp::Problem& P, double* act2m, int32_t* nmin, int32_t* nmax)
{
  const int m = P.m;
  std::vector<bp::RowRec> rec(m);
  std::vector<double2> aux(m);
  if (m) {
    BP_CUDA(cudaMemcpy(rec.data(), P.st.rec, sizeof(bp::RowRec) * m, cudaMemcpyDeviceToHost));
    BP_CUDA(cudaMemcpy(aux.data(), P.st.aux, sizeof(double2) * m, cudaMemcpyDeviceToHost));
  }
  auto boxed = [](double x, int& c) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    if ((u & bp::kBoxMask) == bp::kBoxBase) {
      c = (int)(uint32_t)(u & 0xFFFFFFFFull);
      return true;
    }
    c = 0;
    return false;
  };
  for (int k = 0; k < m; ++k) {
    int c0, c1;
    const bool b0 = boxed(rec[k].min, c0), b1 = boxed(rec[k].max, c1);
    act2m[2 * k]     = b0 ? aux[k].x : rec[k].min;
    act2m[2 * k + 1] = b1 ? aux[k].y : rec[k].max;
    nmin[k]          = c0;
    nmax[k]          = c1;
  }
}

void encode_activities(bp::Problem& P, const double* act2m, const int32_t* nmin,
                       const int32_t* nmax, const double* cons_lower, const double* cons_upper)
{
  const int m = P.m;
  std::vector<bp::RowRec> rec(m);
  std::vector<double2> aux(m);
  for (int k = 0; k < m; ++k) {
    rec[k].min = nmin[k] ? bp::box_count(nmin[k]) : act2m[2 * k];
    rec[k].max = nmax[k] ? bp::box_count(nmax[k]) : act2m[2 * k + 1];
    rec[k].g   = cons_upper[k];
    rec[k].h   = cons_lower[k];
    aux[k]     = make_double2(act2m[2 * k], act2m[2 * k + 1]);
  }
  if (m) {
    BP_CUDA(cudaMemcpy(P.st.rec, rec.data(), sizeof(bp::RowRec) * m, cudaMemcpyHostToDevice));
    BP_CUDA(cudaMemcpy(P.st.aux, aux.data(), sizeof(double2) * m, cudaMemcpyHostToDevice));
  }
}

void upload_bounds(bp::Problem& P, const double* b2n, cudaStream_t s)
{
  if (P.n)
    BP_CUDA(cudaMemcpyAsync(P.st.bounds, b2n, sizeof(double) * 2 * P.n, cudaMemcpyHostToDevice, s));
}
void download_bounds(bp::Problem& P, double* b2n, cudaStream_t s)
{
  if (P.n)
    BP_CUDA(cudaMemcpyAsync(b2n, P.st.bounds, sizeof(double) * 2 * P.n, cudaMemcpyDeviceToHost, s));
  BP_CUDA(cudaStreamSynchronize(s));
}
void reset_ctl(bp::Problem& P, cudaStream_t s)
{
  BP_CUDA(cudaMemsetAsync(P.st.ctl, 0, sizeof(bp::Ctl), s));
}

}  // namespace

struct bp_problem {
  bp::Problem impl;
  std::vector<double> cons_lower, cons_upper;
  bp_problem_host host;
};

bp::Problem& bp_problem_impl(bp_problem* p) { return p->impl; }
const bp_problem_host& bp_problem_hostdata(bp_problem* p) { return p->host; }
void bp_problem_root(bp_problem* p, double* root2n)
{
  for (int i = 0; i < p->impl.n; ++i) {
    root2n[2 * i]     = p->host.var_lower[i];
    root2n[2 * i + 1] = p->host.var_upper[i];
  }
}
void bp_set_last_error(const char* msg) { g_last_error = msg; }

extern "C" {

const char* bp_last_error(void) { return g_last_error.c_str(); }

void bp_limits_default(bp_limits* lim)
{
  lim->max_rounds    = 64;
  lim->time_limit    = INFINITY;
  lim->abs_threshold = 1e-7;
  lim->rel_threshold = 1e-4;
  lim->incremental   = 1;
}

int64_t bp_kernel_launches(void) { return bp::g_kernel_launches; }

int bp_kernel_time(const bp_problem* p, double* last_ms, double* total_ms, int64_t* launches)
{
  return guard([&] {
    need(p, "null problem");
    if (last_ms) *last_ms = p->impl.last_kernel_ms;
    if (total_ms) *total_ms = p->impl.total_kernel_ms;
    if (launches) *launches = p->impl.n_launch;
  });
}

int bp_device_count(int32_t* count)
{
  return guard([&] {
    int c = 0;
    BP_CUDA(cudaGetDeviceCount(&c));
    *count = c;
  });
}

int bp_problem_create(const bp_problem_desc* d, int32_t device, bp_problem** out)
{
  return guard([&] {
    need(d && out, "null argument");
    need(d->n_vars >= 0 && d->n_cons >= 0, "negative dimension");
    need(d->row_start && (d->n_cons == 0 || d->row_start[0] == 0), "row_start must start at 0");
    const long long N = d->row_start[d->n_cons];
    need(N == 0 || (d->row_col && d->row_val), "missing CSR arrays");
    need(d->var_lower && d->var_upper && d->is_integer, "missing variable arrays");
    need(d->n_cons == 0 || (d->cons_lower && d->cons_upper), "missing constraint arrays");
    for (int k = 0; k < d->n_cons; ++k) {
      if (d->row_start[k + 1] < d->row_start[k]) throw std::invalid_argument("row_start not monotone");
      if (d->cons_lower[k] > d->cons_upper[k])
        throw std::runtime_error("constraint " + std::to_string(k) + " has crossed bounds");
    }
    for (long long e = 0; e < N; ++e)
      if (d->row_col[e] < 0 || d->row_col[e] >= d->n_vars)
        throw std::out_of_range("entry col out of range");
    for (int i = 0; i < d->n_vars; ++i)
      if (d->var_lower[i] > d->var_upper[i])
        throw std::runtime_error("variable " + std::to_string(i) +
                                 " has empty domain after bound tightening");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw bp::cuda_error("no CUDA device available (the engine has no CPU fallback)");
    need(device >= 0 && device < ndev, "device index out of range");
    auto p             = std::make_unique<bp_problem>();
    p->impl.device     = device;
    p->cons_lower.assign(d->cons_lower, d->cons_lower + d->n_cons);
    p->cons_upper.assign(d->cons_upper, d->cons_upper + d->n_cons);
    bp::problem_build(p->impl, d->n_vars, d->n_cons, d->row_start, d->row_col, d->row_val,
                      d->col_start, d->col_row, d->col_val, d->var_lower, d->var_upper,
                      d->is_integer, d->cons_lower, d->cons_upper);
    bp_problem_host& H = p->host;
    H.var_lower.assign(d->var_lower, d->var_lower + d->n_vars);
    H.var_upper.assign(d->var_upper, d->var_upper + d->n_vars);
    H.is_integer.assign(d->is_integer, d->is_integer + d->n_vars);
    H.cons_lower = p->cons_lower;
    H.cons_upper = p->cons_upper;
    H.row_col.assign(d->row_col, d->row_col + N);
    H.row_val.assign(d->row_val, d->row_val + N);
    // CSC on the host (the stable transpose, problem.hpp:211-225)
    {
      const int n = d->n_vars, m = d->n_cons;
      const std::vector<int>& cs = p->impl.h_col_start;
      H.col_row.resize(N);
      H.col_val.resize(N);
      std::vector<int> cur(cs.begin(), cs.end() - 1);
      for (int k = 0; k < m; ++k)
        for (int e = d->row_start[k]; e < d->row_start[k + 1]; ++e) {
          const int dst  = cur[d->row_col[e]]++;
          H.col_row[dst] = k;
          H.col_val[dst] = d->row_val[e];
        }
      (void)n;
    }
    *out = p.release();
  });
}

int bp_problem_destroy(bp_problem* p)
{
  return guard([&] {
    if (!p) return;
    cudaSetDevice(p->impl.device);
    if (p->impl.stream) cudaStreamDestroy(p->impl.stream);
    if (p->impl.ev0) cudaEventDestroy(p->impl.ev0);
    if (p->impl.ev1) cudaEventDestroy(p->impl.ev1);
    delete p;
  });
}

int bp_problem_info(const bp_problem* p, int32_t* n_vars, int32_t* n_cons, int64_t* nnz)
{
  return guard([&] {
    need(p, "null problem");
    if (n_vars) *n_vars = p->impl.n;
    if (n_cons) *n_cons = p->impl.m;
    if (nnz) *nnz = p->impl.nnz;
  });
}

int bp_compute_activities(bp_problem* p, const double* bounds2n, const int32_t* rows,
                          int32_t nrows, double* act2m, int32_t* ninf_min, int32_t* ninf_max)
{
  return guard([&] {
    need(p && bounds2n && act2m && ninf_min && ninf_max, "null argument");
    bp::Problem& P = p->impl;
    std::lock_guard<std::mutex> lk(P.mu);
    BP_CUDA(cudaSetDevice(P.device));
    cudaStream_t s = P.stream;
    const bool full = rows == nullptr || nrows < 0;
    if (!full)
      for (int j = 0; j < nrows; ++j)
        if (rows[j] < 0 || rows[j] >= P.m) throw std::out_of_range("row index out of range");
    // rows outside a subset keep the caller's values (propagation.hpp:230)
    encode_activities(P, act2m, ninf_min, ninf_max, p->cons_lower.data(), p->cons_upper.data());
    upload_bounds(P, bounds2n, s);
    reset_ctl(P, s);
    if (!full) bp::stage_rows(P, rows, nrows, s);
    bp::Limits lim = to_limits(nullptr);
    bp::run_engine(P, bp::MODE_ACTIVITY, full, lim, s);
    decode_activities(P, act2m, ninf_min, ninf_max);
  });
}

int bp_tighten_bounds(bp_problem* p, double* bounds2n, int32_t* infeasible, const double* act2m,
                      const int32_t* ninf_min, const int32_t* ninf_max, const int32_t* vars,
                      int32_t nvars, const bp_limits* lim, int32_t* changed, int32_t* n_changed,
                      int32_t* crossed)
{
  return guard([&] {
    need(p && bounds2n && infeasible && act2m && ninf_min && ninf_max && changed && n_changed,
         "null argument");
    bp::Problem& P = p->impl;
    std::lock_guard<std::mutex> lk(P.mu);
    BP_CUDA(cudaSetDevice(P.device));
    cudaStream_t s  = P.stream;
    const bool full = vars == nullptr || nvars < 0;
    if (!full)
      for (int j = 0; j < nvars; ++j)
        if (vars[j] < 0 || vars[j] >= P.n) throw std::out_of_range("var index out of range");
    encode_activities(P, act2m, ninf_min, ninf_max, p->cons_lower.data(), p->cons_upper.data());
    upload_bounds(P, bounds2n, s);
    reset_ctl(P, s);
    if (!full) {
      // the reference's result[] array is indexed by var: duplicates evaluate the same inputs
      std::vector<int> uniq(vars, vars + nvars);
      std::sort(uniq.begin(), uniq.end());
      uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
      bp::stage_vars(P, uniq.data(), (int)uniq.size(), s);
    }
    bp::run_engine(P, bp::MODE_TIGHTEN, full, to_limits(lim), s);
    bp::ParCtl pc;
    BP_CUDA(cudaMemcpy(&pc, &P.st.ctl->par[1], sizeof(pc), cudaMemcpyDeviceToHost));
    std::vector<int> ch(pc.n_changed);
    if (pc.n_changed)
      BP_CUDA(cudaMemcpy(ch.data(), P.st.changed, sizeof(int) * pc.n_changed, cudaMemcpyDeviceToHost));
    std::sort(ch.begin(), ch.end());
    std::copy(ch.begin(), ch.end(), changed);
    *n_changed = (int32_t)ch.size();
    if (crossed) *crossed = pc.n_crossed;
    download_bounds(P, bounds2n, s);
    if (pc.n_crossed > 0) *infeasible = 1;
  });
}

int bp_propagate_device(bp_problem* p, double* d_bounds2n, int32_t* infeasible,
                        const bp_limits* lim, bp_result* res, void* stream)
{
  return bp_propagate_ex(p, d_bounds2n, infeasible, lim, res, stream, 0, nullptr);
}

int bp_propagate_ex(bp_problem* p, double* d_bounds2n, int32_t* infeasible, const bp_limits* lim,
                    bp_result* res, void* stream, int32_t flags, int64_t* d_stats)
{
  return guard([&] {
    need(p && d_bounds2n && infeasible && res, "null argument");
    bp::Problem& P = p->impl;
    std::lock_guard<std::mutex> lk(P.mu);
    BP_CUDA(cudaSetDevice(P.device));
    const bp::Limits l = to_limits(lim);
    res->status        = BP_UNCHANGED;
    res->rounds        = 0;
    res->crossed_vars  = 0;
    if (*infeasible) {  // propagation.hpp:423-426
      res->status = BP_INFEASIBLE;
      return;
    }
    if (l.max_rounds <= 0 || l.time_limit <= 0.0) return;  // loop never entered
    cudaStream_t s = stream ? (cudaStream_t)stream : P.stream;
    if (P.n)
      BP_CUDA(cudaMemcpyAsync(P.st.bounds, d_bounds2n, sizeof(double) * 2 * P.n,
                              cudaMemcpyDeviceToDevice, s));
    reset_ctl(P, s);
    const bp::RunResult r = bp::run_engine(P, bp::MODE_PROPAGATE, true, l, s,
                                           (flags & BP_FORCE_FRONTIER) ? bp::ENGINE_FORCE_FRONTIER : 0,
                                           reinterpret_cast<long long*>(d_stats));
    if (P.n)
      BP_CUDA(cudaMemcpyAsync(d_bounds2n, P.st.bounds, sizeof(double) * 2 * P.n,
                              cudaMemcpyDeviceToDevice, s));
    BP_CUDA(cudaStreamSynchronize(s));
    res->status       = r.status;
    res->rounds       = r.rounds;
    res->crossed_vars = r.crossed;
    if (r.status == BP_INFEASIBLE) *infeasible = 1;
  });
}

int bp_propagate(bp_problem* p, double* bounds2n, int32_t* infeasible, const bp_limits* lim,
                 bp_result* res)
{
  return guard([&] {
    need(p && bounds2n && infeasible && res, "null argument");
    bp::Problem& P = p->impl;
    std::lock_guard<std::mutex> lk(P.mu);
    BP_CUDA(cudaSetDevice(P.device));
    const bp::Limits l = to_limits(lim);
    res->status        = BP_UNCHANGED;
    res->rounds        = 0;
    res->crossed_vars  = 0;
    if (*infeasible) {
      res->status = BP_INFEASIBLE;
      return;
    }
    if (l.max_rounds <= 0 || l.time_limit <= 0.0) return;
    cudaStream_t s = P.stream;
    upload_bounds(P, bounds2n, s);
    reset_ctl(P, s);
    const bp::RunResult r = bp::run_engine(P, bp::MODE_PROPAGATE, true, l, s);
    download_bounds(P, bounds2n, s);
    res->status       = r.status;
    res->rounds       = r.rounds;
    res->crossed_vars = r.crossed;
    if (r.status == BP_INFEASIBLE) *infeasible = 1;
  });
}

}  // extern "C"
