// pulse_gpu.hpp — C++ drop-in for the reference's bound-propagation hot path on the B200 engine.
//
// A maintainer of the reference (`proj/include/pulse`, header-only C++20) adds this header and
// links libbp.so; every function below has the signature, argument meaning, result type and
// exception behaviour of the `pulse::` function it replaces, and computes on the GPU through the
// C-ABI in bp.h (plain pointers; no CUDA or torch types cross it):
//
//   pulse::ProblemBuilder::build       problem.hpp:141       -> bp_build_problem
//   pulse::lpdetail::spmv_rows / cols  lp.hpp:74, :89        -> bp_lp_spmv_rows / bp_lp_spmv_cols
//   (PDHG inner iteration, lp.hpp:315-340)                   -> bp_lp_pdhg_iterate
//   pulse::compute_activities          propagation.hpp:226   -> bp_compute_activities
//   pulse::tighten_bounds              propagation.hpp:378   -> bp_tighten_bounds
//   pulse::propagate                   propagation.hpp:418   -> bp_propagate
//   pulse::prioritize_probe_vars       probing.hpp:105       -> bp_prioritize_probe_vars
//   pulse::probe_variable              probing.hpp:225       -> bp_probe_variables
//   pulse::build_cache                 probing.hpp:243       -> bp_build_cache
//   pulse::assemble_bulk_warm_start    probing.hpp:292       -> bp_assemble_bulk_warm_start
//   pulse::parallel_propagate          rounding.hpp:213      -> bp_parallel_propagate
//   pulse::repair                      rounding.hpp:234      -> bp_repair
//   pulse::propagation_round           rounding.hpp:393      -> bp_propagation_round_rng
//                                                               (+ the reference's own lp_polish)
//
// Usage: `namespace pg = pulse::gpu;` and call pg::propagate(p, b) where pulse::propagate(p, b)
// was called (INTEGRATION.md shows the switch for fp.hpp). Results are bit-identical to the
// reference's (tests/cpp/test_dropin.cpp runs both side by side).
//
// Device problems: one bp_problem per (ProblemDef, device), uploaded on first use and kept in a side
// table keyed by the ProblemDef's address and validated by its array addresses, sizes and an O(1)
// content sample (16 words per array): fp.hpp:253 rebuilds problems, often at the same addresses,
// and a stale entry is re-uploaded. An in-place edit of a problem's arrays must be announced with
// pulse::gpu::invalidate(p). Call pulse::gpu::release(p) before destroying a ProblemDef to free its
// device copies early.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bp.h"
#include "pulse/probing.hpp"
#include "pulse/propagation.hpp"
#include "pulse/lp.hpp"
#include "pulse/rounding.hpp"

namespace pulse::gpu {

namespace detail {

// bp.h error codes -> the exception types the reference throws (problem.hpp:166-180).
inline void check(int rc)
{
  if (rc == BP_OK) return;
  const std::string msg = std::string("bp: ") + bp_last_error();
  switch (rc) {
    case BP_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case BP_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

// Cheap content sample of an array: its size and up to 16 evenly spaced 8-byte words (O(1) per
// call -- the per-call cost of the side table must stay far below a propagate). Together with the
// array addresses and sizes it detects a rebuilt ProblemDef (fp.hpp:253) even at a reused
// address; an IN-PLACE edit of a problem array must be announced with pulse::gpu::invalidate(p).
template <class T>
inline uint64_t sample(uint64_t h, const std::vector<T>& v)
{
  const size_t bytes = v.size() * sizeof(T), words = bytes / 8;
  const unsigned char* c = reinterpret_cast<const unsigned char*>(v.data());
  auto mix = [&](uint64_t w) { h = (h ^ w) * 0x100000001b3ull; h ^= h >> 29; };
  mix(bytes);
  for (size_t j = 0; words && j < 16; ++j) {
    uint64_t w;
    std::memcpy(&w, c + 8 * (j * (words - 1) / 15), 8);
    mix(w);
  }
  return h;
}

struct Key {
  const ProblemDef* p;
  int device;
  const void* arrays[8];
  size_t sizes[3];
  uint64_t content;
  bool operator==(const Key& o) const
  {
    return p == o.p && device == o.device && std::memcmp(arrays, o.arrays, sizeof(arrays)) == 0 &&
           std::memcmp(sizes, o.sizes, sizeof(sizes)) == 0 && content == o.content;
  }
};

inline Key key_of(const ProblemDef& p, int device)
{
  Key k{&p,
        device,
        {p.row_start.data(), p.row_col.data(), p.row_val.data(), p.var_lower.data(),
         p.var_upper.data(), p.is_integer.data(), p.cons_lower.data(), p.cons_upper.data()},
        {(size_t)p.n_vars, (size_t)p.n_cons, p.row_col.size()},
        1469598103934665603ull};
  uint64_t& h = k.content;
  h = sample(h, p.var_lower);
  h = sample(h, p.var_upper);
  h = sample(h, p.cons_lower);
  h = sample(h, p.cons_upper);
  h = sample(h, p.is_integer);
  h = sample(h, p.row_start);
  h = sample(h, p.row_col);
  h = sample(h, p.row_val);
  return k;
}

struct ProblemHandle {
  Key key;
  bp_problem* h = nullptr;
  ~ProblemHandle()
  {
    if (h) bp_problem_destroy(h);
  }
};

struct Registry {
  std::mutex mu;
  std::vector<std::unique_ptr<ProblemHandle>> items;
  int device = 0;
};

inline Registry& registry()
{
  static Registry r;
  return r;
}

// The device copy of p on `device` (default: set_device's), uploaded on first use and re-uploaded
// when p changed (key mismatch) or after invalidate(p).
inline bp_problem* handle(const ProblemDef& p, int device = -1)
{
  Registry& R = registry();
  if (device < 0) device = R.device;
  const Key k = key_of(p, device);
  std::lock_guard<std::mutex> lk(R.mu);
  for (auto it = R.items.begin(); it != R.items.end(); ++it) {
    if ((*it)->key.p != &p || (*it)->key.device != device) continue;
    if ((*it)->key == k) return (*it)->h;
    R.items.erase(it);  // stale: the ProblemDef at this address changed
    break;
  }
  bp_problem_desc d{};
  d.n_vars     = p.n_vars;
  d.n_cons     = p.n_cons;
  d.row_start  = p.row_start.data();
  d.row_col    = p.row_col.data();
  d.row_val    = p.row_val.data();
  d.col_start  = p.col_start.empty() ? nullptr : p.col_start.data();
  d.col_row    = p.col_start.empty() ? nullptr : p.col_row.data();
  d.col_val    = p.col_start.empty() ? nullptr : p.col_val.data();
  d.var_lower  = p.var_lower.data();
  d.var_upper  = p.var_upper.data();
  d.is_integer = p.is_integer.data();
  d.cons_lower = p.cons_lower.data();
  d.cons_upper = p.cons_upper.data();
  auto ph      = std::make_unique<ProblemHandle>();
  ph->key      = k;
  check(bp_problem_create(&d, device, &ph->h));
  R.items.push_back(std::move(ph));
  return R.items.back()->h;
}

inline bp_limits limits(const PropagationLimits& l)
{
  bp_limits o;
  o.max_rounds    = l.max_rounds;
  o.time_limit    = l.time_limit;
  o.abs_threshold = l.abs_threshold;
  o.rel_threshold = l.rel_threshold;
  o.incremental   = l.incremental ? 1 : 0;
  return o;
}

inline void store(BoundsState& b, const std::vector<double>& raw)
{
  for (int i = 0; i < b.n_vars(); ++i) {
    b.set_lower(i, raw[2 * i]);
    b.set_upper(i, raw[2 * i + 1]);
  }
}

inline BoundsState from_raw(const ProblemDef& p, const double* raw, bool infeasible)
{
  BoundsState b(p);
  for (int i = 0; i < p.n_vars; ++i) {
    b.set_lower(i, raw[2 * i]);
    b.set_upper(i, raw[2 * i + 1]);
  }
  if (infeasible) b.mark_infeasible();
  return b;
}

struct CacheDeleter {
  void operator()(bp_cache* c) const
  {
    if (c) bp_cache_destroy(c);
  }
};
using CachePtr = std::unique_ptr<bp_cache, CacheDeleter>;

// Materialises a device-built cache as the reference's pulse::ProbingCache (probing.hpp:87-98).
inline ProbingCache to_pulse(const ProblemDef& p, const bp_cache* c)
{
  ProbingCache out;
  int32_t nv = 0, np = 0, ninf = 0, nfb = 0, cert = 0;
  int64_t nd = 0;
  double ms  = 0.0;
  check(bp_cache_info(c, &nv, &np, &ninf, &nd, &nfb, &cert, &ms));
  std::vector<double> root(2 * (size_t)nv);
  check(bp_cache_root(c, root.data()));
  out.root = from_raw(p, root.data(), false);
  out.entries.resize(nv);
  std::vector<int32_t> dv;
  std::vector<double> dl, du;
  for (int v = 0; v < nv; ++v) {
    int32_t present = 0, hdr[7];
    double br[4];
    check(bp_cache_entry(c, v, &present, hdr, br));
    if (!present) continue;
    ProbeEntry e;
    e.var              = v;
    e.kind             = static_cast<BranchKind>(hdr[0]);
    e.forces_down      = hdr[1] != 0;
    e.forces_up        = hdr[2] != 0;
    e.down.feasible    = hdr[3] != 0;
    e.up.feasible      = hdr[4] != 0;
    e.down.branch_lower = br[0];
    e.down.branch_upper = br[1];
    e.up.branch_lower   = br[2];
    e.up.branch_upper   = br[3];
    for (int side = 0; side < 2; ++side) {
      const int cnt = hdr[5 + side];
      if (cnt == 0) continue;
      dv.resize(cnt);
      dl.resize(cnt);
      du.resize(cnt);
      check(bp_cache_deltas(c, v, side, dv.data(), dl.data(), du.data()));
      auto& d = side ? e.up.deltas : e.down.deltas;
      d.reserve(cnt);
      for (int j = 0; j < cnt; ++j) d.push_back({dv[j], dl[j], du[j]});
    }
    out.entries[v] = std::move(e);
  }
  out.n_probed              = np;
  out.n_infeasible_branches = ninf;
  return out;
}

// Hands a pulse::ProbingCache (e.g. one built on the CPU) to the engine.
inline CachePtr from_pulse(const ProbingCache& cache)
{
  bp_cache* c = nullptr;
  check(bp_cache_create_empty(cache.root.n_vars(), cache.root.raw().data(), &c));
  CachePtr out(c);
  std::vector<int32_t> v0, v1;
  std::vector<double> l0, u0, l1, u1;
  for (const auto& oe : cache.entries) {
    if (!oe) continue;
    const ProbeEntry& e = *oe;
    const int32_t hdr[5] = {static_cast<int32_t>(e.kind), e.forces_down, e.forces_up,
                            e.down.feasible, e.up.feasible};
    const double br[4] = {e.down.branch_lower, e.down.branch_upper, e.up.branch_lower,
                          e.up.branch_upper};
    v0.clear(); l0.clear(); u0.clear(); v1.clear(); l1.clear(); u1.clear();
    for (const auto& d : e.down.deltas) { v0.push_back(d.var); l0.push_back(d.new_lower); u0.push_back(d.new_upper); }
    for (const auto& d : e.up.deltas) { v1.push_back(d.var); l1.push_back(d.new_lower); u1.push_back(d.new_upper); }
    check(bp_cache_set_entry(c, e.var, hdr, br, (int32_t)v0.size(), v0.data(), l0.data(), u0.data(),
                             (int32_t)v1.size(), v1.data(), l1.data(), u1.data()));
  }
  return out;
}

}  // namespace detail

// Frees the device copy of p (optional: copies are also freed at exit).
inline void release(const ProblemDef& p)
{
  auto& R = detail::registry();
  std::lock_guard<std::mutex> lk(R.mu);
  for (auto it = R.items.begin(); it != R.items.end();)
    it = (*it)->key.p == &p ? R.items.erase(it) : it + 1;
}

// Announces an in-place edit of p's arrays: its device copies are dropped and re-uploaded on the
// next call (the side table samples array contents only sparsely).
inline void invalidate(const ProblemDef& p) { release(p); }

// Device used for problems uploaded from now on (default 0).
inline void set_device(int device) { detail::registry().device = device; }

// ---------------------------------------------------------------- propagation.hpp

// propagation.hpp:226. The plan only schedules the reference's CPU sweep; the engine partitions
// work itself (results are plan-independent, test_propagation.cpp:244-262).
inline void compute_activities(const ProblemDef& p, const BoundsState& b,
                               const std::vector<int>* rows, ActivityState& a,
                               const WorkPlan* /*plan*/ = nullptr)
{
  if (static_cast<int>(a.n_inf_min.size()) != p.n_cons) a.resize(p.n_cons);
  detail::check(bp_compute_activities(detail::handle(p), b.raw().data(), rows ? rows->data() : nullptr,
                                      rows ? (int32_t)rows->size() : -1, a.act.data(),
                                      a.n_inf_min.data(), a.n_inf_max.data()));
}

// propagation.hpp:378
inline std::vector<int> tighten_bounds(const ProblemDef& p, BoundsState& b, const ActivityState& a,
                                       const std::vector<int>* vars, const PropagationLimits& lim,
                                       int* crossed_out = nullptr, const WorkPlan* /*plan*/ = nullptr)
{
  double* raw = const_cast<double*>(b.raw().data());  // in place on b's storage (b is non-const)
  std::vector<int32_t> changed(p.n_vars);
  int32_t inf = 0, nch = 0, crossed = 0;
  const bp_limits l = detail::limits(lim);
  detail::check(bp_tighten_bounds(detail::handle(p), raw, &inf, a.act.data(),
                                  a.n_inf_min.data(), a.n_inf_max.data(),
                                  vars ? vars->data() : nullptr, vars ? (int32_t)vars->size() : -1, &l,
                                  changed.data(), &nch, &crossed));
  changed.resize(nch);
  if (crossed > 0) b.mark_infeasible();
  if (crossed_out) *crossed_out = crossed;
  return std::vector<int>(changed.begin(), changed.end());
}

// propagation.hpp:418
inline PropagationResult propagate(const ProblemDef& p, BoundsState& b,
                                   const PropagationLimits& lim = {},
                                   const WorkPlan* /*plan*/ = nullptr)
{
  PropagationResult r;
  if (b.infeasible()) {  // propagation.hpp:423-426
    r.status = PropagationStatus::Infeasible;
    return r;
  }
  // in place on b's own storage (raw() is the state's vector; b is non-const): no 16n-byte copies
  double* raw = const_cast<double*>(b.raw().data());
  int32_t inf = 0;
  bp_result res{};
  const bp_limits l = detail::limits(lim);
  detail::check(bp_propagate(detail::handle(p), raw, &inf, &l, &res));
  if (inf) b.mark_infeasible();
  r.status       = static_cast<PropagationStatus>(res.status);
  r.rounds       = res.rounds;
  r.crossed_vars = res.crossed_vars;
  return r;
}

// ---------------------------------------------------------------- probing.hpp

// probing.hpp:105
inline std::vector<int> prioritize_probe_vars(const ProblemDef& p)
{
  std::vector<int32_t> order(p.n_vars);
  int32_t n = 0;
  detail::check(bp_prioritize_probe_vars(detail::handle(p), order.data(), &n));
  return std::vector<int>(order.begin(), order.begin() + n);
}

// probing.hpp:225 (both branches in one batched launch)
inline ProbeEntry probe_variable(const ProblemDef& p, const BoundsState& root, int v,
                                 const WorkPlan* /*plan*/ = nullptr)
{
  if (v < 0 || v >= p.n_vars) throw std::out_of_range("probe_variable: var out of range");
  bp_cache* c = nullptr;
  const int32_t vv = v;
  detail::check(bp_probe_variables(detail::handle(p), root.raw().data(), &vv, 1, &c));
  detail::CachePtr hold(c);
  ProbingCache pc = detail::to_pulse(p, c);
  if (!pc.entries[v]) throw std::runtime_error("probe_variable: engine returned no entry");
  return std::move(*pc.entries[v]);
}

// probing.hpp:243 (root = original bounds; candidates probed in priority order on the GPU)
inline ProbingCache build_cache(const ProblemDef& p, double budget_sec)
{
  bp_cache* c = nullptr;
  detail::check(bp_build_cache(detail::handle(p), budget_sec, &c));
  detail::CachePtr hold(c);
  return detail::to_pulse(p, c);
}

// probing.hpp:243 over several GPUs of this process (bp_build_cache_multi): the problem is
// replicated on each device of `devices`, candidates are interleaved over them, and the slices are
// gathered to devices[0] with NCCL and merged -- the same cache as build_cache(p, budget_sec).
inline ProbingCache build_cache(const ProblemDef& p, double budget_sec, const std::vector<int>& devices)
{
  if (devices.empty()) return pulse::gpu::build_cache(p, budget_sec);
  std::vector<bp_problem*> hs;
  for (int d : devices) hs.push_back(detail::handle(p, d));
  bp_cache* c = nullptr;
  detail::check(bp_build_cache_multi(hs.data(), (int32_t)hs.size(), budget_sec, nullptr, -1, &c, nullptr));
  detail::CachePtr hold(c);
  return detail::to_pulse(p, c);
}

// probing.hpp:292
inline BulkWarmStart assemble_bulk_warm_start(const ProbingCache& cache,
                                              const std::vector<std::pair<int, double>>& assignments)
{
  detail::CachePtr c = detail::from_pulse(cache);
  const int n        = cache.root.n_vars();
  std::vector<int32_t> vars;
  std::vector<double> vals;
  for (const auto& [v, x] : assignments) {
    vars.push_back(v);
    vals.push_back(x);
  }
  std::vector<double> raw(2 * (size_t)n);
  // capacities per bp.h: one conflict pair and at most one eviction per assignment
  (void)n;
  const size_t na = std::max<size_t>(assignments.size(), 1);
  std::vector<int32_t> conf(2 * na), ev(na);
  int32_t nconf = 0, nev = 0;
  detail::check(bp_assemble_bulk_warm_start(c.get(), vars.data(), vals.data(), (int32_t)vars.size(),
                                            raw.data(), conf.data(), &nconf, ev.data(), &nev));
  BulkWarmStart out;
  out.bounds = cache.root;
  detail::store(out.bounds, raw);
  for (int j = 0; j < nconf; ++j) out.conflicts.push_back({conf[2 * j], conf[2 * j + 1]});
  out.evicted.assign(ev.begin(), ev.begin() + nev);
  return out;
}

// ---------------------------------------------------------------- problem.hpp

// problem.hpp:102-243 with build() on the GPU (bp_build_problem): the same interface, results
// and exceptions as pulse::ProblemBuilder (duplicates of one (row, col) are summed in insertion
// order; the reference's std::sort leaves that order unspecified).
class ProblemBuilder {
 public:
  int add_var(std::string name, double lower, double upper, bool integer, double obj = 0.0)
  {
    var_names_.push_back(std::move(name));
    lower_.push_back(lower);
    upper_.push_back(upper);
    integer_.push_back(integer ? 1 : 0);
    obj_.push_back(obj);
    return static_cast<int>(var_names_.size()) - 1;
  }
  int add_row(std::string name, double lower, double upper)
  {
    cons_names_.push_back(std::move(name));
    cons_lower_.push_back(lower);
    cons_upper_.push_back(upper);
    return static_cast<int>(cons_names_.size()) - 1;
  }
  void add_entry(int row, int col, double val)
  {
    e_row_.push_back(row);
    e_col_.push_back(col);
    e_val_.push_back(val);
  }
  void set_objective(int var, double coeff) { obj_[var] = coeff; }
  void add_to_objective(int var, double coeff) { obj_[var] += coeff; }
  void set_var_lower(int var, double v) { lower_[var] = v; }
  void set_var_upper(int var, double v) { upper_[var] = v; }
  void set_var_integer(int var) { integer_[var] = 1; }
  void set_row_lower(int row, double v) { cons_lower_[row] = v; }
  void set_row_upper(int row, double v) { cons_upper_[row] = v; }
  double row_lower(int row) const { return cons_lower_[row]; }
  double row_upper(int row) const { return cons_upper_[row]; }
  void set_name(std::string n) { name_ = std::move(n); }
  void set_objective_name(std::string n) { obj_name_ = std::move(n); }
  int n_vars() const { return static_cast<int>(var_names_.size()); }
  int n_rows() const { return static_cast<int>(cons_names_.size()); }

  ProblemDef build() const
  {
    ProblemDef p;
    p.n_vars         = n_vars();
    p.n_cons         = n_rows();
    p.var_names      = var_names_;
    p.cons_names     = cons_names_;
    p.obj_coeffs     = obj_;
    p.cons_lower     = cons_lower_;
    p.cons_upper     = cons_upper_;
    p.name           = name_;
    p.objective_name = obj_name_;
    p.is_integer     = integer_;
    // the O(n + m) domain / row checks here for the reference's named messages (problem.hpp:164-173)
    for (int i = 0; i < p.n_vars; ++i) {
      double lo = lower_[i], up = upper_[i];
      if (integer_[i]) {
        if (is_finite(lo)) lo = ceil_eps(lo, 1e-9);
        if (is_finite(up)) up = floor_eps(up, 1e-9);
      }
      if (lo > up)
        throw std::runtime_error("variable '" + var_names_[i] + "' has empty domain after bound tightening");
    }
    for (int k = 0; k < p.n_cons; ++k)
      if (cons_lower_[k] > cons_upper_[k])
        throw std::runtime_error("constraint '" + cons_names_[k] + "' has crossed bounds");
    const size_t N = e_row_.size();
    p.row_start.resize(p.n_cons + 1);
    p.col_start.resize(p.n_vars + 1);
    p.row_col.resize(N);
    p.row_val.resize(N);
    p.col_row.resize(N);
    p.col_val.resize(N);
    p.var_lower.resize(p.n_vars);
    p.var_upper.resize(p.n_vars);
    bp_builder_desc d{p.n_vars, p.n_cons, (int64_t)N, e_row_.data(), e_col_.data(), e_val_.data(),
                      lower_.data(), upper_.data(), integer_.data(), cons_lower_.data(),
                      cons_upper_.data()};
    bp_built o{0, p.row_start.data(), p.row_col.data(), p.row_val.data(), p.col_start.data(),
               p.col_row.data(), p.col_val.data(), p.var_lower.data(), p.var_upper.data()};
    detail::check(bp_build_problem(&d, detail::registry().device, &o, nullptr));
    p.row_col.resize(o.nnz);
    p.row_val.resize(o.nnz);
    p.col_row.resize(o.nnz);
    p.col_val.resize(o.nnz);
    return p;
  }

 private:
  std::vector<std::string> var_names_;
  std::vector<double> lower_, upper_, obj_;
  std::vector<uint8_t> integer_;
  std::vector<std::string> cons_names_;
  std::vector<double> cons_lower_, cons_upper_;
  std::vector<int32_t> e_row_, e_col_;
  std::vector<double> e_val_;
  std::string name_;
  std::string obj_name_ = "OBJ";
};

// ---------------------------------------------------------------- lp.hpp

// Device copy of a pulse::LpInstance (lp.hpp:17-47) for repeated PDHG products; results are
// bit-identical to lpdetail::spmv_rows / spmv_cols.
class LpProducts {
 public:
  explicit LpProducts(const LpInstance& s) : n_(s.n_vars), m_(s.n_rows)
  {
    bp_lp_desc d{s.n_vars,        s.n_rows,           s.row_start.data(), s.row_col.data(),
                 s.row_val.data(), s.col_start.data(), s.col_row.data(),   s.col_val.data(),
                 s.obj.empty() ? nullptr : s.obj.data(), s.row_lower.data(), s.row_upper.data(),
                 s.var_lower.data(), s.var_upper.data()};
    detail::check(bp_lp_create(&d, detail::registry().device, &h_));
  }
  ~LpProducts()
  {
    if (h_) bp_lp_destroy(h_);
  }
  LpProducts(const LpProducts&) = delete;
  LpProducts& operator=(const LpProducts&) = delete;

  // lp.hpp:74-87
  void spmv_rows(const std::vector<double>& x, std::vector<double>& out)
  {
    if ((int)x.size() != n_) throw std::invalid_argument("spmv_rows: x has the wrong size");
    out.resize(m_);
    detail::check(bp_lp_spmv_rows(h_, x.data(), out.data()));
  }
  // lp.hpp:89-102
  void spmv_cols(const std::vector<double>& y, std::vector<double>& out)
  {
    if ((int)y.size() != m_) throw std::invalid_argument("spmv_cols: y has the wrong size");
    out.resize(n_);
    detail::check(bp_lp_spmv_cols(h_, y.data(), out.data()));
  }
  // lp.hpp:134-206. NOT bit-identical: the residual maxima are exact, but primal_obj / dual_obj
  // (and so gap and score) are compensated parallel sums, a few ulps from the reference's
  // sequential Neumaier sums; ax / aty are not returned. Callers that need the reference's exact
  // solve trajectory keep lpdetail::evaluate_kkt.
  lpdetail::KktInfo evaluate_kkt(const std::vector<double>& x, const std::vector<double>& y)
  {
    if ((int)x.size() != n_ || (int)y.size() != m_)
      throw std::invalid_argument("evaluate_kkt: x / y have the wrong size");
    double o[7];
    detail::check(bp_lp_evaluate_kkt(h_, x.data(), y.data(), o));
    lpdetail::KktInfo k;
    k.primal_res = o[0];
    k.dual_res   = o[1];
    k.gap        = o[2];
    k.primal_obj = o[3];
    k.dual_obj   = o[4];
    k.x_norm     = o[5];
    k.score      = o[6];
    return k;
  }
  // `iters` iterations of lp::solve's inner loop (lp.hpp:315-340) with fixed tau / sigma
  void pdhg_iterate(std::vector<double>& x, std::vector<double>& y, std::vector<double>& x_bar,
                    std::vector<double>& x_sum, std::vector<double>& y_sum, double tau, double sigma,
                    int iters)
  {
    for (const auto* v : {&x, &x_bar, &x_sum})
      if ((int)v->size() != n_) throw std::invalid_argument("pdhg_iterate: primal vector size");
    for (const auto* v : {&y, &y_sum})
      if ((int)v->size() != m_) throw std::invalid_argument("pdhg_iterate: dual vector size");
    detail::check(bp_lp_pdhg_iterate(h_, x.data(), y.data(), x_bar.data(), x_sum.data(),
                                     y_sum.data(), tau, sigma, iters));
  }

 private:
  int n_, m_;
  bp_lp* h_ = nullptr;
};

// lp.hpp:74 / :89 one-shot (uploads the instance; keep an LpProducts for repeated products)
inline void spmv_rows(const LpInstance& s, const std::vector<double>& x, std::vector<double>& out)
{
  LpProducts(s).spmv_rows(x, out);
}
inline void spmv_cols(const LpInstance& s, const std::vector<double>& y, std::vector<double>& out)
{
  LpProducts(s).spmv_cols(y, out);
}

// ---------------------------------------------------------------- rounding.hpp

// rounding.hpp:213 (both probes on the GPU engine)
inline ParallelProbeResult parallel_propagate(const ProblemDef& p, const BoundsState& base,
                                              const std::vector<int>& vars,
                                              const std::vector<double>& probe_vec_0,
                                              const std::vector<double>& probe_vec_1,
                                              const ProbingCache* cache, const WorkPlan& /*plan*/)
{
  if (probe_vec_0.size() != vars.size() || probe_vec_1.size() != vars.size())
    throw std::invalid_argument("parallel_propagate: candidate vector size mismatch");
  detail::CachePtr c;
  if (cache) c = detail::from_pulse(*cache);
  const size_t n = (size_t)p.n_vars, k = vars.size();
  std::vector<double> out(4 * n);
  int32_t inf[2], cnt[2], nev[2], nfx[2];
  std::vector<int32_t> ev(2 * k + 1), fv(2 * k + 1);
  std::vector<double> fx(2 * k + 1);
  std::vector<int32_t> vv(vars.begin(), vars.end());
  detail::check(bp_parallel_propagate(detail::handle(p), base.raw().data(), base.infeasible() ? 1 : 0,
                                      vv.data(), (int32_t)k, probe_vec_0.data(), probe_vec_1.data(),
                                      c.get(), out.data(), inf, cnt, ev.data(), nev, fv.data(),
                                      fx.data(), nfx));
  ParallelProbeResult r;
  for (int q = 0; q < 2; ++q) {
    ProbeResult& pr  = r.probe[q];
    pr.bounds        = detail::from_raw(p, out.data() + 2 * n * q, inf[q] != 0);
    pr.infeas_count  = cnt[q];
    pr.evicted.assign(ev.begin() + k * q, ev.begin() + k * q + nev[q]);
    for (int j = 0; j < nfx[q]; ++j) pr.fixed.push_back({fv[k * q + j], fx[k * q + j]});
  }
  return r;
}

// rounding.hpp:234 (device activity sweeps, most-violated-row scan and propagate)
inline std::optional<RepairResult> repair(const ProblemDef& p,
                                          std::vector<std::pair<int, double>> fixed,
                                          const Deadline& deadline, const RoundingConfig& cfg,
                                          const WorkPlan& /*plan*/)
{
  bp_rounding_config bc;
  bp_rounding_config_default(&bc);
  bc.repair_shift_cap = cfg.repair_shift_cap;
  const double rem = deadline.remaining_sec();
  const double dl  = rem == kInf ? 0.0 : (rem > 0.0 ? rem : 1e-300);  // 0 = never in bp.h
  std::vector<int32_t> fv(fixed.size() + 1);
  std::vector<double> fx(fixed.size() + 1), out(fixed.size() + 1), b(2 * (size_t)p.n_vars + 1);
  for (size_t j = 0; j < fixed.size(); ++j) {
    fv[j] = fixed[j].first;
    fx[j] = fixed[j].second;
  }
  int32_t ok = 0;
  detail::check(bp_repair(detail::handle(p), fv.data(), fx.data(), (int32_t)fixed.size(), dl, &bc,
                          &ok, out.data(), b.data()));
  if (!ok) return std::nullopt;
  for (size_t j = 0; j < fixed.size(); ++j) fixed[j].second = out[j];
  return RepairResult{std::move(fixed), detail::from_raw(p, b.data(), false)};
}

// rounding.hpp:393. The bulk loop runs in the engine's driver with device-resident bounds and
// the caller's generator; the continuous polish is the reference's own lp_polish (out of the
// GPU path's scope), applied under the reference's condition (rounding.hpp:551-556).
inline RoundingOutcome propagation_round(const ProblemDef& p, const SolutionVector& s,
                                         const ProbingCache* cache, const Deadline& deadline,
                                         Rng& rng, const RoundingConfig& cfg = {})
{
  if ((int)s.values.size() != p.n_vars) throw std::invalid_argument("solution dimension mismatch");
  detail::CachePtr c;
  if (cache) c = detail::from_pulse(*cache);
  bp_rounding_config bc;
  bp_rounding_config_default(&bc);
  bc.random_band        = cfg.random_band;
  bc.single_var_tail    = cfg.single_var_tail;
  bc.repair_enabled     = cfg.repair_enabled ? 1 : 0;
  bc.repair_attempt_cap = cfg.repair_attempt_cap;
  bc.repair_shift_cap   = cfg.repair_shift_cap;
  std::string st;
  {
    std::ostringstream os;
    os << rng;
    st = os.str();
  }
  std::vector<char> state(BP_RNG_STATE_BYTES, 0);
  if (st.size() + 1 > state.size()) throw std::runtime_error("rng state too large");
  std::memcpy(state.data(), st.c_str(), st.size() + 1);
  const double rem = deadline.remaining_sec();
  const double dl  = rem == kInf ? 0.0 : (rem > 0.0 ? rem : 1e-300);  // 0 = never in bp.h
  std::vector<double> values(p.n_vars);
  bp_rounding_outcome o{};
  detail::check(bp_propagation_round_rng(detail::handle(p), s.values.data(), c.get(), state.data(),
                                         (int64_t)state.size(), dl, &bc, values.data(), &o));
  {
    std::istringstream is(std::string(state.data()));
    is >> rng;
  }
  RoundingOutcome out;
  out.rounding_infeasible = o.rounding_infeasible != 0;
  out.timed_out           = o.timed_out != 0;
  out.completed           = o.completed != 0;
  out.repair_attempts     = o.repair_attempts;
  out.bulks_committed     = o.bulks_committed;
  out.set_count           = o.set_count;
  out.point = o.bounds_feasible ? lp_polish(p, values, cfg, deadline) : make_solution(p, values);
  return out;
}

}  // namespace pulse::gpu
