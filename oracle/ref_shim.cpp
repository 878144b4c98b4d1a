// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference headers (`/root/reference/proj/include/pulse/*.hpp`)
// compiled in place by oracle/Makefile into oracle/_ref/libpulse_ref.so. It lets the Python
// tests, the golden-fixture generator and bench.py's CPU baseline call the reference's own
// hot-path functions on plain arrays:
//   propagation.hpp:226 compute_activities, :378 tighten_bounds, :418 propagate
//   probing.hpp:30 make_branch_spec, :105 prioritize_probe_vars, :225 probe_variable,
//              :243 build_cache, :292 assemble_bulk_warm_start
//   rounding.hpp:35 initial_sort, :71 implied_slack_sort, :127 generate_candidate_values,
//              :213 parallel_propagate, :393 propagation_round
//   tests/testkit.hpp:69 random_instance (the acceptance/unit-test instance generator)
// Only glue lives here (array <-> std::vector marshalling); no algorithm is restated.
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "pulse/probing.hpp"
#include "pulse/propagation.hpp"
#include "pulse/rounding.hpp"
#include "pulse/lp.hpp"
#include "testkit.hpp"

using namespace pulse;

namespace {

struct RefCache {
  ProbingCache cache;
};

void bounds_from(BoundsState& b, const ProblemDef& p, const double* bounds2n, int infeasible)
{
  b = BoundsState(p);
  for (int i = 0; i < p.n_vars; ++i) {
    b.set_lower(i, bounds2n[2 * i]);
    b.set_upper(i, bounds2n[2 * i + 1]);
  }
  if (infeasible) b.mark_infeasible();
}

void bounds_to(const BoundsState& b, double* bounds2n, int* infeasible)
{
  std::memcpy(bounds2n, b.raw().data(), sizeof(double) * b.raw().size());
  if (infeasible) *infeasible = b.infeasible() ? 1 : 0;
}

PropagationLimits limits_from(const double* lim)
{
  // lim = {max_rounds, time_limit, abs_threshold, rel_threshold, incremental}
  PropagationLimits l;
  if (lim) {
    l.max_rounds    = static_cast<int>(lim[0]);
    l.time_limit    = lim[1];
    l.abs_threshold = lim[2];
    l.rel_threshold = lim[3];
    l.incremental   = lim[4] != 0.0;
  }
  return l;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- problems
// Builds through ProblemBuilder::build (problem.hpp:141): sort, coalesce, drop zeros,
// integral bound rounding, stable transpose.
void* ref_problem_build(int n_vars, int n_cons, const double* var_lower, const double* var_upper,
                        const uint8_t* is_integer, const double* obj, const double* cons_lower,
                        const double* cons_upper, long long n_entries, const int* e_row,
                        const int* e_col, const double* e_val)
{
  ProblemBuilder b;
  for (int i = 0; i < n_vars; ++i) {
    b.add_var("x" + std::to_string(i), var_lower[i], var_upper[i], is_integer[i] != 0,
              obj ? obj[i] : 0.0);
  }
  for (int k = 0; k < n_cons; ++k) b.add_row("c" + std::to_string(k), cons_lower[k], cons_upper[k]);
  for (long long e = 0; e < n_entries; ++e) b.add_entry(e_row[e], e_col[e], e_val[e]);
  return new ProblemDef(b.build());
}

// Wraps an already-built CSR (sorted, coalesced, zero-free, integral bounds applied) without
// re-sorting; the CSC is the stable transpose exactly as problem.hpp:211-225 builds it.
void* ref_problem_from_csr(int n_vars, int n_cons, const int* row_start, const int* row_col,
                           const double* row_val, const double* var_lower, const double* var_upper,
                           const uint8_t* is_integer, const double* cons_lower,
                           const double* cons_upper)
{
  auto* p   = new ProblemDef();
  p->n_vars = n_vars;
  p->n_cons = n_cons;
  const int nnz = row_start[n_cons];
  p->var_lower.assign(var_lower, var_lower + n_vars);
  p->var_upper.assign(var_upper, var_upper + n_vars);
  p->is_integer.assign(is_integer, is_integer + n_vars);
  p->obj_coeffs.assign(n_vars, 0.0);
  p->cons_lower.assign(cons_lower, cons_lower + n_cons);
  p->cons_upper.assign(cons_upper, cons_upper + n_cons);
  p->row_start.assign(row_start, row_start + n_cons + 1);
  p->row_col.assign(row_col, row_col + nnz);
  p->row_val.assign(row_val, row_val + nnz);
  p->col_start.assign(n_vars + 1, 0);
  for (int c : p->row_col) p->col_start[c + 1]++;
  for (int i = 0; i < n_vars; ++i) p->col_start[i + 1] += p->col_start[i];
  p->col_row.resize(nnz);
  p->col_val.resize(nnz);
  std::vector<int> cursor(p->col_start.begin(), p->col_start.end() - 1);
  for (int k = 0; k < n_cons; ++k) {
    for (int e = p->row_start[k]; e < p->row_start[k + 1]; ++e) {
      const int i   = p->row_col[e];
      const int dst = cursor[i]++;
      p->col_row[dst] = k;
      p->col_val[dst] = p->row_val[e];
    }
  }
  p->var_names.resize(n_vars);
  p->cons_names.resize(n_cons);
  return p;
}

void ref_problem_free(void* p) { delete static_cast<ProblemDef*>(p); }
void ref_problem_set_obj(void* pv, const double* obj)
{
  auto* p = static_cast<ProblemDef*>(pv);
  p->obj_coeffs.assign(obj, obj + p->n_vars);
}

void ref_problem_dims(const void* pv, int* n_vars, int* n_cons, int* nnz)
{
  const auto* p = static_cast<const ProblemDef*>(pv);
  *n_vars = p->n_vars;
  *n_cons = p->n_cons;
  *nnz    = p->nnz();
}

void ref_problem_export(const void* pv, int* row_start, int* row_col, double* row_val,
                        int* col_start, int* col_row, double* col_val, double* var_lower,
                        double* var_upper, uint8_t* is_integer, double* cons_lower,
                        double* cons_upper, double* obj)
{
  const auto* p = static_cast<const ProblemDef*>(pv);
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
  };
  cp(row_start, p->row_start);
  cp(row_col, p->row_col);
  cp(row_val, p->row_val);
  cp(col_start, p->col_start);
  cp(col_row, p->col_row);
  cp(col_val, p->col_val);
  cp(var_lower, p->var_lower);
  cp(var_upper, p->var_upper);
  cp(is_integer, p->is_integer);
  cp(cons_lower, p->cons_lower);
  cp(cons_upper, p->cons_upper);
  cp(obj, p->obj_coeffs);
}

// ---------------------------------------------------------------- testkit generator
void* ref_rng_new(unsigned long long seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }

// testkit.hpp:69 random_instance with RandomInstanceOptions (testkit.hpp:57-65).
void* ref_random_instance(void* rng, int max_vars, int max_rows, int max_bound_span,
                          double density, int force_feasible, int allow_continuous,
                          int allow_one_sided)
{
  testkit::RandomInstanceOptions opt;
  opt.max_vars         = max_vars;
  opt.max_rows         = max_rows;
  opt.max_bound_span   = max_bound_span;
  opt.density          = density;
  opt.force_feasible   = force_feasible != 0;
  opt.allow_continuous = allow_continuous != 0;
  opt.allow_one_sided  = allow_one_sided != 0;
  return new ProblemDef(testkit::random_instance(*static_cast<std::mt19937_64*>(rng), opt));
}

// Draws uniform_int(lo, hi) from the rng (the call testkit/tests make for assignments).
int ref_rng_uniform_int(void* rng, int lo, int hi)
{
  std::uniform_int_distribution<int> d(lo, hi);
  return d(*static_cast<std::mt19937_64*>(rng));
}
double ref_rng_uniform_real(void* rng, double lo, double hi)
{
  std::uniform_real_distribution<double> d(lo, hi);
  return d(*static_cast<std::mt19937_64*>(rng));
}

int ref_max_threads() { return max_threads(); }

// ---------------------------------------------------------------- propagation
// propagation.hpp:226. rows == nullptr && nrows < 0 => all rows. use_plan selects the binned path.
void ref_compute_activities(const void* pv, const double* bounds2n, const int* rows, int nrows,
                            int use_plan, double* act2m, int* ninf_min, int* ninf_max)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  BoundsState b;
  bounds_from(b, p, bounds2n, 0);
  ActivityState a;
  a.resize(p.n_cons);
  // Seed with caller values so rows outside a subset keep them (compute_activities only resizes
  // on size mismatch, propagation.hpp:230).
  std::memcpy(a.act.data(), act2m, sizeof(double) * 2 * p.n_cons);
  std::memcpy(a.n_inf_min.data(), ninf_min, sizeof(int) * p.n_cons);
  std::memcpy(a.n_inf_max.data(), ninf_max, sizeof(int) * p.n_cons);
  std::vector<int> r;
  if (nrows >= 0) r.assign(rows, rows + nrows);
  WorkPlan plan;
  if (use_plan) plan = build_work_plan(p);
  compute_activities(p, b, nrows >= 0 ? &r : nullptr, a, use_plan ? &plan : nullptr);
  std::memcpy(act2m, a.act.data(), sizeof(double) * 2 * p.n_cons);
  std::memcpy(ninf_min, a.n_inf_min.data(), sizeof(int) * p.n_cons);
  std::memcpy(ninf_max, a.n_inf_max.data(), sizeof(int) * p.n_cons);
}

// propagation.hpp:378. Returns the number of changed vars written to `changed`.
int ref_tighten_bounds(const void* pv, double* bounds2n, int* infeasible, const double* act2m,
                       const int* ninf_min, const int* ninf_max, const int* vars, int nvars,
                       const double* lim, int* changed, int* crossed)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  BoundsState b;
  bounds_from(b, p, bounds2n, *infeasible);
  ActivityState a;
  a.act.assign(act2m, act2m + 2 * p.n_cons);
  a.n_inf_min.assign(ninf_min, ninf_min + p.n_cons);
  a.n_inf_max.assign(ninf_max, ninf_max + p.n_cons);
  std::vector<int> v;
  if (nvars >= 0) v.assign(vars, vars + nvars);
  const auto ch = tighten_bounds(p, b, a, nvars >= 0 ? &v : nullptr, limits_from(lim), crossed);
  bounds_to(b, bounds2n, infeasible);
  for (size_t j = 0; j < ch.size(); ++j) changed[j] = ch[j];
  return static_cast<int>(ch.size());
}

// propagation.hpp:418. out3 = {status (0 Tightened, 1 Infeasible, 2 Unchanged), rounds, crossed}.
void ref_propagate(const void* pv, double* bounds2n, int* infeasible, const double* lim,
                   int use_plan, int* out3)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  BoundsState b;
  bounds_from(b, p, bounds2n, *infeasible);
  WorkPlan plan;
  if (use_plan) plan = build_work_plan(p);
  const auto r = propagate(p, b, limits_from(lim), use_plan ? &plan : nullptr);
  bounds_to(b, bounds2n, infeasible);
  out3[0] = static_cast<int>(r.status);
  out3[1] = r.rounds;
  out3[2] = r.crossed_vars;
}

// ---------------------------------------------------------------- probing
// probing.hpp:30. Returns 0 if no spec; else kind+1, and fills spec4 = {dl, du, ul, uu}.
int ref_make_branch_spec(double lo, double up, double* spec4)
{
  ProblemBuilder pb;
  pb.add_var("v", -kInf, kInf, false);
  const ProblemDef p = pb.build();
  BoundsState b(p);
  b.set_lower(0, lo);
  b.set_upper(0, up);
  const auto s = make_branch_spec(b, 0);
  if (!s) return 0;
  spec4[0] = s->down_lower;
  spec4[1] = s->down_upper;
  spec4[2] = s->up_lower;
  spec4[3] = s->up_upper;
  return static_cast<int>(s->kind) + 1;
}

int ref_prioritize_probe_vars(const void* pv, int* order)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  const auto o  = prioritize_probe_vars(p);
  for (size_t j = 0; j < o.size(); ++j) order[j] = o[j];
  return static_cast<int>(o.size());
}

// Cache handle API (probing.hpp:87-98). The handle owns a ProbingCache.
void* ref_cache_new_empty(const void* pv)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  auto* c       = new RefCache();
  c->cache.root = BoundsState(p);
  c->cache.entries.resize(p.n_vars);
  return c;
}
void* ref_build_cache(const void* pv, double budget_sec)
{
  auto* c  = new RefCache();
  c->cache = build_cache(*static_cast<const ProblemDef*>(pv), budget_sec);
  return c;
}
// probe_variable (probing.hpp:225) from a caller root; stores the entry into the cache handle.
void ref_cache_probe_into(void* cv, const void* pv, const double* root2n, int v, int use_plan)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  auto* c       = static_cast<RefCache*>(cv);
  BoundsState root;
  bounds_from(root, p, root2n, 0);
  WorkPlan plan;
  if (use_plan) plan = build_work_plan(p);
  c->cache.entries[v] = probe_variable(p, root, v, use_plan ? &plan : nullptr);
}
void ref_cache_free(void* cv) { delete static_cast<RefCache*>(cv); }
void ref_cache_stats(const void* cv, int* n_probed, int* n_infeasible_branches)
{
  const auto* c          = static_cast<const RefCache*>(cv);
  *n_probed              = c->cache.n_probed;
  *n_infeasible_branches = c->cache.n_infeasible_branches;
}
// Entry header: returns 0 if absent; else fills hdr = {kind, forces_down, forces_up,
// down.feasible, up.feasible, n_down, n_up} and br4 = {down.lo, down.up, up.lo, up.up}.
int ref_cache_entry(const void* cv, int v, int* hdr7, double* br4)
{
  const auto* c = static_cast<const RefCache*>(cv);
  if (!c->cache.has(v)) return 0;
  const auto& e = c->cache.at(v);
  hdr7[0]       = static_cast<int>(e.kind);
  hdr7[1]       = e.forces_down;
  hdr7[2]       = e.forces_up;
  hdr7[3]       = e.down.feasible;
  hdr7[4]       = e.up.feasible;
  hdr7[5]       = static_cast<int>(e.down.deltas.size());
  hdr7[6]       = static_cast<int>(e.up.deltas.size());
  br4[0]        = e.down.branch_lower;
  br4[1]        = e.down.branch_upper;
  br4[2]        = e.up.branch_lower;
  br4[3]        = e.up.branch_upper;
  return 1;
}
void ref_cache_deltas(const void* cv, int v, int side, int* vars, double* lo, double* up)
{
  const auto* c   = static_cast<const RefCache*>(cv);
  const auto& br  = side ? c->cache.at(v).up : c->cache.at(v).down;
  for (size_t j = 0; j < br.deltas.size(); ++j) {
    vars[j] = br.deltas[j].var;
    lo[j]   = br.deltas[j].new_lower;
    up[j]   = br.deltas[j].new_upper;
  }
}
// Installs an externally produced entry (e.g. a GPU-built cache) into the handle so the
// reference rounding driver can consume it.
void ref_cache_set_entry(void* cv, int v, const int* hdr7, const double* br4, const int* dvars,
                         const double* dlo, const double* dup)
{
  auto* c = static_cast<RefCache*>(cv);
  ProbeEntry e;
  e.var               = v;
  e.kind              = static_cast<BranchKind>(hdr7[0]);
  e.forces_down       = hdr7[1] != 0;
  e.forces_up         = hdr7[2] != 0;
  e.down.feasible     = hdr7[3] != 0;
  e.up.feasible       = hdr7[4] != 0;
  e.down.branch_lower = br4[0];
  e.down.branch_upper = br4[1];
  e.up.branch_lower   = br4[2];
  e.up.branch_upper   = br4[3];
  int off = 0;
  for (int j = 0; j < hdr7[5]; ++j, ++off) e.down.deltas.push_back({dvars[off], dlo[off], dup[off]});
  for (int j = 0; j < hdr7[6]; ++j, ++off) e.up.deltas.push_back({dvars[off], dlo[off], dup[off]});
  c->cache.entries[v] = std::move(e);
  c->cache.n_probed = 0;
  c->cache.n_infeasible_branches = 0;
  for (const auto& x : c->cache.entries) {
    if (!x) continue;
    c->cache.n_probed++;
    if (!x->down.feasible) c->cache.n_infeasible_branches++;
    if (!x->up.feasible) c->cache.n_infeasible_branches++;
  }
}

// A reference ProbingCache holding every entry of a packed engine cache (bp_cache_pack layout:
// header {ne, nd, n_fallback, certified}, per entry {i32 var, i32 kind, u8 feas[2], u8 force[2],
// f64 branch[4], i64 count[2]}, then the deltas SoA) -- the bulk form of ref_cache_set_entry.
void* ref_cache_from_packed(const void* pv, const char* buf, long long bytes)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  auto* c       = new RefCache();
  c->cache.root = BoundsState(p);
  c->cache.entries.resize(p.n_vars);
  long long hdr[4];
  std::memcpy(hdr, buf, 32);
  const long long ne = hdr[0], nd = hdr[1];
  if (bytes < 32 + ne * 60 + nd * 20) {
    delete c;
    return nullptr;
  }
  const char* q   = buf + 32;
  const char* dvp = buf + 32 + ne * 60;
  const char* dlp = dvp + 4 * nd;
  const char* dup = dlp + 8 * nd;
  long long off   = 0;
  for (long long e = 0; e < ne; ++e, q += 60) {
    int var, kind;
    unsigned char feas[2], force[2];
    double br[4];
    long long cnt[2];
    std::memcpy(&var, q, 4);
    std::memcpy(&kind, q + 4, 4);
    std::memcpy(feas, q + 8, 2);
    std::memcpy(force, q + 10, 2);
    std::memcpy(br, q + 12, 32);
    std::memcpy(cnt, q + 44, 16);
    ProbeEntry x;
    x.var               = var;
    x.kind              = static_cast<BranchKind>(kind);
    x.forces_down       = force[0] != 0;
    x.forces_up         = force[1] != 0;
    x.down.feasible     = feas[0] != 0;
    x.up.feasible       = feas[1] != 0;
    x.down.branch_lower = br[0];
    x.down.branch_upper = br[1];
    x.up.branch_lower   = br[2];
    x.up.branch_upper   = br[3];
    for (int side = 0; side < 2; ++side)
      for (long long j = 0; j < cnt[side]; ++j, ++off) {
        int dv;
        double lo, up;
        std::memcpy(&dv, dvp + 4 * off, 4);
        std::memcpy(&lo, dlp + 8 * off, 8);
        std::memcpy(&up, dup + 8 * off, 8);
        (side ? x.up : x.down).deltas.push_back({dv, lo, up});
      }
    c->cache.entries[var] = std::move(x);
  }
  for (const auto& x : c->cache.entries) {
    if (!x) continue;
    c->cache.n_probed++;
    if (!x->down.feasible) c->cache.n_infeasible_branches++;
    if (!x->up.feasible) c->cache.n_infeasible_branches++;
  }
  return c;
}

// probing.hpp:292. Writes merged bounds; returns #conflicts; fills conflicts (pairs) and
// evicted list (count in *n_evicted).
int ref_assemble_bulk_warm_start(const void* cv, const int* vars, const double* vals, int nassign,
                                 double* bounds2n, int* conflicts, int* evicted, int* n_evicted)
{
  const auto* c = static_cast<const RefCache*>(cv);
  std::vector<std::pair<int, double>> as;
  for (int j = 0; j < nassign; ++j) as.push_back({vars[j], vals[j]});
  const auto ws = assemble_bulk_warm_start(c->cache, as);
  bounds_to(ws.bounds, bounds2n, nullptr);
  for (size_t j = 0; j < ws.conflicts.size(); ++j) {
    conflicts[2 * j]     = ws.conflicts[j].first;
    conflicts[2 * j + 1] = ws.conflicts[j].second;
  }
  for (size_t j = 0; j < ws.evicted.size(); ++j) evicted[j] = ws.evicted[j];
  *n_evicted = static_cast<int>(ws.evicted.size());
  return static_cast<int>(ws.conflicts.size());
}

// ---------------------------------------------------------------- rounding
int ref_initial_sort(const void* pv, const double* values, int* order)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  SolutionVector s;
  s.values.assign(values, values + p.n_vars);
  const auto o = initial_sort(p, s);
  for (size_t j = 0; j < o.size(); ++j) order[j] = o[j];
  return static_cast<int>(o.size());
}

void ref_implied_slack_sort(const void* pv, const double* act2m, const int* ninf_min,
                            const int* ninf_max, int* vars, int nvars)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  ActivityState a;
  a.act.assign(act2m, act2m + 2 * p.n_cons);
  a.n_inf_min.assign(ninf_min, ninf_min + p.n_cons);
  a.n_inf_max.assign(ninf_max, ninf_max + p.n_cons);
  std::vector<int> v(vars, vars + nvars);
  implied_slack_sort(p, a, v);
  for (int j = 0; j < nvars; ++j) vars[j] = v[j];
}

int ref_get_bulk_size(int remaining, int recovery, int tail)
{
  return get_bulk_size(remaining, recovery != 0, tail);
}

void ref_generate_candidate_values(void* rng, const double* values, int n_vars, const int* vars,
                                   int nvars, const double* bounds2n, double band, double* v0,
                                   double* v1)
{
  SolutionVector s;
  s.values.assign(values, values + n_vars);
  ProblemBuilder pb;
  for (int i = 0; i < n_vars; ++i) pb.add_var("x", -kInf, kInf, false);
  const ProblemDef p = pb.build();
  BoundsState b;
  bounds_from(b, p, bounds2n, 0);
  std::vector<int> vv(vars, vars + nvars);
  auto [a, c] = generate_candidate_values(s, vv, b, *static_cast<std::mt19937_64*>(rng), band);
  for (int j = 0; j < nvars; ++j) {
    v0[j] = a[j];
    v1[j] = c[j];
  }
}

// rounding.hpp:213. For each probe k: bounds (2n), infeasible flag, infeas_count, evicted list,
// fixed list. Outputs are sized by the caller (n_vars bounds, nvars lists).
void ref_parallel_propagate(const void* pv, const double* base2n, int base_infeasible,
                            const int* vars, int nvars, const double* pv0, const double* pv1,
                            const void* cv, double* out_bounds0, double* out_bounds1,
                            int* out_info /* [2][4]: infeasible, infeas_count, n_evicted, n_fixed */,
                            int* evicted0, int* evicted1, int* fixed_vars0, double* fixed_vals0,
                            int* fixed_vars1, double* fixed_vals1)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  BoundsState base;
  bounds_from(base, p, base2n, base_infeasible);
  const WorkPlan plan = build_work_plan(p);
  std::vector<int> v(vars, vars + nvars);
  std::vector<double> a(pv0, pv0 + nvars), b(pv1, pv1 + nvars);
  const auto* cache = cv ? &static_cast<const RefCache*>(cv)->cache : nullptr;
  const auto r      = parallel_propagate(p, base, v, a, b, cache, plan);
  double* ob[2]     = {out_bounds0, out_bounds1};
  int* ev[2]        = {evicted0, evicted1};
  int* fv[2]        = {fixed_vars0, fixed_vars1};
  double* fx[2]     = {fixed_vals0, fixed_vals1};
  for (int k = 0; k < 2; ++k) {
    int inf = 0;
    bounds_to(r.probe[k].bounds, ob[k], &inf);
    out_info[4 * k + 0] = inf;
    out_info[4 * k + 1] = r.probe[k].infeas_count;
    out_info[4 * k + 2] = static_cast<int>(r.probe[k].evicted.size());
    out_info[4 * k + 3] = static_cast<int>(r.probe[k].fixed.size());
    for (size_t j = 0; j < r.probe[k].evicted.size(); ++j) ev[k][j] = r.probe[k].evicted[j];
    for (size_t j = 0; j < r.probe[k].fixed.size(); ++j) {
      fv[k][j] = r.probe[k].fixed[j].first;
      fx[k][j] = r.probe[k].fixed[j].second;
    }
  }
}

// rounding.hpp:234 repair(p, fixed, Deadline::never(), cfg{shift_cap}, plan). Returns 1 when a
// RepairResult is present (shifted values in out_vals, its bounds in out_bounds2n), else 0.
int ref_repair(const void* pv, const int* fixed_vars, const double* fixed_vals, int nfixed,
               int shift_cap, double* out_vals, double* out_bounds2n)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  std::vector<std::pair<int, double>> fixed(nfixed);
  for (int j = 0; j < nfixed; ++j) fixed[j] = {fixed_vars[j], fixed_vals[j]};
  RoundingConfig cfg;
  cfg.repair_shift_cap = shift_cap;
  const WorkPlan plan  = build_work_plan(p);
  const auto r         = repair(p, fixed, Deadline::never(), cfg, plan);
  if (!r) return 0;
  for (int j = 0; j < nfixed; ++j) out_vals[j] = r->values[j].second;
  bounds_to(r->bounds, out_bounds2n, nullptr);
  return 1;
}

// lp.hpp:74-102 on LpInstance::relax(p) (the products only read the CSR / CSC).
void ref_lp_spmv_rows(const void* pv, const double* x, double* out)
{
  const auto s = LpInstance::relax(*static_cast<const ProblemDef*>(pv));
  std::vector<double> xv(x, x + s.n_vars), o(s.n_rows);
  lpdetail::spmv_rows(s, xv, o);
  std::copy(o.begin(), o.end(), out);
}
void ref_lp_spmv_cols(const void* pv, const double* y, double* out)
{
  const auto s = LpInstance::relax(*static_cast<const ProblemDef*>(pv));
  std::vector<double> yv(y, y + s.n_rows), o(s.n_vars);
  lpdetail::spmv_cols(s, yv, o);
  std::copy(o.begin(), o.end(), out);
}

// lpdetail::evaluate_kkt (lp.hpp:134) at (x, y): out7 = {primal_res, dual_res, gap, primal_obj,
// dual_obj, x_norm, score}.
void ref_lp_evaluate_kkt(const void* pv, const double* x, const double* y, double* out7)
{
  const auto s = LpInstance::relax(*static_cast<const ProblemDef*>(pv));
  std::vector<double> X(x, x + s.n_vars), Y(y, y + s.n_rows), ax(s.n_rows), aty(s.n_vars);
  const auto k = lpdetail::evaluate_kkt(s, X, Y, ax, aty);
  const double v[7] = {k.primal_res, k.dual_res, k.gap, k.primal_obj, k.dual_obj, k.x_norm, k.score};
  std::copy(v, v + 7, out7);
}

// The inner PDHG iteration of lp::solve (lp.hpp:315-340) restated verbatim around the reference's
// own lpdetail::spmv_rows / spmv_cols and pulse::clamp, `iters` times with fixed tau / sigma.
void ref_lp_pdhg_iterate(const void* pv, double* x, double* y, double* x_bar, double* x_sum,
                         double* y_sum, double tau, double sigma, int iters)
{
  const auto s = LpInstance::relax(*static_cast<const ProblemDef*>(pv));
  const int n = s.n_vars, m = s.n_rows;
  std::vector<double> X(x, x + n), Y(y, y + m), XB(x_bar, x_bar + n), XS(x_sum, x_sum + n),
      YS(y_sum, y_sum + m), xn(n), ax(m), aty(n);
  for (int it = 0; it < iters; ++it) {
    lpdetail::spmv_rows(s, XB, ax);
    for (int k = 0; k < m; ++k) {
      const double v    = Y[k] + sigma * ax[k];
      const double proj = clamp(v / sigma, s.row_lower[k], s.row_upper[k]);
      Y[k]              = v - sigma * proj;
    }
    lpdetail::spmv_cols(s, Y, aty);
    for (int i = 0; i < n; ++i) {
      const double v = X[i] - tau * (s.obj[i] + aty[i]);
      xn[i]          = clamp(v, s.var_lower[i], s.var_upper[i]);
      XB[i]          = 2.0 * xn[i] - X[i];
    }
    std::swap(X, xn);
    for (int i = 0; i < n; ++i) XS[i] += X[i];
    for (int k = 0; k < m; ++k) YS[k] += Y[k];
  }
  std::copy(X.begin(), X.end(), x);
  std::copy(Y.begin(), Y.end(), y);
  std::copy(XB.begin(), XB.end(), x_bar);
  std::copy(XS.begin(), XS.end(), x_sum);
  std::copy(YS.begin(), YS.end(), y_sum);
}

// rounding.hpp:393 with a cache handle (or null) and Rng(seed). lp_polish runs inside (OUT OF
// SCOPE for parity; callers compare integer values and flags). out_values has n_vars entries.
// flags = {rounding_infeasible, timed_out, completed, repair_attempts, bulks_committed, set_count}
void ref_propagation_round(const void* pv, const double* start, const void* cv,
                           unsigned long long seed, double deadline_sec, double random_band,
                           int repair_enabled, double* out_values, int* flags6)
{
  const auto& p = *static_cast<const ProblemDef*>(pv);
  std::vector<double> x(start, start + p.n_vars);
  const auto s = make_solution(p, x);
  Rng rng(seed);
  RoundingConfig cfg;
  cfg.random_band    = random_band;
  cfg.repair_enabled = repair_enabled != 0;
  const auto* cache  = cv ? &static_cast<const RefCache*>(cv)->cache : nullptr;
  const Deadline dl  = deadline_sec > 0 ? Deadline(deadline_sec) : Deadline::never();
  const auto out     = propagation_round(p, s, cache, dl, rng, cfg);
  for (int i = 0; i < p.n_vars; ++i) out_values[i] = out.point.values[i];
  flags6[0] = out.rounding_infeasible;
  flags6[1] = out.timed_out;
  flags6[2] = out.completed;
  flags6[3] = out.repair_attempts;
  flags6[4] = out.bulks_committed;
  flags6[5] = out.set_count;
}

}  // extern "C"
