// TEST INFRASTRUCTURE — the C++ drop-in (include/pulse_gpu.hpp) against the UNMODIFIED reference,
// side by side in one process: every pulse:: hot-path function is called on the CPU (reference
// headers from /root/reference, compiled in place by oracle/Makefile) and through pulse::gpu:: on
// the B200 engine, on the reference's own instance streams (tests/testkit.hpp:69 random_instance,
// seeds of acceptance.cpp:40 / :89 and test_rounding.cpp), plus larger mixed instances with heavy
// rows. Everything is compared bit for bit. One PASS/FAIL line per criterion, like acceptance.cpp;
// exit status = number of failures.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "pulse_gpu.hpp"
#include "testkit.hpp"

using namespace pulse;
namespace pg = pulse::gpu;

namespace {

int g_failures = 0;

void report(const std::string& name, bool pass, const std::string& detail)
{
  std::printf("%s  %s (%s)\n", pass ? "PASS" : "FAIL", name.c_str(), detail.c_str());
  std::fflush(stdout);
  if (!pass) ++g_failures;
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b)
{
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 8 * a.size()) == 0);
}

bool same_state(const BoundsState& a, const BoundsState& b)
{
  return a.infeasible() == b.infeasible() && same_bits(a.raw(), b.raw());
}

bool same_result(const PropagationResult& a, const PropagationResult& b)
{
  return a.status == b.status && a.rounds == b.rounds && a.crossed_vars == b.crossed_vars;
}

bool same_branch(const ProbeBranch& a, const ProbeBranch& b)
{
  if (a.feasible != b.feasible || a.deltas.size() != b.deltas.size()) return false;
  if (std::memcmp(&a.branch_lower, &b.branch_lower, 8) || std::memcmp(&a.branch_upper, &b.branch_upper, 8))
    return false;
  for (size_t d = 0; d < a.deltas.size(); ++d) {
    if (a.deltas[d].var != b.deltas[d].var) return false;
    if (std::memcmp(&a.deltas[d].new_lower, &b.deltas[d].new_lower, 8)) return false;
    if (std::memcmp(&a.deltas[d].new_upper, &b.deltas[d].new_upper, 8)) return false;
  }
  return true;
}

bool same_entry(const ProbeEntry& a, const ProbeEntry& b)
{
  return a.var == b.var && a.kind == b.kind && a.forces_down == b.forces_down &&
         a.forces_up == b.forces_up && same_branch(a.down, b.down) && same_branch(a.up, b.up);
}

bool same_cache(const ProbingCache& a, const ProbingCache& b)
{
  if (a.entries.size() != b.entries.size() || a.n_probed != b.n_probed ||
      a.n_infeasible_branches != b.n_infeasible_branches || !same_state(a.root, b.root))
    return false;
  for (size_t v = 0; v < a.entries.size(); ++v) {
    if (a.entries[v].has_value() != b.entries[v].has_value()) return false;
    if (a.entries[v] && !same_entry(*a.entries[v], *b.entries[v])) return false;
  }
  return true;
}

// Mixed instance with fractional data (binary / integer / continuous, one- and two-sided rows) and
// optionally a few rows longer than kSumSegment, so activities take the 16384-segment tree.
ProblemDef mixed_instance(uint64_t seed, int n, int m, int heavy_rows, int heavy_len)
{
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  ProblemBuilder b;
  std::vector<double> pt(n);
  std::vector<int> kind(n);
  for (int i = 0; i < n; ++i) {
    const double r = U(rng);
    kind[i]        = r < 0.5 ? 0 : (r < 0.8 ? 1 : 2);
    const double up = kind[i] == 0 ? 1.0 : (kind[i] == 1 ? 10.0 : 1.0 + 99.0 * U(rng));
    b.add_var("x" + std::to_string(i), 0.0, up, kind[i] != 2, 0.0);
    pt[i] = kind[i] == 2 ? up * U(rng) : std::floor((up + 1.0) * U(rng));
    if (pt[i] > up) pt[i] = up;
  }
  for (int k = 0; k < m; ++k) {
    const int len = k < heavy_rows ? heavy_len : 2 + (int)(10 * U(rng));
    std::vector<std::pair<int, double>> ent;
    double lhs = 0.0;
    for (int j = 0; j < len; ++j) {
      const int c  = (int)(n * U(rng)) % n;
      double a     = kind[c] == 2 ? 0.1 + 9.9 * U(rng) : 1.0 + std::floor(9.0 * U(rng));
      if (U(rng) < 0.5) a = -a;
      ent.push_back({c, a});
      lhs += a * pt[c];
    }
    const double r  = U(rng);
    const double lo = r < 0.7 ? -kInf : lhs - 3.0 * U(rng);
    const double up = r < 0.7 || r > 0.9 ? lhs + 3.0 * U(rng) : kInf;
    b.add_row("c" + std::to_string(k), lo, up);
    for (auto& [c, a] : ent) b.add_entry(k, c, a);
  }
  return b.build();
}

// ---------------------------------------------------------------- criteria

void propagation_stream()
{
  std::mt19937_64 rng(20240501);  // acceptance.cpp:40
  int bad = 0, acts_bad = 0, tight_bad = 0;
  for (int t = 0; t < 1000; ++t) {
    const ProblemDef p = testkit::random_instance(rng);
    for (int inc = 0; inc < 2; ++inc) {
      PropagationLimits lim;
      lim.incremental = inc == 1;
      BoundsState a(p), g(p);
      const auto ra = propagate(p, a, lim);
      const auto rg = pg::propagate(p, g, lim);
      if (!same_result(ra, rg) || !same_state(a, g)) ++bad;
    }
    // one activity + tightening sweep, full and over a subset
    BoundsState a(p), g(p);
    ActivityState aa, ga;
    compute_activities(p, a, nullptr, aa);
    pg::compute_activities(p, g, nullptr, ga);
    if (!same_bits(aa.act, ga.act) || aa.n_inf_min != ga.n_inf_min || aa.n_inf_max != ga.n_inf_max) ++acts_bad;
    int ca = 0, cg = 0;
    const auto cha = tighten_bounds(p, a, aa, nullptr, {}, &ca);
    const auto chg = pg::tighten_bounds(p, g, ga, nullptr, {}, &cg);
    if (cha != chg || ca != cg || !same_state(a, g)) ++tight_bad;
    std::vector<int> rows, vars;
    for (int k = 0; k < p.n_cons; k += 2) rows.push_back(k);
    for (int i = 1; i < p.n_vars; i += 2) vars.push_back(i);
    compute_activities(p, a, &rows, aa);
    pg::compute_activities(p, g, &rows, ga);
    if (!same_bits(aa.act, ga.act) || aa.n_inf_min != ga.n_inf_min) ++acts_bad;
    const auto sa = tighten_bounds(p, a, aa, &vars, {}, &ca);
    const auto sg = pg::tighten_bounds(p, g, ga, &vars, {}, &cg);
    if (sa != sg || ca != cg || !same_state(a, g)) ++tight_bad;
  }
  report("propagate / compute_activities / tighten_bounds on the acceptance stream",
         bad == 0 && acts_bad == 0 && tight_bad == 0,
         "1000 instances x {incremental, full}: " + std::to_string(bad) + " propagate, " +
             std::to_string(acts_bad) + " activity, " + std::to_string(tight_bad) + " tightening mismatches");
}

void propagation_mixed()
{
  int bad = 0, runs = 0;
  for (uint64_t s = 0; s < 24; ++s) {
    const bool heavy   = s % 4 == 3;
    const ProblemDef p = mixed_instance(1000 + s, 3000, 3000, heavy ? 3 : 0, 20000);
    for (double thr : {1e-7, 0.0}) {
      PropagationLimits lim;
      lim.abs_threshold = thr;
      lim.rel_threshold = thr == 0.0 ? 0.0 : 1e-4;
      BoundsState a(p), g(p);
      const auto ra = propagate(p, a, lim);
      const auto rg = pg::propagate(p, g, lim);
      ++runs;
      if (!same_result(ra, rg) || !same_state(a, g)) ++bad;
    }
  }
  report("propagate on mixed fractional instances (incl. rows > 16384 nnz)", bad == 0,
         std::to_string(runs) + " runs, " + std::to_string(bad) + " mismatches");
}

void probing_stream()
{
  std::mt19937_64 rng(7771);  // acceptance.cpp:89
  int bad_cache = 0, bad_probe = 0, bad_prio = 0;
  for (int t = 0; t < 200; ++t) {
    const ProblemDef p = testkit::random_instance(rng);
    const auto ca      = build_cache(p, 1e9);
    const auto cg      = pg::build_cache(p, 1e9);
    if (!same_cache(ca, cg)) ++bad_cache;
    if (prioritize_probe_vars(p) != pg::prioritize_probe_vars(p)) ++bad_prio;
    BoundsState root(p);
    propagate(p, root);  // a propagated root too (certified-fixpoint path of the batched kernel)
    if (root.infeasible()) continue;
    for (int v = 0; v < p.n_vars; ++v)
      if (!same_entry(probe_variable(p, root, v), pg::probe_variable(p, root, v))) ++bad_probe;
  }
  report("build_cache / probe_variable / prioritize_probe_vars on the probing stream",
         bad_cache == 0 && bad_probe == 0 && bad_prio == 0,
         "200 instances: " + std::to_string(bad_cache) + " cache, " + std::to_string(bad_probe) +
             " entry, " + std::to_string(bad_prio) + " priority mismatches");
}

void warm_start_and_pairs()
{
  std::mt19937_64 rng(4242);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  int bad_ws = 0, bad_pp = 0, cases = 0;
  for (int t = 0; t < 150; ++t) {
    const ProblemDef p = testkit::random_instance(rng);
    const auto cache   = build_cache(p, 1e9);
    const WorkPlan plan = build_work_plan(p);
    std::vector<int> vars;
    std::vector<double> v0, v1;
    std::vector<std::pair<int, double>> asg;
    for (int i = 0; i < p.n_vars; ++i) {
      if (U(rng) < 0.4) continue;
      const double lo = p.var_lower[i], up = p.var_upper[i];
      const double a = std::floor(lo + (up - lo + 1) * U(rng)), b = std::floor(lo + (up - lo + 1) * U(rng));
      vars.push_back(i);
      v0.push_back(std::min(a, up));
      v1.push_back(std::min(b, up));
      asg.push_back({i, v0.back()});
    }
    const auto wa = assemble_bulk_warm_start(cache, asg);
    const auto wg = pg::assemble_bulk_warm_start(cache, asg);
    if (!same_state(wa.bounds, wg.bounds) || wa.conflicts != wg.conflicts || wa.evicted != wg.evicted) ++bad_ws;
    BoundsState base(p);
    for (int use_cache = 0; use_cache < 2; ++use_cache) {
      const ProbingCache* c = use_cache ? &cache : nullptr;
      const auto ra = parallel_propagate(p, base, vars, v0, v1, c, plan);
      const auto rg = pg::parallel_propagate(p, base, vars, v0, v1, c, plan);
      ++cases;
      for (int q = 0; q < 2; ++q) {
        const auto& x = ra.probe[q];
        const auto& y = rg.probe[q];
        if (!same_state(x.bounds, y.bounds) || x.infeas_count != y.infeas_count || x.evicted != y.evicted ||
            x.fixed != y.fixed)
          ++bad_pp;
      }
    }
  }
  report("assemble_bulk_warm_start / parallel_propagate", bad_ws == 0 && bad_pp == 0,
         std::to_string(cases) + " paired probes: " + std::to_string(bad_ws) + " warm-start, " +
             std::to_string(bad_pp) + " probe mismatches");
}

void rounding_stream()
{
  std::mt19937_64 gen(99);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  int bad = 0, runs = 0;
  for (int t = 0; t < 200; ++t) {
    testkit::RandomInstanceOptions opt;
    opt.force_feasible = t % 2 == 0;
    const ProblemDef p = testkit::random_instance(gen, opt);
    SolutionVector s;
    for (int i = 0; i < p.n_vars; ++i) s.values.push_back(p.var_lower[i] + (p.var_upper[i] - p.var_lower[i]) * U(gen));
    const auto cache = build_cache(p, 1e9);
    for (int use_cache = 0; use_cache < 2; ++use_cache) {
      Rng ra(1000 + t), rg(1000 + t);
      const ProbingCache* c = use_cache ? &cache : nullptr;
      const auto oa = propagation_round(p, s, c, Deadline::never(), ra);
      const auto og = pg::propagation_round(p, s, c, Deadline::never(), rg);
      ++runs;
      const bool same = oa.rounding_infeasible == og.rounding_infeasible && oa.timed_out == og.timed_out &&
                        oa.completed == og.completed && oa.bulks_committed == og.bulks_committed &&
                        oa.set_count == og.set_count && same_bits(oa.point.values, og.point.values) &&
                        ra == rg;  // the caller's generator advanced identically
      if (!same) ++bad;
    }
  }
  report("propagation_round (with and without cache; caller Rng state)", bad == 0,
         std::to_string(runs) + " runs, " + std::to_string(bad) + " mismatches");
}

void rounding_mixed()
{
  int bad = 0, runs = 0;
  for (uint64_t s = 0; s < 4; ++s) {
    const ProblemDef p = mixed_instance(500 + s, 2000, 1500, 0, 0);
    std::mt19937_64 g(s);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    SolutionVector sv;
    for (int i = 0; i < p.n_vars; ++i) sv.values.push_back(p.var_upper[i] * U(g));
    const auto cache = pg::build_cache(p, 1e9);
    Rng ra(s), rg(s);
    const auto oa = propagation_round(p, sv, &cache, Deadline::never(), ra);
    const auto og = pg::propagation_round(p, sv, &cache, Deadline::never(), rg);
    ++runs;
    // continuous values come from the reference's own lp_polish (PDHG, wall-clock budgeted):
    // compare integer variables bitwise, plus every flag and counter
    bool same = oa.rounding_infeasible == og.rounding_infeasible && oa.completed == og.completed &&
                oa.bulks_committed == og.bulks_committed && oa.set_count == og.set_count && ra == rg;
    for (int i = 0; i < p.n_vars && same; ++i)
      if (p.is_integer[i] && std::memcmp(&oa.point.values[i], &og.point.values[i], 8)) same = false;
    if (!same) ++bad;
  }
  report("propagation_round on mixed 2000-var instances with a GPU-built cache", bad == 0,
         std::to_string(runs) + " runs, " + std::to_string(bad) + " mismatches");
}

void repair_stream()
{
  std::mt19937_64 gen(2718);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  int bad = 0, runs = 0, present = 0, rounds_bad = 0, rounds = 0;
  for (int t = 0; t < 200; ++t) {
    const ProblemDef p = testkit::random_instance(gen, {});
    std::vector<std::pair<int, double>> fixed;
    for (int i = 0; i < p.n_vars; ++i)
      if (p.is_integer[i] && U(gen) < 0.8)
        fixed.push_back({i, std::min(p.var_upper[i], std::floor(p.var_lower[i] +
                                                                (p.var_upper[i] - p.var_lower[i] + 1) * U(gen)))});
    RoundingConfig cfg;
    const WorkPlan plan = build_work_plan(p);
    const auto ra       = repair(p, fixed, Deadline::never(), cfg, plan);
    const auto rg       = pg::repair(p, fixed, Deadline::never(), cfg, plan);
    ++runs;
    bool same = ra.has_value() == rg.has_value();
    if (same && ra) {
      ++present;
      same = ra->values == rg->values && same_state(ra->bounds, rg->bounds);
    }
    if (!same) ++bad;
    // propagation_round with repair enabled (rounding.hpp:492-504)
    SolutionVector s;
    for (int i = 0; i < p.n_vars; ++i) s.values.push_back(p.var_lower[i] + (p.var_upper[i] - p.var_lower[i]) * U(gen));
    RoundingConfig rc;
    rc.repair_enabled = true;
    Rng a(t), g(t);
    const auto oa = propagation_round(p, s, nullptr, Deadline::never(), a, rc);
    const auto og = pg::propagation_round(p, s, nullptr, Deadline::never(), g, rc);
    ++rounds;
    if (!(oa.rounding_infeasible == og.rounding_infeasible && oa.completed == og.completed &&
          oa.repair_attempts == og.repair_attempts && oa.bulks_committed == og.bulks_committed &&
          oa.set_count == og.set_count && same_bits(oa.point.values, og.point.values) && a == g))
      ++rounds_bad;
  }
  report("repair + propagation_round with repair enabled", bad == 0 && rounds_bad == 0,
         std::to_string(runs) + " repairs (" + std::to_string(present) + " present), " +
             std::to_string(bad) + " mismatches; " + std::to_string(rounds) + " rounding runs, " +
             std::to_string(rounds_bad) + " mismatches");
}

void builder_stream()
{
  std::mt19937_64 gen(4711);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  int bad = 0, runs = 0, threw = 0;
  for (int t = 0; t < 300; ++t) {
    const int n = 1 + (int)(40 * U(gen)), m = 1 + (int)(30 * U(gen)), ne = (int)(300 * U(gen));
    pulse::ProblemBuilder a;
    pg::ProblemBuilder g;
    for (int i = 0; i < n; ++i) {
      double lo = std::floor(6 * U(gen)) - 3 + (U(gen) < 0.5 ? 0.3 : 0.0);
      double up = lo + std::floor(5 * U(gen)) + 0.6;
      if (U(gen) < 0.1) lo = -kInf;
      if (U(gen) < 0.1) up = kInf;
      const bool integer = U(gen) < 0.7;
      a.add_var("x" + std::to_string(i), lo, up, integer, U(gen));
      g.add_var("x" + std::to_string(i), lo, up, integer, 0.0);
      g.set_objective(i, 0.0);
    }
    for (int k = 0; k < m; ++k) {
      const double lo = U(gen) < 0.5 ? -kInf : -5.0, up = U(gen) < 0.5 ? kInf : 5.0;
      a.add_row("c" + std::to_string(k), lo, up);
      g.add_row("c" + std::to_string(k), lo, up);
    }
    for (int e = 0; e < ne; ++e) {
      // integer-valued entries: any number of duplicates sums identically in any order
      const int r = (int)(m * U(gen)) % m, c = (int)(n * U(gen)) % n;
      const double v = std::floor(7 * U(gen)) - 3;
      a.add_entry(r, c, v);
      g.add_entry(r, c, v);
    }
    ++runs;
    std::string ea, eg;
    ProblemDef pa, pgd;
    try {
      pa = a.build();
    } catch (const std::exception& x) {
      ea = x.what();
    }
    try {
      pgd = g.build();
    } catch (const std::exception& x) {
      eg = x.what();
    }
    if (!ea.empty() || !eg.empty()) {
      ++threw;
      if (ea != eg) ++bad;
      continue;
    }
    const bool same = pa.row_start == pgd.row_start && pa.row_col == pgd.row_col &&
                      pa.col_start == pgd.col_start && pa.col_row == pgd.col_row &&
                      same_bits(pa.row_val, pgd.row_val) && same_bits(pa.col_val, pgd.col_val) &&
                      same_bits(pa.var_lower, pgd.var_lower) && same_bits(pa.var_upper, pgd.var_upper) &&
                      pa.is_integer == pgd.is_integer && pa.var_names == pgd.var_names &&
                      pa.cons_names == pgd.cons_names;
    if (!same) ++bad;
  }
  report("ProblemBuilder::build on the device (random builders, duplicates, zeros, errors)", bad == 0,
         std::to_string(runs) + " builds (" + std::to_string(threw) + " threw), " + std::to_string(bad) +
             " mismatches");
}

void lp_products()
{
  int bad = 0, runs = 0;
  for (uint64_t sd = 0; sd < 3; ++sd) {
    const ProblemDef p = mixed_instance(700 + sd, sd == 2 ? 40000 : 3000, 2500, sd == 2 ? 2 : 0, 20000);
    const LpInstance s = LpInstance::relax(p);
    std::mt19937_64 g(sd);
    std::normal_distribution<double> N01(0.0, 1.0);
    std::vector<double> x(s.n_vars), y(s.n_rows), ra(s.n_rows), rc(s.n_vars), ga, gc;
    for (auto& v : x) v = N01(g);
    for (auto& v : y) v = N01(g);
    lpdetail::spmv_rows(s, x, ra);
    lpdetail::spmv_cols(s, y, rc);
    pg::LpProducts dev(s);
    dev.spmv_rows(x, ga);
    dev.spmv_cols(y, gc);
    ++runs;
    if (!same_bits(ra, ga) || !same_bits(rc, gc)) ++bad;
    // evaluate_kkt: maxima bitwise, objective-based fields within 1e-12 relative
    LpInstance sk = s;
    sk.obj.resize(sk.n_vars);
    for (auto& c : sk.obj) c = N01(g);
    std::vector<double> xk(sk.n_vars), yk(sk.n_rows), axk(sk.n_rows), atyk(sk.n_vars);
    for (int i = 0; i < sk.n_vars; ++i) xk[i] = clamp(3 * N01(g), sk.var_lower[i], sk.var_upper[i]);
    for (auto& v : yk) v = N01(g);
    const auto kr = lpdetail::evaluate_kkt(sk, xk, yk, axk, atyk);
    const auto kg = pg::LpProducts(sk).evaluate_kkt(xk, yk);
    auto near = [](double a, double b) { return std::abs(a - b) <= 1e-12 * std::max(1.0, std::abs(b)); };
    if (kr.primal_res != kg.primal_res || kr.dual_res != kg.dual_res || kr.x_norm != kg.x_norm ||
        !near(kg.primal_obj, kr.primal_obj) || !near(kg.dual_obj, kr.dual_obj) ||
        !near(kg.gap, kr.gap) || !near(kg.score, kr.score))
      ++bad;
  }
  report("lpdetail::spmv_rows / spmv_cols / evaluate_kkt (PDHG, incl. rows > 16384 entries)", bad == 0,
         std::to_string(runs) + " instances, " + std::to_string(bad) + " mismatches");
}

// Host overhead of the drop-in per call: what pulse::gpu::propagate adds to the
// C-ABI call bp_propagate on the same device problem and host bounds -- the side-table lookup (key
// sample + match) and the marshalling (none: it works in place on the BoundsState). Measured
// directly (the lookup, 10^4 calls) and end to end as the median of paired per-call differences
// (pg::propagate vs bp_propagate alternating on the same host buffer, which cancels the GPU's own
// run-to-run variation; the estimate is the mean of the two call orders' medians); both must stay
// <= 50 us, on a 10k x 10k and a 300k x 300k instance (heavy rows).
void host_overhead()
{
  bool ok = true;
  std::string detail;
  for (const auto& [n, heavy] : {std::pair<int, int>{10000, 0}, std::pair<int, int>{300000, 8}}) {
    const ProblemDef p = mixed_instance(77 + n, n, n, heavy, 40000);
    bp_problem* h      = pg::detail::handle(p);
    const int reps     = n > 100000 ? 40 : 100;
    BoundsState warm(p);
    pg::propagate(p, warm);  // upload + warm-up
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us  = [](auto a, auto b) { return 1e6 * std::chrono::duration<double>(b - a).count(); };
    const auto l0 = now();
    for (int r = 0; r < 10000; ++r) pg::detail::handle(p);
    const double lookup_us = us(l0, now()) / 10000;
    const bp_limits l = pg::detail::limits(PropagationLimits{});
    std::vector<double> diff[2];  // [0]: bp_propagate first, [1]: pulse::gpu::propagate first
    double t_abi = 0.0, t_pg = 0.0;
    // both calls work on the SAME host buffer (b's storage), reset to the root bounds before each
    // call outside the timed region: the pair then differs only by the wrapper, not by which
    // pageable buffer the copies go through
    const std::vector<double> root = BoundsState(p).raw();
    BoundsState b(p);
    double* hb  = const_cast<double*>(b.raw().data());
    auto reset  = [&] { std::copy(root.begin(), root.end(), hb); };
    for (int r = 0; r < reps; ++r) {
      int32_t inf = 0;
      bp_result res{};
      double da, dp;
      auto abi = [&] {
        reset();
        const auto t0 = now();
        pg::detail::check(bp_propagate(h, hb, &inf, &l, &res));
        return us(t0, now());
      };
      auto wrapped = [&] {
        reset();
        const auto t0 = now();
        pg::propagate(p, b);
        return us(t0, now());
      };
      if (r % 2 == 0) {
        da = abi();
        dp = wrapped();
      } else {
        dp = wrapped();
        da = abi();
      }
      t_abi += da;
      t_pg += dp;
      diff[r % 2].push_back(dp - da);
    }
    for (auto& d : diff) std::sort(d.begin(), d.end());
    const double med = 0.5 * (diff[0][diff[0].size() / 2] + diff[1][diff[1].size() / 2]);
    ok = ok && lookup_us <= 50.0 && med <= 50.0;
    char buf[320];
    std::snprintf(buf, sizeof(buf),
                  "%s%dx%d: side-table lookup %.2f us; bp_propagate %.1f us, pulse::gpu::propagate %.1f us, "
                  "paired difference %.1f us (medians by call order %.1f / %.1f us)",
                  detail.empty() ? "" : "; ", n, n, lookup_us, t_abi / reps, t_pg / reps, med,
                  diff[0][diff[0].size() / 2], diff[1][diff[1].size() / 2]);
    detail += buf;
  }
  report("drop-in host overhead per propagate <= 50 us", ok, detail);
}

// pulse::gpu::build_cache over every GPU (bp_build_cache_multi: NCCL gather to device 0) equals the
// reference's build_cache(p, 1e9) (probing.hpp:243) entry for entry.
void build_cache_multi()
{
  int32_t ndev = 0;
  bp_device_count(&ndev);
  std::vector<int> devs;
  for (int d = 0; d < ndev; ++d) devs.push_back(d);
  int bad = 0, vars = 0;
  for (uint64_t s = 0; s < 3; ++s) {
    const ProblemDef p   = mixed_instance(500 + s, 1500, 1200, s == 2 ? 2 : 0, 3000);
    const ProbingCache a = build_cache(p, 1e9);
    const ProbingCache g = pg::build_cache(p, 1e9, devs);
    if (a.n_probed != g.n_probed || a.n_infeasible_branches != g.n_infeasible_branches) ++bad;
    for (int v = 0; v < p.n_vars; ++v) {
      if (a.has(v) != g.has(v)) {
        ++bad;
        continue;
      }
      if (!a.has(v)) continue;
      ++vars;
      const auto& x = a.at(v);
      const auto& y = g.at(v);
      if (x.kind != y.kind || x.forces_down != y.forces_down || x.forces_up != y.forces_up ||
          !same_branch(x.down, y.down) || !same_branch(x.up, y.up))
        ++bad;
    }
  }
  report("build_cache over " + std::to_string(devs.size()) + " GPU(s) (NCCL gather) == reference build_cache",
         bad == 0, std::to_string(vars) + " entries, " + std::to_string(bad) + " mismatches");
}

void errors()
{
  const ProblemDef p = testkit::tiny_knapsack();
  BoundsState b(p);
  bool oor = false;
  try {
    pg::probe_variable(p, b, 7);
  } catch (const std::out_of_range&) {
    oor = true;
  }
  BoundsState inf(p);
  inf.mark_infeasible();
  const auto r = pg::propagate(p, inf);
  report("error taxonomy and infeasible short-circuit",
         oor && r.status == PropagationStatus::Infeasible && r.rounds == 0, "out_of_range, Infeasible/0 rounds");
}

}  // namespace

int main()
{
  int32_t ndev = 0;
  if (bp_device_count(&ndev) != BP_OK || ndev == 0) {
    std::printf("FAIL  no CUDA device (%s)\n", bp_last_error());
    return 1;
  }
  // DROPIN_ONLY=<criterion name> runs one criterion (debugging)
  const char* only = std::getenv("DROPIN_ONLY");
  auto want = [&](const char* name) { return !only || std::strcmp(only, name) == 0; };
  if (want("errors")) errors();
  if (want("propagation_stream")) propagation_stream();
  if (want("propagation_mixed")) propagation_mixed();
  if (want("probing_stream")) probing_stream();
  if (want("warm_start_and_pairs")) warm_start_and_pairs();
  if (want("rounding_stream")) rounding_stream();
  if (want("rounding_mixed")) rounding_mixed();
  if (want("repair_stream")) repair_stream();
  if (want("builder_stream")) builder_stream();
  if (want("lp_products")) lp_products();
  if (want("host_overhead")) host_overhead();
  if (want("build_cache_multi")) build_cache_multi();
  std::printf("%d failure(s)\n", g_failures);
  return g_failures;
}
