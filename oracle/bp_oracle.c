/* TEST INFRASTRUCTURE ONLY — plain-C restatement ("port") of the reference bound-propagation
 * hot path. Each function cites the reference file:line it restates
 * (/root/reference/proj/include/pulse/...). Sequential (the reference's results are independent
 * of its thread count, parallel.hpp:98-101). Compiled with -ffp-contract=off: products and sums
 * are separately rounded exactly like the reference Release build.
 *
 * Semantics notes carried over verbatim from the reference:
 *  - std::max(a,b) == (a < b ? b : a), std::min(a,b) == (b < a ? b : a): the FIRST operand is kept
 *    on ties, which decides the sign of tied zeros. We never use fmax/fmin.
 *  - activities are sequential sums inside fixed kSumSegment=16384 segments, segments summed in
 *    order (problem.hpp:274, propagation.hpp:177-193).
 */
#include "bp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define K_SUM_SEGMENT 16384 /* problem.hpp:274 */
#define K_INT_EPS 1e-6      /* common.hpp:24 */

static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline int is_fin(double v) { return isfinite(v); }

void orc_default_limits(orc_limits* lim)
{ /* propagation.hpp:253-259 */
  lim->max_rounds    = 64;
  lim->abs_threshold = 1e-7;
  lim->rel_threshold = 1e-4;
  lim->incremental   = 1;
}

/* propagation.hpp:153-172 activity_segment + :177-193 row_activity */
static void row_activity(const orc_problem* p, const double* b, int k, double* act, int* nmin,
                         int* nmax)
{
  const int s0 = p->row_start[k], n = p->row_start[k + 1] - s0;
  double min_total = 0.0, max_total = 0.0;
  int inf_min = 0, inf_max = 0;
  for (int s = 0; s < n; s += K_SUM_SEGMENT) {
    const int hi = (n < s + K_SUM_SEGMENT) ? n : s + K_SUM_SEGMENT;
    double min_part = 0.0, max_part = 0.0;
    int pmin = 0, pmax = 0;
    for (int e = s; e < hi; ++e) {
      const double a  = p->row_val[s0 + e];
      const int c     = p->row_col[s0 + e];
      const double lo = b[2 * c], up = b[2 * c + 1];
      if (a > 0.0) {
        if (lo == -INFINITY) ++pmin; else min_part += a * lo;
        if (up == INFINITY) ++pmax; else max_part += a * up;
      } else {
        if (up == INFINITY) ++pmin; else min_part += a * up;
        if (lo == -INFINITY) ++pmax; else max_part += a * lo;
      }
    }
    min_total += min_part;
    max_total += max_part;
    inf_min += pmin;
    inf_max += pmax;
  }
  act[2 * k]     = min_total;
  act[2 * k + 1] = max_total;
  nmin[k]        = inf_min;
  nmax[k]        = inf_max;
}

/* propagation.hpp:226-251 (binned and unbinned paths give identical bits) */
void orc_compute_activities(const orc_problem* p, const double* b, const int* rows, int nrows,
                            double* act, int* ninf_min, int* ninf_max)
{
  if (nrows >= 0) {
    for (int j = 0; j < nrows; ++j) row_activity(p, b, rows[j], act, ninf_min, ninf_max);
  } else {
    for (int k = 0; k < p->n_cons; ++k) row_activity(p, b, k, act, ninf_min, ninf_max);
  }
}

/* propagation.hpp:273-282 */
static int counts_as_change(double improvement, int integer, double width, const orc_limits* lim)
{
  if (improvement <= 0.0) return 0;
  if (improvement == INFINITY) return 1;
  if (integer) return improvement >= 1.0 - 1e-9;
  double thr = lim->abs_threshold;
  if (is_fin(width)) thr = smax(thr, lim->rel_threshold * width);
  return improvement > thr;
}

/* propagation.hpp:286-370 */
int orc_tighten_variable(const orc_problem* p, double* b, const double* act, const int* ninf_min,
                         const int* ninf_max, int i, const orc_limits* lim)
{
  const double lo = b[2 * i], up = b[2 * i + 1];
  double new_lo = lo, new_up = up;
  const int integer = p->is_integer[i] != 0;
  for (int e = p->col_start[i]; e < p->col_start[i + 1]; ++e) {
    const int k    = p->col_row[e];
    const double a = p->col_val[e];
    const double g = p->cons_upper[k];
    if (is_fin(g)) { /* :301-325 */
      const int my_inf = (a > 0.0) ? (lo == -INFINITY) : (up == INFINITY);
      const int n_inf  = ninf_min[k];
      double rest = 0.0;
      int usable  = 0;
      if (n_inf == 0) {
        rest   = act[2 * k] - (a > 0.0 ? a * lo : a * up);
        usable = 1;
      } else if (n_inf == 1 && my_inf) {
        rest   = act[2 * k];
        usable = 1;
      }
      if (usable) {
        const double cand = (g - rest) / a;
        if (a > 0.0) new_up = smin(new_up, integer ? floor(cand + K_INT_EPS) : cand);
        else new_lo = smax(new_lo, integer ? ceil(cand - K_INT_EPS) : cand);
      }
    }
    const double h = p->cons_lower[k];
    if (is_fin(h)) { /* :327-351 */
      const int my_inf = (a > 0.0) ? (up == INFINITY) : (lo == -INFINITY);
      const int n_inf  = ninf_max[k];
      double rest = 0.0;
      int usable  = 0;
      if (n_inf == 0) {
        rest   = act[2 * k + 1] - (a > 0.0 ? a * up : a * lo);
        usable = 1;
      } else if (n_inf == 1 && my_inf) {
        rest   = act[2 * k + 1];
        usable = 1;
      }
      if (usable) {
        const double cand = (h - rest) / a;
        if (a > 0.0) new_lo = smax(new_lo, integer ? ceil(cand - K_INT_EPS) : cand);
        else new_up = smin(new_up, integer ? floor(cand + K_INT_EPS) : cand);
      }
    }
  }
  if (new_lo > new_up + 1e-9) return -1; /* :354 */
  if (new_lo > new_up) new_lo = new_up;  /* :355 */
  const double width = up - lo;
  int changed        = 0;
  const double lo_imp = (lo == -INFINITY && new_lo > -INFINITY) ? INFINITY : new_lo - lo;
  if (counts_as_change(lo_imp, integer, width, lim)) {
    b[2 * i] = new_lo;
    changed  = 1;
  }
  const double up_imp = (up == INFINITY && new_up < INFINITY) ? INFINITY : up - new_up;
  if (counts_as_change(up_imp, integer, width, lim)) {
    b[2 * i + 1] = new_up;
    changed      = 1;
  }
  return changed;
}

/* propagation.hpp:378-412. Jacobi: every var reads activities computed before the sweep and
 * writes only its own slots, so a sequential sweep equals the parallel one. */
int orc_tighten_bounds(const orc_problem* p, double* b, int* infeasible, const double* act,
                       const int* ninf_min, const int* ninf_max, const int* vars, int nvars,
                       const orc_limits* lim, int* changed, int* crossed)
{
  signed char* result = (signed char*)calloc((size_t)p->n_vars + 1, 1);
  if (nvars >= 0) {
    for (int j = 0; j < nvars; ++j)
      result[vars[j]] = (signed char)orc_tighten_variable(p, b, act, ninf_min, ninf_max, vars[j], lim);
  } else {
    for (int i = 0; i < p->n_vars; ++i)
      result[i] = (signed char)orc_tighten_variable(p, b, act, ninf_min, ninf_max, i, lim);
  }
  int nch = 0, ncr = 0;
  for (int i = 0; i < p->n_vars; ++i) {
    if (result[i] > 0) changed[nch++] = i;
    if (result[i] < 0) ++ncr;
  }
  if (ncr > 0) *infeasible = 1;
  if (crossed) *crossed = ncr;
  free(result);
  return nch;
}

static int cmp_int(const void* a, const void* b)
{
  const int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* propagation.hpp:418-486 (time limit infinite). */
void orc_propagate(const orc_problem* p, double* b, int* infeasible, const orc_limits* lim,
                   int* out3)
{
  out3[0] = ORC_UNCHANGED;
  out3[1] = 0;
  out3[2] = 0;
  if (*infeasible) {
    out3[0] = ORC_INFEASIBLE;
    return;
  }
  const int n = p->n_vars, m = p->n_cons;
  double* act    = (double*)calloc(2 * (size_t)m + 1, sizeof(double));
  int* nmin      = (int*)calloc((size_t)m + 1, sizeof(int));
  int* nmax      = (int*)calloc((size_t)m + 1, sizeof(int));
  int* drows     = (int*)malloc(((size_t)m + 1) * sizeof(int));
  int* dvars     = (int*)malloc(((size_t)n + 1) * sizeof(int));
  int* changed   = (int*)malloc(((size_t)n + 1) * sizeof(int));
  char* row_mark = (char*)calloc((size_t)m + 1, 1);
  char* var_mark = (char*)calloc((size_t)n + 1, 1);
  int ndr = 0, ndv = 0, first = 1, any_change = 0;
  while (out3[1] < lim->max_rounds) {
    ++out3[1];
    const int full = first || !lim->incremental;
    orc_compute_activities(p, b, drows, full ? -1 : ndr, act, nmin, nmax);
    int crossed = 0;
    const int nch = orc_tighten_bounds(p, b, infeasible, act, nmin, nmax, dvars, full ? -1 : ndv,
                                       lim, changed, &crossed);
    if (*infeasible) {
      out3[0] = ORC_INFEASIBLE;
      out3[2] = crossed;
      goto done;
    }
    if (nch == 0) break;
    any_change = 1;
    memset(row_mark, 0, (size_t)m);
    memset(var_mark, 0, (size_t)n);
    ndr = ndv = 0;
    for (int j = 0; j < nch; ++j) {
      const int i = changed[j];
      for (int e = p->col_start[i]; e < p->col_start[i + 1]; ++e) {
        const int k = p->col_row[e];
        if (!row_mark[k]) {
          row_mark[k]  = 1;
          drows[ndr++] = k;
        }
      }
    }
    qsort(drows, (size_t)ndr, sizeof(int), cmp_int);
    for (int j = 0; j < ndr; ++j) {
      const int k = drows[j];
      for (int e = p->row_start[k]; e < p->row_start[k + 1]; ++e) {
        const int i = p->row_col[e];
        if (!var_mark[i]) {
          var_mark[i]  = 1;
          dvars[ndv++] = i;
        }
      }
    }
    qsort(dvars, (size_t)ndv, sizeof(int), cmp_int);
    first = 0;
    if (ndr == 0) break;
  }
  out3[0] = any_change ? ORC_TIGHTENED : ORC_UNCHANGED;
done:
  free(act); free(nmin); free(nmax); free(drows); free(dvars); free(changed);
  free(row_mark); free(var_mark);
}

/* probing.hpp:30-60 */
int orc_make_branch_spec(double lo, double up, double* s)
{
  if (lo == up) return 0;
  if (is_fin(lo) && is_fin(up)) {
    const double mid = ceil((lo + up) / 2.0);
    s[0] = lo; s[1] = mid - 1.0; s[2] = mid; s[3] = up;
    return 1;
  }
  if (is_fin(lo)) {
    s[0] = lo; s[1] = lo; s[2] = lo + 1.0; s[3] = up;
    return 2;
  }
  if (is_fin(up)) {
    s[0] = lo; s[1] = up - 1.0; s[2] = up; s[3] = up;
    return 3;
  }
  return 0;
}

/* probing.hpp:194-219 probe_branch */
static void probe_branch(const orc_problem* p, const double* root, int v, double blo, double bup,
                         double* scratch, int* feasible, int* nd, int* dvar, double* dlo,
                         double* dup)
{
  const int n = p->n_vars;
  memcpy(scratch, root, sizeof(double) * 2 * (size_t)n);
  scratch[2 * v]     = smax(root[2 * v], blo);
  scratch[2 * v + 1] = smin(root[2 * v + 1], bup);
  *nd = 0;
  if (scratch[2 * v] > scratch[2 * v + 1]) {
    *feasible = 0;
    return;
  }
  orc_limits lim;
  orc_default_limits(&lim);
  int inf = 0, out3[3];
  orc_propagate(p, scratch, &inf, &lim, out3);
  if (out3[0] == ORC_INFEASIBLE) {
    *feasible = 0;
    return;
  }
  *feasible = 1;
  for (int i = 0; i < n; ++i) {
    if (scratch[2 * i] != root[2 * i] || scratch[2 * i + 1] != root[2 * i + 1]) {
      dvar[*nd] = i;
      dlo[*nd]  = scratch[2 * i];
      dup[*nd]  = scratch[2 * i + 1];
      ++*nd;
    }
  }
}

/* probing.hpp:225-238 probe_variable */
int orc_probe_variable(const orc_problem* p, const double* root, int v, int* feasible,
                       int* ndeltas, int* dvar, double* dlo, double* dup)
{
  double spec[4];
  const int kind = orc_make_branch_spec(root[2 * v], root[2 * v + 1], spec);
  feasible[0] = feasible[1] = 1;
  ndeltas[0] = ndeltas[1] = 0;
  if (!kind) return 0;
  const size_t n = (size_t)p->n_vars;
  double* scratch = (double*)malloc(sizeof(double) * 2 * (n + 1));
  probe_branch(p, root, v, spec[0], spec[1], scratch, &feasible[0], &ndeltas[0], dvar, dlo, dup);
  probe_branch(p, root, v, spec[2], spec[3], scratch, &feasible[1], &ndeltas[1], dvar + n, dlo + n,
               dup + n);
  free(scratch);
  return kind;
}

/* probing.hpp:292-352 assemble_bulk_warm_start */
int orc_assemble_bulk_warm_start(const orc_cache* c, const int* vars, const double* vals,
                                 int nassign, double* bounds, int* conflicts, int* evicted,
                                 int* n_evicted)
{
  const int n = c->n_vars;
  memcpy(bounds, c->root, sizeof(double) * 2 * (size_t)n);
  int* last_writer = (int*)malloc(sizeof(int) * ((size_t)n + 1));
  char* ev_mark    = (char*)calloc((size_t)n + 1, 1);
  for (int i = 0; i < n; ++i) last_writer[i] = -1;
  /* undo log sized by the largest branch */
  int* u_var = NULL; double* u_lo = NULL; double* u_up = NULL; int* u_w = NULL;
  long long u_cap = 0;
  int ncf = 0;
  *n_evicted = 0;
  for (int j = 0; j < nassign; ++j) {
    const int v = vars[j];
    const int e = c->entry_of[v];
    if (e < 0) continue;
    const int side = (vals[j] <= c->e_branch[4 * e + 1]) ? 0 : 1; /* :304 value <= down.upper */
    if (!c->e_feas[2 * e + side]) {
      conflicts[2 * ncf] = v; conflicts[2 * ncf + 1] = v; ++ncf;
      if (!ev_mark[v]) { ev_mark[v] = 1; evicted[(*n_evicted)++] = v; }
      continue;
    }
    const long long d0 = c->d_off[2 * e + side], d1 = c->d_off[2 * e + side + 1];
    if (d1 - d0 > u_cap) {
      u_cap = d1 - d0;
      u_var = (int*)realloc(u_var, sizeof(int) * (size_t)u_cap);
      u_lo  = (double*)realloc(u_lo, sizeof(double) * (size_t)u_cap);
      u_up  = (double*)realloc(u_up, sizeof(double) * (size_t)u_cap);
      u_w   = (int*)realloc(u_w, sizeof(int) * (size_t)u_cap);
    }
    int nu = 0, conflict = 0, conflicting = -1;
    for (long long d = d0; d < d1; ++d) {
      const int dv    = c->d_var[d];
      const double nl = smax(bounds[2 * dv], c->d_lo[d]);
      const double nu_ = smin(bounds[2 * dv + 1], c->d_up[d]);
      if (nl > nu_ + 1e-9) {
        conflict    = 1;
        conflicting = last_writer[dv] >= 0 ? last_writer[dv] : v;
        break;
      }
      if (nl != bounds[2 * dv] || nu_ != bounds[2 * dv + 1]) {
        u_var[nu] = dv; u_lo[nu] = bounds[2 * dv]; u_up[nu] = bounds[2 * dv + 1];
        u_w[nu] = last_writer[dv]; ++nu;
        bounds[2 * dv] = nl; bounds[2 * dv + 1] = nu_;
        last_writer[dv] = v;
      }
    }
    if (conflict) {
      for (int u = nu - 1; u >= 0; --u) {
        bounds[2 * u_var[u]] = u_lo[u]; bounds[2 * u_var[u] + 1] = u_up[u];
        last_writer[u_var[u]] = u_w[u];
      }
      conflicts[2 * ncf] = conflicting; conflicts[2 * ncf + 1] = v; ++ncf;
      if (!ev_mark[v]) { ev_mark[v] = 1; evicted[(*n_evicted)++] = v; }
    }
  }
  free(last_writer); free(ev_mark); free(u_var); free(u_lo); free(u_up); free(u_w);
  return ncf;
}

/* rounding.hpp:167-207 run_probe */
int orc_run_probe(const orc_problem* p, const double* base, int base_infeasible, const int* vars,
                  const double* values, int nvars, const orc_cache* c, double* out_bounds,
                  int* out_infeasible, int* evicted, int* n_evicted, int* fixed_vars,
                  double* fixed_vals, int* n_fixed)
{
  const int n = p->n_vars;
  memcpy(out_bounds, base, sizeof(double) * 2 * (size_t)n);
  *out_infeasible = base_infeasible;
  *n_evicted = 0;
  *n_fixed   = 0;
  char* ev_mark = (char*)calloc((size_t)n + 1, 1);
  if (c) {
    double* ws = (double*)malloc(sizeof(double) * 2 * ((size_t)n + 1));
    int* conf  = (int*)malloc(sizeof(int) * 2 * ((size_t)nvars + 1));
    orc_assemble_bulk_warm_start(c, vars, values, nvars, ws, conf, evicted, n_evicted);
    for (int j = 0; j < *n_evicted; ++j) ev_mark[evicted[j]] = 1;
    for (int i = 0; i < n; ++i) { /* propagation.hpp:49-56 meet */
      out_bounds[2 * i]     = smax(out_bounds[2 * i], ws[2 * i]);
      out_bounds[2 * i + 1] = smin(out_bounds[2 * i + 1], ws[2 * i + 1]);
      if (out_bounds[2 * i] > out_bounds[2 * i + 1]) *out_infeasible = 1;
    }
    free(ws); free(conf);
  }
  int crossings = *out_infeasible ? 1 : 0;
  for (int j = 0; j < nvars; ++j) {
    const int v = vars[j];
    if (ev_mark[v]) continue;
    const double val = values[j];
    if (val < out_bounds[2 * v] - 1e-9 || val > out_bounds[2 * v + 1] + 1e-9) {
      ++crossings;
      continue;
    }
    out_bounds[2 * v] = val; out_bounds[2 * v + 1] = val;
    fixed_vars[*n_fixed] = v; fixed_vals[*n_fixed] = val; ++*n_fixed;
  }
  free(ev_mark);
  if (crossings > 0) {
    *out_infeasible = 1;
    return crossings;
  }
  orc_limits lim;
  orc_default_limits(&lim);
  int out3[3];
  orc_propagate(p, out_bounds, out_infeasible, &lim, out3);
  if (out3[0] == ORC_INFEASIBLE) return out3[2] > 1 ? out3[2] : 1;
  return 0;
}

/* rounding.hpp:71-115 implied_slack_sort: S_i fold + stable ascending sort on (S, position). */
typedef struct { double key; int pos; } keyed_t;
static int cmp_keyed(const void* a, const void* b)
{
  const keyed_t* x = (const keyed_t*)a;
  const keyed_t* y = (const keyed_t*)b;
  if (x->key < y->key) return -1;
  if (y->key < x->key) return 1;
  return (x->pos > y->pos) - (x->pos < y->pos); /* stability */
}
void orc_implied_slack_sort(const orc_problem* p, const double* act, const int* ninf_min,
                            const int* ninf_max, int* vars, int nvars)
{
  keyed_t* kv = (keyed_t*)malloc(sizeof(keyed_t) * ((size_t)nvars + 1));
  for (int pos = 0; pos < nvars; ++pos) {
    const int i  = vars[pos];
    double total = 0.0;
    for (int e = p->col_start[i]; e < p->col_start[i + 1]; ++e) {
      const int k    = p->col_row[e];
      const double a = p->col_val[e];
      if (is_fin(p->cons_upper[k]) && ninf_min[k] == 0) {
        const double slack = p->cons_upper[k] - act[2 * k];
        if (slack <= 0.0) { total = INFINITY; break; }
        const double s = a / slack;
        total += s * s;
      }
      if (is_fin(p->cons_lower[k]) && ninf_max[k] == 0) {
        const double slack = act[2 * k + 1] - p->cons_lower[k];
        if (slack <= 0.0) { total = INFINITY; break; }
        const double s = a / slack;
        total += s * s;
      }
    }
    kv[pos].key = total;
    kv[pos].pos = pos;
  }
  qsort(kv, (size_t)nvars, sizeof(keyed_t), cmp_keyed);
  int* tmp = (int*)malloc(sizeof(int) * ((size_t)nvars + 1));
  for (int j = 0; j < nvars; ++j) tmp[j] = vars[kv[j].pos];
  memcpy(vars, tmp, sizeof(int) * (size_t)nvars);
  free(tmp); free(kv);
}
