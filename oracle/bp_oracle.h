/* TEST INFRASTRUCTURE ONLY — the plain-C restatement ("port") of the reference hot path, used by
 * tests/ and bench.py's cpu_baseline leg as a checker. Never linked into the product.
 * Pinned against the reference itself (oracle/_ref/libpulse_ref.so) and the committed golden
 * vectors in tests/golden/ (see tests/test_oracle.py). */
#ifndef BP_ORACLE_H
#define BP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int n_vars, n_cons;
  const int* row_start;  /* n_cons + 1 */
  const int* row_col;
  const double* row_val;
  const int* col_start;  /* n_vars + 1 */
  const int* col_row;
  const double* col_val;
  const double* var_lower;
  const double* var_upper;
  const uint8_t* is_integer;
  const double* cons_lower;
  const double* cons_upper;
} orc_problem;

typedef struct {
  int max_rounds;
  double abs_threshold;
  double rel_threshold;
  int incremental;
} orc_limits;

enum { ORC_TIGHTENED = 0, ORC_INFEASIBLE = 1, ORC_UNCHANGED = 2 };

void orc_default_limits(orc_limits* lim);

/* propagation.hpp:226 (subset when nrows >= 0; rows outside keep their values). */
void orc_compute_activities(const orc_problem* p, const double* b, const int* rows, int nrows,
                            double* act, int* ninf_min, int* ninf_max);
/* propagation.hpp:286 — returns 1 changed, 0 unchanged, -1 crossing. */
int orc_tighten_variable(const orc_problem* p, double* b, const double* act, const int* ninf_min,
                         const int* ninf_max, int i, const orc_limits* lim);
/* propagation.hpp:378 — returns #changed (ascending in `changed`); crossings set *infeasible. */
int orc_tighten_bounds(const orc_problem* p, double* b, int* infeasible, const double* act,
                       const int* ninf_min, const int* ninf_max, const int* vars, int nvars,
                       const orc_limits* lim, int* changed, int* crossed);
/* propagation.hpp:418 — out3 = {status, rounds, crossed}. time_limit is infinite here. */
void orc_propagate(const orc_problem* p, double* b, int* infeasible, const orc_limits* lim,
                   int* out3);

/* probing.hpp:30 — 0 = none, else kind + 1 (1 BoxedSplit, 2 AtLowerBound, 3 AtUpperBound). */
int orc_make_branch_spec(double lo, double up, double* spec4);

/* probing.hpp:194-238 for one variable from `root` (2n). For each branch s (0 down, 1 up):
 * feasible[s], ndeltas[s], and deltas (var, lo, up) written at dvar[s*n_vars ...].
 * Returns the spec code (0 = no entry probed). */
int orc_probe_variable(const orc_problem* p, const double* root, int v, int* feasible,
                       int* ndeltas, int* dvar, double* dlo, double* dup);

/* probing.hpp:292 over a flat cache: entry_off[v] = -1 (absent) or index e into per-entry
 * arrays: e_feas[2e+s], e_bu[4e..] = {dl, du, ul, uu}, deltas of branch s at
 * [d_off[2e+s], d_off[2e+s+1]) — requires d_off monotone per entry pair.
 * Writes bounds (starting from root); returns #conflicts; fills conflicts/evicted. */
typedef struct {
  int n_vars;
  const double* root;       /* 2n */
  const int* entry_of;      /* n: -1 or entry index */
  const int* e_feas;        /* 2 per entry */
  const double* e_branch;   /* 4 per entry: down lo, down up, up lo, up up */
  const int* e_force;       /* 2 per entry: forces_down, forces_up */
  const long long* d_off;   /* 2 per entry + 1: branch s of entry e is [d_off[2e+s], d_off[2e+s+1]) */
  const int* d_var;
  const double* d_lo;
  const double* d_up;
} orc_cache;

int orc_assemble_bulk_warm_start(const orc_cache* c, const int* vars, const double* vals,
                                 int nassign, double* bounds, int* conflicts, int* evicted,
                                 int* n_evicted);

/* rounding.hpp:167 run_probe. Returns infeas_count; bounds/infeasible written; evicted list and
 * fixed list (vars + values) with counts. cache may be NULL. */
int orc_run_probe(const orc_problem* p, const double* base, int base_infeasible, const int* vars,
                  const double* values, int nvars, const orc_cache* c, double* out_bounds,
                  int* out_infeasible, int* evicted, int* n_evicted, int* fixed_vars,
                  double* fixed_vals, int* n_fixed);

/* rounding.hpp:71 implied_slack_sort (stable), in place. */
void orc_implied_slack_sort(const orc_problem* p, const double* act, const int* ninf_min,
                            const int* ninf_max, int* vars, int nvars);

#ifdef __cplusplus
}
#endif
#endif
