/* bp.h — C-ABI of the B200-native bound-propagation engine (drop-in for the reference's
 * bound propagation / probing / fix-and-propagate hot path, /root/reference/proj/include/pulse).
 *
 * Conventions (mirroring the reference):
 *  - plain host pointers and sizes; bounds are interleaved `b[2i] = lower, b[2i+1] = upper`
 *    exactly like pulse::BoundsState (propagation.hpp:16-18); activities are interleaved
 *    `act[2k] = finite part of min activity, act[2k+1] = max` like pulse::ActivityState
 *    (propagation.hpp:74-93).
 *  - every entry point returns BP_OK or an error code; the message is in bp_last_error().
 *    Error codes map 1:1 onto the exception types the reference throws
 *    (std::invalid_argument / std::out_of_range / std::runtime_error, problem.hpp:166-180).
 *  - infeasibility is data (a status / flag), never an error (propagation.hpp:261).
 *  - one bp_problem is the device-resident copy of one immutable pulse::ProblemDef
 *    (CSR + CSC + SoA bounds). Calls on one handle are serialized internally.
 *  - there is no CPU fallback: without a usable sm_100 device every compute call fails with
 *    BP_ERR_CUDA.
 */
#ifndef BP_H
#define BP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_OK 0
#define BP_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define BP_ERR_OUT_OF_RANGE 2     /* std::out_of_range */
#define BP_ERR_RUNTIME 3          /* std::runtime_error */
#define BP_ERR_CUDA 4             /* device / driver failure (no reference counterpart) */

/* pulse::PropagationStatus order (propagation.hpp:261). */
#define BP_TIGHTENED 0
#define BP_INFEASIBLE 1
#define BP_UNCHANGED 2

typedef struct bp_problem bp_problem;

/* Built problem (pulse::ProblemDef, problem.hpp:25-84): CSR with sorted, coalesced, zero-free
 * rows and integral integer-variable bounds (ProblemBuilder::build, problem.hpp:141-227).
 * col_* may be NULL, in which case the CSC is derived by the same stable transpose. */
typedef struct {
  int32_t n_vars;
  int32_t n_cons;
  const int32_t* row_start; /* n_cons + 1 */
  const int32_t* row_col;
  const double* row_val;
  const int32_t* col_start; /* n_vars + 1, or NULL */
  const int32_t* col_row;
  const double* col_val;
  const double* var_lower; /* n_vars, +-INFINITY for unbounded */
  const double* var_upper;
  const uint8_t* is_integer;
  const double* cons_lower; /* n_cons */
  const double* cons_upper;
} bp_problem_desc;

/* pulse::PropagationLimits (propagation.hpp:253-259). */
typedef struct {
  int32_t max_rounds;   /* 64 */
  double time_limit;    /* seconds, INFINITY */
  double abs_threshold; /* 1e-7 */
  double rel_threshold; /* 1e-4 */
  int32_t incremental;  /* 1 */
} bp_limits;

/* pulse::PropagationResult (propagation.hpp:263-267). */
typedef struct {
  int32_t status; /* BP_TIGHTENED / BP_INFEASIBLE / BP_UNCHANGED */
  int32_t rounds;
  int32_t crossed_vars;
} bp_result;

const char* bp_last_error(void);
void bp_limits_default(bp_limits* lim);
int bp_device_count(int32_t* count);

/* Device problem. Replaces the implicit "ProblemDef is shared by const reference" of the
 * reference: one upload per ProblemDef. */
int bp_problem_create(const bp_problem_desc* desc, int32_t device, bp_problem** out);
int bp_problem_destroy(bp_problem* p);
int bp_problem_info(const bp_problem* p, int32_t* n_vars, int32_t* n_cons, int64_t* nnz);

/* pulse::ProblemBuilder state (problem.hpp:102-242): variables, rows and the entries in
 * insertion order (add_entry), before build(). */
typedef struct {
  int32_t n_vars;
  int32_t n_cons;
  int64_t n_entries;
  const int32_t* entry_row;
  const int32_t* entry_col;
  const double* entry_val;
  const double* var_lower; /* as given to add_var (not yet integrally tightened) */
  const double* var_upper;
  const uint8_t* is_integer;
  const double* cons_lower;
  const double* cons_upper;
} bp_builder_desc;

/* The built pulse::ProblemDef arrays (caller-allocated): row_start n_cons + 1, col_start
 * n_vars + 1, row_col / row_val / col_row / col_val capacity n_entries, var_lower / var_upper
 * n_vars (integrally tightened). nnz is written. */
typedef struct {
  int64_t nnz;
  int32_t* row_start;
  int32_t* row_col;
  double* row_val;
  int32_t* col_start;
  int32_t* col_row;
  double* col_val;
  double* var_lower;
  double* var_upper;
} bp_built;

/* pulse::ProblemBuilder::build (problem.hpp:141-227) on the device: integral tightening, the
 * reference's checks (BP_ERR_RUNTIME for an empty domain / crossed row, BP_ERR_OUT_OF_RANGE for
 * an entry index), stable sort by (row, col), coalescing of duplicates (summed in insertion
 * order), zero dropping, CSR + stable-transpose CSC. If prob != NULL the built problem is also
 * created on `device` (as bp_problem_create). */
int bp_build_problem(const bp_builder_desc* desc, int32_t device, bp_built* out, bp_problem** prob);

/* pulse::compute_activities (propagation.hpp:226). rows == NULL with nrows < 0 recomputes all
 * rows; otherwise only rows[0..nrows) and the others keep the values passed in. */
int bp_compute_activities(bp_problem* p, const double* bounds2n, const int32_t* rows,
                          int32_t nrows, double* act2m, int32_t* ninf_min, int32_t* ninf_max);

/* pulse::tighten_bounds (propagation.hpp:378). vars == NULL with nvars < 0 sweeps all vars.
 * Writes changed vars ascending into `changed` (capacity n_vars) and their count; a crossing
 * sets *infeasible = 1 (BoundsState::mark_infeasible). crossed may be NULL. */
int bp_tighten_bounds(bp_problem* p, double* bounds2n, int32_t* infeasible, const double* act2m,
                      const int32_t* ninf_min, const int32_t* ninf_max, const int32_t* vars,
                      int32_t nvars, const bp_limits* lim, int32_t* changed, int32_t* n_changed,
                      int32_t* crossed);

/* pulse::propagate (propagation.hpp:418), in place on host bounds. lim may be NULL (defaults). */
int bp_propagate(bp_problem* p, double* bounds2n, int32_t* infeasible, const bp_limits* lim,
                 bp_result* res);

/* Same, on a device-resident bounds buffer (2n doubles) on `stream` (cudaStream_t or NULL). */
int bp_propagate_device(bp_problem* p, double* d_bounds2n, int32_t* infeasible,
                        const bp_limits* lim, bp_result* res, void* stream);

/* Device-resident propagate with options. flags: BP_FORCE_FRONTIER (bit 0) disables the engine's
 * full-round substitution for large frontiers, i.e. runs the reference's exact dirty-set
 * trajectory (results are bit-identical either way). d_stats, if non-NULL, is a DEVICE array of
 * 12 * max_rounds int64 receiving per round {full, |dirty rows|, row nnz visited, |dirty vars|,
 * col nnz visited, |changed vars|, and the phase-end times in ns since kernel start: activity,
 * tightening, row expansion, var expansion, gather, spare} — the reference's algorithmic work. */
#define BP_FORCE_FRONTIER 1
int bp_propagate_ex(bp_problem* p, double* d_bounds2n, int32_t* infeasible, const bp_limits* lim,
                    bp_result* res, void* stream, int32_t flags, int64_t* d_stats);

/* ---------------------------------------------------------------- probing cache
 * pulse::ProbingCache (probing.hpp:87-98) as an opaque host object built on the GPU. */
typedef struct bp_cache bp_cache;

/* Batched double probing: both branches of every listed variable, from root2n (NULL = the
 * problem's original bounds). Entries follow pulse::probe_variable (probing.hpp:225-238),
 * including default entries for variables without a branch spec. */
int bp_probe_variables(bp_problem* p, const double* root2n, const int32_t* vars, int32_t nvars,
                       bp_cache** out);
/* pulse::prioritize_probe_vars (probing.hpp:105-190): integer vars in probing priority order. */
int bp_prioritize_probe_vars(bp_problem* p, int32_t* order, int32_t* n_order);
/* pulse::build_cache (probing.hpp:243-281): root = original bounds; candidates = priority order
 * minus root-fixed vars; stops launching batches once budget_sec has elapsed. */
int bp_build_cache(bp_problem* p, double budget_sec, bp_cache** out);
int bp_cache_destroy(bp_cache* c);
/* Stats: n_probed / n_infeasible_branches as ProbingCache; n_fallback = branches that ran on the
 * full engine (uncertified root or overlay overflow); probe_ms = device time of the batch. */
int bp_cache_info(const bp_cache* c, int32_t* n_vars, int32_t* n_probed,
                  int32_t* n_infeasible_branches, int64_t* n_deltas, int32_t* n_fallback,
                  int32_t* certified, double* probe_ms);
/* Branches of the cache computed by the block-per-branch kernel (overlay overflows of the batched
 * warp kernel, or every branch when the root was not a certified fixpoint). */
int bp_cache_block_branches(const bp_cache* c, int32_t* n_block);
/* Work of the probed branches, summed over their rounds (the reference trajectory's dirty sets,
 * SURVEY §8d): {Σ|R_r|, Σ row nnz of R_r, Σ|V_r|, Σ col nnz of V_r, Σ|C_r|}. */
int bp_cache_work(const bp_cache* c, int64_t* work5);
/* Entry of v: *present = 0 if absent; hdr7 = {kind, forces_down, forces_up, down.feasible,
 * up.feasible, n_down_deltas, n_up_deltas}; br4 = {down lo, down up, up lo, up up}. */
int bp_cache_entry(const bp_cache* c, int32_t v, int32_t* present, int32_t* hdr7, double* br4);
/* Deltas of branch side (0 down, 1 up) of v, ascending by var (probing.hpp:213-217). */
int bp_cache_deltas(const bp_cache* c, int32_t v, int32_t side, int32_t* vars, double* lo,
                    double* up);
int bp_cache_root(const bp_cache* c, double* root2n);
int bp_cache_create_empty(int32_t n_vars, const double* root2n, bp_cache** out);
/* Adds the entry of v (pulse::ProbeEntry, probing.hpp:80-85) to a cache, e.g. to hand a host-built
 * pulse::ProbingCache to the engine: hdr5 = {kind, forces_down, forces_up, down.feasible,
 * up.feasible}, br4 = {down lo, down up, up lo, up up}, deltas ascending by var. An existing entry
 * of v is an error (BP_ERR_INVALID_ARGUMENT). */
int bp_cache_set_entry(bp_cache* c, int32_t v, const int32_t* hdr5, const double* br4,
                       int32_t n_down, const int32_t* down_vars, const double* down_lo,
                       const double* down_up, int32_t n_up, const int32_t* up_vars,
                       const double* up_lo, const double* up_up);
/* pulse::build_cache over several GPUs of one process (probing.hpp:243-281, the worker pool of
 * :256-272 with GPUs as workers). probs[d] is the same problem uploaded on a distinct
 * device. Candidates: `vars` (nvars >= 0, all probed) or, with vars == NULL, build_cache's own
 * (priority order minus root-fixed variables, each device's share under `budget_sec`). Device d
 * probes positions d, d + nprob, ... of the candidate list; the packed slices are gathered to
 * probs[0]'s device with NCCL send/recv (libnccl.so.2 resolved at run time) and merged there.
 * probe_ms_per_device (nprob, may be NULL) receives each device's probe-kernel time. The result
 * equals the single-GPU cache of the same candidates. */
int bp_build_cache_multi(bp_problem* const* probs, int32_t nprob, double budget_sec,
                         const int32_t* vars, int32_t nvars, bp_cache** out,
                         double* probe_ms_per_device);
/* Serialisation of a cache slice for the multi-GPU gather (NCCL) and merge on rank 0. */
int bp_cache_pack_size(const bp_cache* c, int64_t* bytes);
int bp_cache_pack(const bp_cache* c, void* buf, int64_t bytes);
int bp_cache_merge_packed(bp_cache* dst, const void* buf, int64_t bytes);
/* pulse::assemble_bulk_warm_start (probing.hpp:292-352): merged bounds (2n), conflicts as
 * (kept, evicted) pairs (capacity 2 * nvars ints: each assignment adds at most one pair, repeated
 * variables included), evicted vars (capacity nvars). */
int bp_assemble_bulk_warm_start(const bp_cache* c, const int32_t* vars, const double* vals,
                                int32_t n, double* bounds2n, int32_t* conflicts,
                                int32_t* n_conflicts, int32_t* evicted, int32_t* n_evicted);

/* ---------------------------------------------------------------- fix-and-propagate
 * pulse::RoundingConfig (rounding.hpp:18-31); the lp_polish fields are out of scope. */
typedef struct {
  double random_band;         /* 0.25 */
  int32_t single_var_tail;    /* 36 */
  int32_t repair_enabled;     /* 0 (rounding.hpp:25; on: failed single-var probes call bp_repair) */
  int32_t repair_attempt_cap; /* 16 */
  int32_t repair_shift_cap;   /* 64 */
} bp_rounding_config;

/* pulse::RoundingOutcome (rounding.hpp:347-355) minus the polished point; bounds_feasible = the
 * reference's lp_polish condition (completed && !rounding_infeasible && !ws.infeasible()). */
typedef struct {
  int32_t rounding_infeasible;
  int32_t timed_out;
  int32_t completed;
  int32_t repair_attempts;
  int32_t bulks_committed;
  int32_t set_count;
  int32_t bounds_feasible;
  int32_t bp_calls;   /* engine propagate launches */
  double device_ms;   /* device time of engine launches */
} bp_rounding_outcome;

void bp_rounding_config_default(bp_rounding_config* cfg);

/* pulse::propagation_round (rounding.hpp:393-558) with Rng(seed); deadline_sec <= 0 = never.
 * out_values (n_vars) receives the point before lp_polish: integer vars from the fixed bounds
 * (else nearest rounding), continuous vars clamped into their original bounds. cache may be NULL. */
int bp_propagation_round(bp_problem* p, const double* start_values, const bp_cache* cache,
                         uint64_t seed, double deadline_sec, const bp_rounding_config* cfg,
                         double* out_values, bp_rounding_outcome* out);

/* Same with the caller's generator instead of a seed (pulse::propagation_round takes Rng&): the
 * std::mt19937_64 text representation (`os << rng`) is read from rng_state and the advanced
 * state written back, so the caller's stream continues exactly as after the reference call. */
#define BP_RNG_STATE_BYTES 8192
int bp_propagation_round_rng(bp_problem* p, const double* start_values, const bp_cache* cache,
                             char* rng_state, int64_t rng_state_bytes, double deadline_sec,
                             const bp_rounding_config* cfg, double* out_values,
                             bp_rounding_outcome* out);

/* pulse::repair (rounding.hpp:234-311): shifts the fixed values (v, val) in list order, one variable
 * per most-violated row, until propagation from the original bounds with every value fixed
 * succeeds. *repaired = 1 on success (RepairResult present) with the shifted values in out_vals
 * (nfixed, same order as the input) and the propagated bounds in out_bounds2n; 0 = std::nullopt
 * (no in-bounds shift, shift cap cfg->repair_shift_cap reached, deadline expired, or propagation
 * infeasible without violated rows). deadline_sec <= 0 = never. cfg may be NULL (defaults). */
int bp_repair(bp_problem* p, const int32_t* fixed_vars, const double* fixed_vals, int32_t nfixed,
              double deadline_sec, const bp_rounding_config* cfg, int32_t* repaired,
              double* out_vals, double* out_bounds2n);

/* pulse::parallel_propagate (rounding.hpp:213-224; detail::run_probe :167-207): both candidate
 * vectors v0 / v1 for `vars` from host bounds base2n (+ its infeasible flag), warm-started from
 * `cache` when non-NULL. Per probe q in {0, 1}: out_bounds2n[q*2n .. (q+1)*2n) = ProbeResult.bounds,
 * out_infeasible[q] = bounds.infeasible(), infeas_count[q], evicted[q*nvars ..] / n_evicted[q],
 * fixed_vars / fixed_vals[q*nvars ..] / n_fixed[q] (ProbeResult.fixed). */
int bp_parallel_propagate(bp_problem* p, const double* base2n, int32_t base_infeasible,
                          const int32_t* vars, int32_t nvars, const double* v0, const double* v1,
                          const bp_cache* cache, double* out_bounds2n, int32_t* out_infeasible,
                          int32_t* infeas_count, int32_t* evicted, int32_t* n_evicted,
                          int32_t* fixed_vars, double* fixed_vals, int32_t* n_fixed);

/* ---------------------------------------------------------------- PDHG (lp.hpp)
 * pulse::LpInstance (lp.hpp:17-47) on the device: the sparse products of the PDHG solver and its
 * inner iteration, bit-identical to the reference (16384-entry segment summation, no FMA). */
typedef struct bp_lp bp_lp;
typedef struct {
  int32_t n_vars;
  int32_t n_rows;
  const int32_t* row_start; /* CSR, n_rows + 1 */
  const int32_t* row_col;
  const double* row_val;
  const int32_t* col_start; /* CSC, n_vars + 1 */
  const int32_t* col_row;
  const double* col_val;
  const double* obj;        /* n_vars, may be NULL (then bp_lp_pdhg_iterate is unavailable) */
  const double* row_lower;  /* n_rows */
  const double* row_upper;
  const double* var_lower;  /* n_vars */
  const double* var_upper;
} bp_lp_desc;

int bp_lp_create(const bp_lp_desc* desc, int32_t device, bp_lp** out);
int bp_lp_destroy(bp_lp* lp);
/* lpdetail::spmv_rows (lp.hpp:74-87): ax[k] = sum_e row_val[e] * x[row_col[e]]. */
int bp_lp_spmv_rows(bp_lp* lp, const double* x, double* ax);
/* lpdetail::spmv_cols (lp.hpp:89-102): aty[i] = sum_e col_val[e] * y[col_row[e]]. */
int bp_lp_spmv_cols(bp_lp* lp, const double* y, double* aty);
/* `iters` PDHG iterations of pulse::lp::solve's inner loop (lp.hpp:315-340) with fixed step sizes:
 * dual ascent y <- prox(y + sigma A x_bar), primal descent x <- clamp(x - tau (c + A'y)),
 * x_bar <- 2 x_new - x, x_sum += x, y_sum += y. All five vectors are read and written back. */
int bp_lp_pdhg_iterate(bp_lp* lp, double* x, double* y, double* x_bar, double* x_sum, double* y_sum,
                       double tau, double sigma, int32_t iters);
/* lpdetail::evaluate_kkt (lp.hpp:134-206) at (x, y): out7 = {primal_res, dual_res, gap,
 * primal_obj, dual_obj, x_norm, score}. The residual maxima are exact; the objective sums are
 * compensated (double-double, fixed order) where the reference uses a sequential Neumaier sum, so
 * primal_obj / dual_obj (and gap / score) agree with it to a few ulps, not bitwise. */
int bp_lp_evaluate_kkt(bp_lp* lp, const double* x, const double* y, double* out7);
/* Device time (CUDA events on the LP's stream) of the last spmv / iterate / KKT call. */
int bp_lp_last_ms(const bp_lp* lp, double* ms);

/* Number of engine kernels launched by this process. */
int64_t bp_kernel_launches(void);

/* Device time of engine launches on this problem, measured with CUDA events recorded on the
 * launching stream around each launch: the last one, the running total, and the launch count. */
int bp_kernel_time(const bp_problem* p, double* last_ms, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* BP_H */
