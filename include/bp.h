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

/* Number of engine kernels launched by this process. */
int64_t bp_kernel_launches(void);

/* Device time of engine launches on this problem, measured with CUDA events recorded on the
 * launching stream around each launch: the last one, the running total, and the launch count. */
int bp_kernel_time(const bp_problem* p, double* last_ms, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* BP_H */
