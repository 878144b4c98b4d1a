// Batched probing: device structures and the host-side cache (probing.hpp:62-98).
#pragma once
#include <cstdint>
#include <vector>

#include "bp_engine.cuh"

namespace bp {

// Read-only root state shared by all branches of a batch.
struct ProbeRoot {
  const double2* bounds;  // root bounds (n)
  const RowRec* rec;      // root row activities (certified fixpoint)
  const double2* aux;
};

// One branch per task: variable + branch interval. Outputs per task and a delta pool.
struct ProbeBatch {
  int n_task;
  const int* var;
  const double* lo;
  const double* up;
  int* cursor;
  int* status;      // 0 feasible, 1 infeasible, 2 overlay overflow, 3 pool exhausted
  int* dcount;
  long long* doff;
  unsigned long long* pool_cursor;
  long long pool_cap;
  int* pvar;
  double* plo;
  double* pup;
};

void probe_launch(Problem& P, const ProbeRoot& R, ProbeBatch& B, const Limits& lim, cudaStream_t s);

// pulse::ProbingCache restated as flat arrays (probing.hpp:87-98).
struct HostCache {
  int n = 0;
  std::vector<double> root;        // 2n
  std::vector<int> entry_of;       // n: -1 or entry index
  // per entry
  std::vector<int> e_var, e_kind;  // kind: BranchKind (0 BoxedSplit, 1 AtLowerBound, 2 AtUpperBound)
  std::vector<uint8_t> e_feas;     // 2 per entry (down, up)
  std::vector<uint8_t> e_force;    // 2 per entry (forces_down, forces_up)
  std::vector<double> e_branch;    // 4 per entry
  std::vector<long long> d_off;    // 2 per entry + 1 (branch s of entry e: [d_off[2e+s], d_off[2e+s+1]))
  std::vector<int> d_var;
  std::vector<double> d_lo, d_up;
  int n_probed = 0, n_infeasible_branches = 0, n_fallback = 0;
  bool certified = false;
  double probe_ms = 0.0;  // device time of the batched probe kernel(s)

  void finalize_stats();
};

}  // namespace bp
