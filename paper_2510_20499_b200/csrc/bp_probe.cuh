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
  // work of the branches (the reference trajectory's per-round dirty sets):
  // Σ|R_r|, Σ row nnz of R_r, Σ|V_r|, Σ col nnz of V_r, Σ|C_r| -- accumulated per warp / block
  unsigned long long* work;
};

void probe_launch(Problem& P, const ProbeRoot& R, ProbeBatch& B, const Limits& lim, cudaStream_t s);

// Dense per-block state of the block-per-branch kernel (bp_probe_block.cu): `nblocks` regions of
// `stride` bytes, zero-initialised once (stamps compare against ever-increasing tags).
struct BlockScratch {
  int nblocks = 0, n = 0, m = 0;
  size_t stride = 0;
  char* base    = nullptr;
  // per-block views (for_block)
  double2 *bnd = nullptr, *chgv = nullptr, *act = nullptr;
  int2* ainf = nullptr;
  unsigned *bst = nullptr, *vmark = nullptr, *ast = nullptr, *rmark = nullptr, *tagc = nullptr;
  int *dvar = nullptr, *chg = nullptr, *touch = nullptr, *drow = nullptr;

  __host__ __device__ BlockScratch for_block(int b) const
  {
    BlockScratch w = *this;
    char* p        = base + (size_t)b * stride;
    const size_t nn = n > 0 ? (size_t)n : 1, mm = m > 0 ? (size_t)m : 1;
    auto take = [&](size_t bytes) {
      char* q = p;
      p += (bytes + 15) / 16 * 16;
      return q;
    };
    w.bnd   = reinterpret_cast<double2*>(take(16 * nn));
    w.chgv  = reinterpret_cast<double2*>(take(16 * nn));
    w.act   = reinterpret_cast<double2*>(take(16 * mm));
    w.ainf  = reinterpret_cast<int2*>(take(8 * mm));
    w.bst   = reinterpret_cast<unsigned*>(take(4 * nn));
    w.vmark = reinterpret_cast<unsigned*>(take(4 * nn));
    w.dvar  = reinterpret_cast<int*>(take(4 * nn));
    w.chg   = reinterpret_cast<int*>(take(4 * nn));
    w.touch = reinterpret_cast<int*>(take(4 * nn));
    w.ast   = reinterpret_cast<unsigned*>(take(4 * mm));
    w.rmark = reinterpret_cast<unsigned*>(take(4 * mm));
    w.drow  = reinterpret_cast<int*>(take(4 * mm));
    w.tagc  = reinterpret_cast<unsigned*>(take(16));
    return w;
  }
};
size_t block_scratch_bytes(int n, int m);  // per block (upper bound of for_block's carving)
void probe_block_launch(Problem& P, const ProbeRoot& R, ProbeBatch& B, const Limits& lim,
                        BlockScratch& W, int full_first, cudaStream_t s);

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
  int n_block = 0;  // branches run by the block-per-branch kernel (large frontiers / uncertified root)
  unsigned long long work[5] = {0, 0, 0, 0, 0};  // ProbeBatch::work summed over the batches
  bool certified = false;
  double probe_ms = 0.0;  // device time of the batched probe kernel(s)

  void finalize_stats();
};

}  // namespace bp
