// Internal glue shared by the C-ABI translation units (not part of the public ABI).
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/bp.h"
#include "bp_engine.cuh"

// Host copies of the problem kept for host-side steps (priority keys, rounding driver).
struct bp_problem_host {
  std::vector<int> col_row;
  std::vector<double> col_val, var_lower, var_upper, cons_lower, cons_upper;
  std::vector<uint8_t> is_integer;
  std::vector<int> row_col;
  std::vector<double> row_val;
};

bp::Problem& bp_problem_impl(bp_problem* p);
const bp_problem_host& bp_problem_hostdata(bp_problem* p);
void bp_problem_root(bp_problem* p, double* root2n);
void bp_set_last_error(const char* msg);

namespace bp {
struct HostCache;
void warm_start_sparse(const HostCache& C, const int* vars, const double* vals, int na,
                       std::vector<int>& dv, std::vector<double>& dl, std::vector<double>& du,
                       std::vector<int>& conflicts, std::vector<int>& evicted);
}  // namespace bp
const bp::HostCache* bp_cache_host(const bp_cache* c);
// A new cache handle owning `c` (moved in).
bp_cache* bp_cache_adopt(bp::HostCache&& c);
