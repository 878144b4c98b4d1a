// Problem build on the device: pulse::ProblemBuilder::build (problem.hpp:141-227).
//
// The reference's build is O(N log N) host work per problem (a std::sort of (row, col, val)
// tuples, a sequential coalescing pass and a stable transpose); fp.hpp:253 rebuilds a problem
// for every objective cut. Here the N entries are uploaded once and every O(N) / O(N log N) step
// runs on the GPU:
//   1. integral tightening of integer-variable bounds, ceil(l - 1e-9) / floor(u + 1e-9)
//      (problem.hpp:157-163; an integer lower bound in (-1, 0] becomes -0.0, as there), and the
//      reference's error checks in its order (empty domains, crossed rows, entry indices);
//   2. packed (row, col) keys sorted by a stable LSD radix sort (CUB) over their used bits only, so
//      duplicates keep insertion order;
//   3. duplicates coalesced by one thread per (row, col) run, summing left to right from the first
//      value like the reference's `merged.back() += t` pass, then explicit zeros dropped;
//   4. CSR offsets by histogram + scan; the CSC by a stable radix sort of the CSR positions on
//      their column (columns list their rows ascending, problem.hpp:211-225).
// The built arrays are copied back for the caller's pulse::ProblemDef and, optionally, uploaded
// into a bp_problem (bp_problem_create with the CSC given, so nothing is recomputed on the host).
//
// Duplicate order: std::sort is not stable, so the reference sums >= 3 duplicates of one
// (row, col) in an unspecified order; here it is insertion order. Two duplicates (a + b == b + a)
// and integer-valued duplicates give identical bits either way.
#include <cub/cub.cuh>

#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bp.h"
#include "bp_capi_internal.h"
#include "bp_engine.cuh"

namespace bp {
namespace {

inline int nblk(long long n) { return (int)std::max(1ll, std::min(4096ll, (n + 255) / 256)); }

// problem.hpp:157-168: integral tightening, then the first empty domain (atomicMin of its index).
__global__ void k_round_bounds(int n, const uint8_t* isint, double* lo, double* up, int* first_bad)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double l = lo[i], u = up[i];
    if (isint[i]) {
      if (isfinite(l)) l = ceil(__dsub_rn(l, 1e-9));
      if (isfinite(u)) u = floor(__dadd_rn(u, 1e-9));
      lo[i] = l;
      up[i] = u;
    }
    if (l > u) atomicMin(first_bad, i);
  }
}

__global__ void k_crossed_rows(int m, const double* lo, const double* up, int* first_bad)
{
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x)
    if (lo[k] > up[k]) atomicMin(first_bad, k);
}

// problem.hpp:178-181: first entry (insertion order) with a bad row or col; keys
// (row << cbits | col), cbits = bits of n, so the sort touches only rbits + cbits bits.
__global__ void k_entry_keys(long long N, int n, int m, int cbits, const int* row, const int* col,
                             unsigned long long* key, unsigned long long* first_bad)
{
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = row[e], c = col[e];
    if (r < 0 || r >= m || c < 0 || c >= n) {
      atomicMin(first_bad, (unsigned long long)e);
      key[e] = 0;
      continue;
    }
    key[e] = ((unsigned long long)(unsigned)r << cbits) | (unsigned)c;
  }
}

__global__ void k_run_heads(long long N, const unsigned long long* key, unsigned char* head)
{
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N;
       e += (long long)gridDim.x * blockDim.x)
    head[e] = (e == 0 || key[e] != key[e - 1]) ? 1 : 0;
}

// problem.hpp:188-199: one thread per run of equal keys, left-to-right sum from its first value;
// keep = the coalesced value is not zero (problem.hpp:200-203).
__global__ void k_coalesce(long long R, long long N, const long long* start,
                           const unsigned long long* key, const double* val,
                           unsigned long long* ukey, double* uval, unsigned char* keep)
{
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < R;
       j += (long long)gridDim.x * blockDim.x) {
    const long long s = start[j], e = j + 1 < R ? start[j + 1] : N;
    double acc = val[s];
    for (long long q = s + 1; q < e; ++q) acc = __dadd_rn(acc, val[q]);
    ukey[j] = key[s];
    uval[j] = acc;
    keep[j] = acc != 0.0 ? 1 : 0;
  }
}

// CSR split of the final keys + per-row / per-column counts.
__global__ void k_split(long long nnz, int cbits, const unsigned long long* key, int* row, int* col,
                        unsigned* col_key, int* rcount, int* ccount)
{
  const unsigned long long cmask = (1ull << cbits) - 1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(key[e] >> cbits), c = (int)(key[e] & cmask);
    row[e]     = r;
    col[e]     = c;
    col_key[e] = (unsigned)c;
    atomicAdd(rcount + r, 1);
    atomicAdd(ccount + c, 1);
  }
}

__global__ void k_iota(long long N, long long* out)
{
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = e;
}

__global__ void k_iota32(int N, int* out)
{
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N; e += gridDim.x * blockDim.x) out[e] = e;
}

__global__ void k_csc_gather(int nnz, const int* perm, const int* row, const double* val,
                             int* col_row, double* col_val)
{
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += gridDim.x * blockDim.x) {
    const int e = perm[j];
    col_row[j]  = row[e];
    col_val[j]  = val[e];
  }
}

template <class T>
void h2d(DBuf<T>& b, const T* src, size_t n, cudaStream_t s)
{
  b.alloc(std::max<size_t>(n, 1));
  if (n) BP_CUDA(cudaMemcpyAsync(b.p, src, sizeof(T) * n, cudaMemcpyHostToDevice, s));
}

struct CubTmp {
  DBuf<unsigned char> b;
  void* get(size_t bytes)
  {
    if (bytes > b.n) b.alloc(bytes);
    return b.p;
  }
};

}  // namespace
}  // namespace bp

extern "C" int bp_build_problem(const bp_builder_desc* d, int32_t device, bp_built* out,
                                bp_problem** prob)
{
  using namespace bp;
  try {
    if (!d || !out) throw std::invalid_argument("null argument");
    if (d->n_vars < 0 || d->n_cons < 0 || d->n_entries < 0) throw std::invalid_argument("negative size");
    const int n = d->n_vars, m = d->n_cons;
    const long long N = d->n_entries;
    if ((n && (!d->var_lower || !d->var_upper || !d->is_integer)) || (m && (!d->cons_lower || !d->cons_upper)) ||
        (N && (!d->entry_row || !d->entry_col || !d->entry_val)))
      throw std::invalid_argument("missing builder arrays");
    if (!out->row_start || !out->col_start || (n && (!out->var_lower || !out->var_upper)) ||
        (N && (!out->row_col || !out->row_val || !out->col_row || !out->col_val)))
      throw std::invalid_argument("missing output arrays");
    if (N >= (1ll << 31)) throw std::invalid_argument("more than 2^31 - 1 entries");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw cuda_error("no CUDA device available (the engine has no CPU fallback)");
    if (device < 0 || device >= ndev) throw std::invalid_argument("device index out of range");
    BP_CUDA(cudaSetDevice(device));
    cudaStream_t s;
    BP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    CubTmp tmp;

    // 1. bounds and the reference's checks, in its order
    DBuf<double> lo, up, clo, cup;
    DBuf<uint8_t> isint;
    h2d(lo, d->var_lower, n, s);
    h2d(up, d->var_upper, n, s);
    h2d(isint, d->is_integer, n, s);
    h2d(clo, d->cons_lower, m, s);
    h2d(cup, d->cons_upper, m, s);
    DBuf<int> bad;
    bad.alloc(2);
    BP_CUDA(cudaMemsetAsync(bad.p, 0x7f, 2 * sizeof(int), s));
    if (n) k_round_bounds<<<nblk(n), 256, 0, s>>>(n, isint.p, lo.p, up.p, bad.p);
    if (m) k_crossed_rows<<<nblk(m), 256, 0, s>>>(m, clo.p, cup.p, bad.p + 1);
    // 2. entry keys (+ the first bad entry), stable sort by (row, col)
    DBuf<int> erow, ecol;
    DBuf<double> eval;
    h2d(erow, d->entry_row, N, s);
    h2d(ecol, d->entry_col, N, s);
    h2d(eval, d->entry_val, N, s);
    DBuf<unsigned long long> key, key2, badE;
    key.alloc(std::max(N, 1ll));
    key2.alloc(std::max(N, 1ll));
    badE.alloc(1);
    BP_CUDA(cudaMemsetAsync(badE.p, 0xff, sizeof(unsigned long long), s));
    auto bits = [](long long x) {
      int b = 1;
      while ((1ll << b) < x) ++b;
      return b;
    };
    const int cbits = bits(std::max(n, 1)), rbits = bits(std::max(m, 1));
    if (N) k_entry_keys<<<nblk(N), 256, 0, s>>>(N, n, m, cbits, erow.p, ecol.p, key.p, badE.p);
    int hbad[2];
    unsigned long long hbadE = 0;
    BP_CUDA(cudaMemcpyAsync(hbad, bad.p, sizeof(hbad), cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaMemcpyAsync(&hbadE, badE.p, sizeof(hbadE), cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaStreamSynchronize(s));
    if (hbad[0] != 0x7f7f7f7f)
      throw std::runtime_error("variable " + std::to_string(hbad[0]) + " has empty domain after bound tightening");
    if (hbad[1] != 0x7f7f7f7f)
      throw std::runtime_error("constraint " + std::to_string(hbad[1]) + " has crossed bounds");
    if (hbadE != ~0ull) {
      const int r = d->entry_row[hbadE];
      throw std::out_of_range(r < 0 || r >= m ? "entry row out of range" : "entry col out of range");
    }
    // stable LSD radix sort over the rbits + cbits key bits only
    DBuf<double> val2;
    val2.alloc(std::max(N, 1ll));
    if (N) {
      size_t nb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, nb, key.p, key2.p, eval.p, val2.p, (int)N, 0,
                                      rbits + cbits, s);
      size_t have = nb;
      cub::DeviceRadixSort::SortPairs(tmp.get(nb), have, key.p, key2.p, eval.p, val2.p, (int)N, 0,
                                      rbits + cbits, s);
    }
    // 3. coalesce runs of equal keys, drop zeros
    DBuf<unsigned char> head, keep;
    DBuf<long long> iota, start;
    DBuf<int> nsel;
    head.alloc(std::max(N, 1ll));
    iota.alloc(std::max(N, 1ll));
    start.alloc(std::max(N, 1ll));
    nsel.alloc(2);
    long long R = 0;
    if (N) {
      k_run_heads<<<nblk(N), 256, 0, s>>>(N, key2.p, head.p);
      k_iota<<<nblk(N), 256, 0, s>>>(N, iota.p);
      size_t nb = 0;
      cub::DeviceSelect::Flagged(nullptr, nb, iota.p, head.p, start.p, nsel.p, (int)N, s);
      size_t have = nb;
      cub::DeviceSelect::Flagged(tmp.get(nb), have, iota.p, head.p, start.p, nsel.p, (int)N, s);
      int hR = 0;
      BP_CUDA(cudaMemcpyAsync(&hR, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaStreamSynchronize(s));
      R = hR;
    }
    DBuf<unsigned long long> ukey, fkey;
    DBuf<double> uval, fval;
    ukey.alloc(std::max(R, 1ll));
    uval.alloc(std::max(R, 1ll));
    keep.alloc(std::max(R, 1ll));
    fkey.alloc(std::max(R, 1ll));
    fval.alloc(std::max(R, 1ll));
    long long nnz = 0;
    if (R) {
      k_coalesce<<<nblk(R), 256, 0, s>>>(R, N, start.p, key2.p, val2.p, ukey.p, uval.p, keep.p);
      size_t nb = 0;
      cub::DeviceSelect::Flagged(nullptr, nb, ukey.p, keep.p, fkey.p, nsel.p, (int)R, s);
      size_t have = nb;
      cub::DeviceSelect::Flagged(tmp.get(nb), have, ukey.p, keep.p, fkey.p, nsel.p, (int)R, s);
      cub::DeviceSelect::Flagged(nullptr, nb, uval.p, keep.p, fval.p, nsel.p + 1, (int)R, s);
      have = nb;
      cub::DeviceSelect::Flagged(tmp.get(nb), have, uval.p, keep.p, fval.p, nsel.p + 1, (int)R, s);
      int hn = 0;
      BP_CUDA(cudaMemcpyAsync(&hn, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaStreamSynchronize(s));
      nnz = hn;
    }
    // 4. CSR offsets, CSC by a stable sort of the CSR positions on their column
    DBuf<int> row, col, rcount, ccount, rstart, cstart, pos, perm, crow;
    DBuf<unsigned> ckey, ckey2;
    DBuf<double> cval;
    const size_t z = (size_t)std::max(nnz, 1ll);
    row.alloc(z);
    col.alloc(z);
    ckey.alloc(z);
    ckey2.alloc(z);
    pos.alloc(z);
    perm.alloc(z);
    crow.alloc(z);
    cval.alloc(z);
    rcount.alloc(m + 1);
    ccount.alloc(n + 1);
    rstart.alloc(m + 1);
    cstart.alloc(n + 1);
    BP_CUDA(cudaMemsetAsync(rcount.p, 0, sizeof(int) * (m + 1), s));
    BP_CUDA(cudaMemsetAsync(ccount.p, 0, sizeof(int) * (n + 1), s));
    if (nnz) k_split<<<nblk(nnz), 256, 0, s>>>(nnz, cbits, fkey.p, row.p, col.p, ckey.p, rcount.p, ccount.p);
    {
      size_t nb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, nb, rcount.p, rstart.p, m + 1, s);
      size_t have = nb;
      cub::DeviceScan::ExclusiveSum(tmp.get(nb), have, rcount.p, rstart.p, m + 1, s);
      cub::DeviceScan::ExclusiveSum(nullptr, nb, ccount.p, cstart.p, n + 1, s);
      have = nb;
      cub::DeviceScan::ExclusiveSum(tmp.get(nb), have, ccount.p, cstart.p, n + 1, s);
    }
    if (nnz) {
      k_iota32<<<nblk(nnz), 256, 0, s>>>((int)nnz, pos.p);
      size_t nb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, nb, ckey.p, ckey2.p, pos.p, perm.p, (int)nnz, 0, cbits, s);
      size_t have = nb;
      cub::DeviceRadixSort::SortPairs(tmp.get(nb), have, ckey.p, ckey2.p, pos.p, perm.p, (int)nnz, 0,
                                      cbits, s);
      k_csc_gather<<<nblk(nnz), 256, 0, s>>>((int)nnz, perm.p, row.p, fval.p, crow.p, cval.p);
    }
    // 5. results to the caller's ProblemDef arrays
    out->nnz = nnz;
    BP_CUDA(cudaMemcpyAsync(out->row_start, rstart.p, sizeof(int) * (m + 1), cudaMemcpyDeviceToHost, s));
    BP_CUDA(cudaMemcpyAsync(out->col_start, cstart.p, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, s));
    if (nnz) {
      BP_CUDA(cudaMemcpyAsync(out->row_col, col.p, sizeof(int) * nnz, cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaMemcpyAsync(out->row_val, fval.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaMemcpyAsync(out->col_row, crow.p, sizeof(int) * nnz, cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaMemcpyAsync(out->col_val, cval.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
    }
    if (n) {
      BP_CUDA(cudaMemcpyAsync(out->var_lower, lo.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      BP_CUDA(cudaMemcpyAsync(out->var_upper, up.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    }
    BP_CUDA(cudaStreamSynchronize(s));
    if (prob) {
      *prob = nullptr;
      bp_problem_desc pd;
      pd.n_vars     = n;
      pd.n_cons     = m;
      pd.row_start  = out->row_start;
      pd.row_col    = out->row_col;
      pd.row_val    = out->row_val;
      pd.col_start  = out->col_start;
      pd.col_row    = out->col_row;
      pd.col_val    = out->col_val;
      pd.var_lower  = out->var_lower;
      pd.var_upper  = out->var_upper;
      pd.is_integer = d->is_integer;
      pd.cons_lower = d->cons_lower;
      pd.cons_upper = d->cons_upper;
      const int rc  = bp_problem_create(&pd, device, prob);
      if (rc != BP_OK) return rc;
    }
    return BP_OK;
  } catch (const std::invalid_argument& e) {
    bp_set_last_error(e.what());
    return BP_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    bp_set_last_error(e.what());
    return BP_ERR_OUT_OF_RANGE;
  } catch (const bp::cuda_error& e) {
    bp_set_last_error(e.what());
    return BP_ERR_CUDA;
  } catch (const std::exception& e) {
    bp_set_last_error(e.what());
    return BP_ERR_RUNTIME;
  }
}
