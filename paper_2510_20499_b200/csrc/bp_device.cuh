// Device-side data model and arithmetic helpers of the bound-propagation engine.
//
// Bit-exactness contract: every floating-point expression below reproduces the
// reference's operation order with separately rounded IEEE operations (the library is compiled
// with --fmad=false, so no multiply-add is ever contracted), `std::min/max` are restated as
// "keep the first operand on ties" (never fmin/fmax: they differ on signed zeros), and
// activities are sequential sums within fixed 16384-entry segments (problem.hpp:274).
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace bp {

enum { BP_STATUS_UNSET = -1, BP_STATUS_TIGHTENED = 0, BP_STATUS_INFEASIBLE = 1, BP_STATUS_UNCHANGED = 2 };

constexpr int kSumSegment = 16384;   // problem.hpp:274
constexpr int kShortNnz   = 32;      // rows/cols at or below: one lane each
constexpr double kIntEps  = 1e-6;    // common.hpp:24

// Row record gathered by the tightening sweep: one 32-byte sector, one LDG.256.
//   min/max = finite parts of the min/max activity when no infinite contributor exists;
//             otherwise a NaN box carrying the infinite-contributor count, with the finite part
//             in RowAux (read only in the rare "single infinite contributor" case,
//             propagation.hpp:311-313).
//   g/h     = cons_upper / cons_lower (static), co-located so a gather fetches everything.
struct alignas(32) RowRec {
  double min, max, g, h;
};

constexpr unsigned long long kBoxMask = 0xFFFFFFFF00000000ull;
constexpr unsigned long long kBoxBase = 0x7FF4B0B000000000ull;  // payload arithmetic never makes

__host__ __device__ __forceinline__ double box_count(int c)
{
  unsigned long long u = kBoxBase | (unsigned long long)(unsigned)c;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
__device__ __forceinline__ bool is_box(double x)
{
  return ((unsigned long long)__double_as_longlong(x) & kBoxMask) == kBoxBase;
}
__device__ __forceinline__ int box_value(double x)
{
  return (int)(unsigned)((unsigned long long)__double_as_longlong(x) & 0xFFFFFFFFull);
}

// std::min / std::max semantics (first operand kept on ties).
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

__device__ __forceinline__ RowRec ld_rec(const RowRec* p)
{
  RowRec r;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.min), "=d"(r.max), "=d"(r.g), "=d"(r.h)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_rec(RowRec* p, const RowRec& r)
{
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r.min), "d"(r.max), "d"(r.g),
               "d"(r.h)
               : "memory");
}

// Activity contribution of one entry (propagation.hpp:159-170). Infinite contributors return a
// 0.0 contribution plus a count: adding +0.0 to a running sum that starts at +0.0 never changes
// it (the running sum can never be -0.0 under round-to-nearest), so this equals "skip".
__device__ __forceinline__ void contrib(double a, double lo, double up, double& cmin, double& cmax,
                                        int& imin, int& imax)
{
  if (a > 0.0) {
    imin = (lo == -INFINITY);
    imax = (up == INFINITY);
    cmin = imin ? 0.0 : __dmul_rn(a, lo);
    cmax = imax ? 0.0 : __dmul_rn(a, up);
  } else {
    imin = (up == INFINITY);
    imax = (lo == -INFINITY);
    cmin = imin ? 0.0 : __dmul_rn(a, up);
    cmax = imax ? 0.0 : __dmul_rn(a, lo);
  }
}

struct Limits {
  int max_rounds;
  double time_limit;
  double abs_threshold;
  double rel_threshold;
  int incremental;
};

// propagation.hpp:273-282
__device__ __forceinline__ bool counts_as_change(double imp, bool integer, double width,
                                                 const Limits& lim)
{
  if (imp <= 0.0) return false;
  if (imp == INFINITY) return true;
  if (integer) return imp >= 1.0 - 1e-9;
  double thr = lim.abs_threshold;
  if (isfinite(width)) thr = smax(thr, __dmul_rn(lim.rel_threshold, width));
  return imp > thr;
}

// Candidate fold state of one variable: new bound value + CSC position of the element that
// set it (-1 = the current bound). The sequential std::min fold of the reference keeps the
// FIRST minimal element, i.e. the lexicographic minimum of (value, position) under numeric
// equality -- which is associative, so long columns may be reduced in parallel.
struct Fold {
  double lo;
  int lo_pos;
  double up;
  int up_pos;
};

// Candidate bounds one row implies for one of its variables (propagation.hpp:297-352), from the
// row's activity given explicitly: finite parts mnf/mxf and infinite-contributor counts nmn/nmx.
// cl = lower-bound candidate or -inf, cu = upper-bound candidate or +inf (at most one of each per
// entry; the sentinels are never taken by the strict comparisons of the fold).
__device__ __forceinline__ void cand_explicit(double lo, double up, bool integer, double a,
                                              double mnf, int nmn, double mxf, int nmx, double g,
                                              double h, double& cl, double& cu)
{
  cl = -INFINITY;
  cu = INFINITY;
  if (isfinite(g)) {
    const bool my_inf = (a > 0.0) ? (lo == -INFINITY) : (up == INFINITY);
    bool usable       = false;
    double rest       = 0.0;
    if (nmn == 0) {
      rest   = __dsub_rn(mnf, (a > 0.0) ? __dmul_rn(a, lo) : __dmul_rn(a, up));
      usable = true;
    } else if (nmn == 1 && my_inf) {
      rest   = mnf;
      usable = true;
    }
    if (usable) {
      const double cand = __ddiv_rn(__dsub_rn(g, rest), a);
      if (a > 0.0) cu = integer ? floor(__dadd_rn(cand, kIntEps)) : cand;
      else cl = integer ? ceil(__dsub_rn(cand, kIntEps)) : cand;
    }
  }
  if (isfinite(h)) {
    const bool my_inf = (a > 0.0) ? (up == INFINITY) : (lo == -INFINITY);
    bool usable       = false;
    double rest       = 0.0;
    if (nmx == 0) {
      rest   = __dsub_rn(mxf, (a > 0.0) ? __dmul_rn(a, up) : __dmul_rn(a, lo));
      usable = true;
    } else if (nmx == 1 && my_inf) {
      rest   = mxf;
      usable = true;
    }
    if (usable) {
      const double cand = __ddiv_rn(__dsub_rn(h, rest), a);
      if (a > 0.0) cl = integer ? ceil(__dsub_rn(cand, kIntEps)) : cand;
      else cu = integer ? floor(__dadd_rn(cand, kIntEps)) : cand;
    }
  }
}

// Candidate gating. An entry (a, lo, up) of a row can only publish a candidate
// from side g (cons upper, min activity) if the row's slack g - act_min is below |a|·(width + 1
// for integers): its exact candidate is lo + slack/a (a > 0) or up - slack/|a| (a < 0), and the
// computed one differs from it by at most 5u(|a·x| + |act| + |g|)/|a|. So when
//   slack >= tw·(1 + 1e-12) + 1e-12·(|g| + |act| + pm),  tw = |a|(w + int), pm = |a|max(|lo|,|up|)
// the computed candidate is provably not strictly improving (for integers: floor/ceil land at or
// beyond the bound), i.e. cand_explicit would publish nothing from that side. The same holds for
// side h with slack act_max - h. Gating only skips work whose outcome is known: results are
// bit-identical with or without it.
__device__ __forceinline__ void entry_reach(double a, double lo, double up, bool integer, double& tw,
                                            double& pm)
{
  const double aa = fabs(a);
  const double w  = __dsub_rn(up, lo);  // +inf when either bound is infinite
  tw              = __dmul_rn(aa, integer ? __dadd_rn(w, 1.0) : w);
  pm              = __dmul_rn(aa, fmax(fabs(lo), fabs(up)));
}

// Side with slack `slack` (finite rhs, no infinite contributor) cannot yield a candidate for an
// entry of reach (tw, pm).
__device__ __forceinline__ bool side_quiet(double slack, double tw, double pm, double rhs, double act)
{
  const double margin = __dmul_rn(1e-12, __dadd_rn(__dadd_rn(fabs(rhs), fabs(act)), pm));
  return slack >= __dadd_rn(__dmul_rn(tw, 1.0 + 1e-12), margin) + 1e-300;
}

// True when neither side of the row can give this entry a candidate (see entry_reach).
__device__ __forceinline__ bool entry_quiet(double tw, double pm, double mnf, int nmn, double mxf,
                                            int nmx, double g, double h)
{
  const bool qg = !isfinite(g) || nmn >= 2 || (nmn == 0 && side_quiet(__dsub_rn(g, mnf), tw, pm, g, mnf));
  const bool qh = !isfinite(h) || nmx >= 2 || (nmx == 0 && side_quiet(__dsub_rn(mxf, h), tw, pm, h, mxf));
  return qg && qh;
}

// Decodes a row record (+ its aux finite parts when boxed).
__device__ __forceinline__ void decode_rec(const RowRec& r, const double2* aux, int k, double& mnf,
                                           int& nmn, double& mxf, int& nmx)
{
  nmn = is_box(r.min) ? box_value(r.min) : 0;
  nmx = is_box(r.max) ? box_value(r.max) : 0;
  mnf = r.min;
  mxf = r.max;
  if (nmn | nmx) {
    const double2 x = aux[k];
    if (nmn) mnf = x.x;
    if (nmx) mxf = x.y;
  }
}

// One CSC entry's contribution to the fold (propagation.hpp:297-352), position-tagged.
__device__ __forceinline__ void fold_entry(Fold& f, double lo, double up, bool integer, double a,
                                           const RowRec& r, const double2* aux, int k, int pos)
{
  double mnf, mxf, cl, cu;
  int nmn, nmx;
  decode_rec(r, aux, k, mnf, nmn, mxf, nmx);
  double tw, pm;
  entry_reach(a, lo, up, integer, tw, pm);
  if (entry_quiet(tw, pm, mnf, nmn, mxf, nmx, r.g, r.h)) return;
  cand_explicit(lo, up, integer, a, mnf, nmn, mxf, nmx, r.g, r.h, cl, cu);
  if (cu < f.up) { f.up = cu; f.up_pos = pos; }
  if (f.lo < cl) { f.lo = cl; f.lo_pos = pos; }
}

// Candidates of one CSC entry from the gathered row record.
__device__ __forceinline__ void entry_candidates(double lo, double up, bool integer, double a,
                                                 const RowRec& r, const double2* aux, int k,
                                                 double& cl, double& cu)
{
  double mnf, mxf;
  int nmn, nmx;
  decode_rec(r, aux, k, mnf, nmn, mxf, nmx);
  double tw, pm;
  entry_reach(a, lo, up, integer, tw, pm);
  if (entry_quiet(tw, pm, mnf, nmn, mxf, nmx, r.g, r.h)) {
    cl = -INFINITY;
    cu = INFINITY;
    return;
  }
  cand_explicit(lo, up, integer, a, mnf, nmn, mxf, nmx, r.g, r.h, cl, cu);
}

// Combine two partial folds of disjoint position sets (lexicographic (value, position)).
__device__ __forceinline__ void fold_combine(Fold& f, double olo, int olo_pos, double oup,
                                             int oup_pos)
{
  if (f.lo < olo || (olo == f.lo && olo_pos < f.lo_pos)) { f.lo = olo; f.lo_pos = olo_pos; }
  if (oup < f.up || (oup == f.up && oup_pos < f.up_pos)) { f.up = oup; f.up_pos = oup_pos; }
}

// propagation.hpp:354-369. Returns 1 changed, 0 unchanged, -1 crossing; writes *b on change.
__device__ __forceinline__ int finish_var(double2* b, double lo, double up, double new_lo,
                                          double new_up, bool integer, const Limits& lim)
{
  if (new_lo > __dadd_rn(new_up, 1e-9)) return -1;
  if (new_lo > new_up) new_lo = new_up;
  const double width = __dsub_rn(up, lo);
  bool changed       = false;
  double wlo = lo, wup = up;
  const double lo_imp = (lo == -INFINITY && new_lo > -INFINITY) ? INFINITY : __dsub_rn(new_lo, lo);
  if (counts_as_change(lo_imp, integer, width, lim)) { wlo = new_lo; changed = true; }
  const double up_imp = (up == INFINITY && new_up < INFINITY) ? INFINITY : __dsub_rn(up, new_up);
  if (counts_as_change(up_imp, integer, width, lim)) { wup = new_up; changed = true; }
  if (changed) *b = make_double2(wlo, wup);
  return changed ? 1 : 0;
}

// Per-variable candidate slot of the fused full round: the minimum upper-bound / maximum
// lower-bound candidate strictly improving on the round-start bound, published with
// order-preserving 64-bit atomics. Equal doubles have equal bits except +-0.0, so the only
// order-dependent case of the reference's std::min/max fold (a tie at zero, first operand kept)
// is resolved by also recording the smallest row (= first CSC position) with a zero candidate
// and that candidate's sign: (row << 1) | signbit.
struct alignas(32) CandSlot {
  unsigned long long lo_key, up_key;
  unsigned lo_zero, up_zero;
  unsigned pad0, pad1;
};
constexpr unsigned long long kLoEmpty = 0ull, kUpEmpty = ~0ull;
constexpr unsigned kZeroEmpty         = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned long long okey(double d)
{
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dekey(unsigned long long k)
{
  const unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)u);
}

// Immutable device problem: the matrix twice (CSR + CSC) plus work-partition tables built once
// at upload (SURVEY §8a A4's LRB bins, re-designed for warps: see DESIGN.md §3).
struct DevProblem {
  int n, m;
  long long nnz;
  const int* row_start;
  const int* row_col;
  const double* row_val;
  const int* row_ci;        // row_col | is_integer(col) << 31 (the fused pass needs integrality)
  const int* col_start;
  const int* col_row;
  const double* col_val;
  const double2* cons;      // (lower, upper) per row
  const uint8_t* is_int;
  // Rows with nnz <= kPackNnz in SELL-32 slices (build: problem_build): n_srtile slices, slice s
  // has 32 rows srow[32 s + i] (-1 padding) and entries sr_ci / sr_val[sr_tile[s] + 32 j + i].
  int n_srow, n_srtile, n_srow_long;  // n_srow_long: leading slices with rows > kShortNnz
  const int* srow;          // slice lane -> row id
  const int* sell_pos;      // row -> 32 * slice + lane for rows in SELL slices (-1 otherwise)
  const int* sr_ptr;        // unused
  const int* sr_ci;         // column | integrality << 31, -1 = padding
  const double* sr_val;
  const uint8_t* sr_own;    // unused
  const int* sr_tile;       // n_srtile + 1 slice offsets
  // Heavy rows (nnz > kHeavyFold): pieces of kPiece entries compute their contributions in
  // parallel and compact the non-zero ones into the min / max contribution streams (+ per-128-
  // chunk aggregates), then one warp per 16384-entry segment streams them and runs the
  // reference's sequential sums: the chain is the only serial part of a round, so it is fed
  // from dense streams.
  const int* long_off;      // per row: 128-aligned offset of its entries in the streams, -1 otherwise
  const int* hpiece;        // per heavy row: index of its first piece in piece_task
  int n_piece;
  const int2* piece_task;   // (row, piece) of heavy rows, longest rows first
  int n_fold, n_fold_heavy;  // n_fold_heavy: leading tasks that are heavy-row segments
  const int2* fold_task;    // (row, segment): heavy-row segments, then medium rows, longest first
  int n_cpiece;
  const int2* cpiece_task;  // (row, piece) candidate tasks of rows with nnz > kCandSplit
  const int* seg_base;      // per row: first partial slot if the row has > 1 segment, else -1
  // Short columns, packed the same way (tile lanes fold one variable each).
  int n_scol, n_sctile;
  const int* scol;
  const int* sc_ptr;
  const int* sc_row;
  const double* sc_val;
  const uint8_t* sc_own;    // owner's local index inside its tile, per packed entry
  const int* sc_tile;
  // Long columns (nnz > kShortNnz), nnz descending: one warp per variable.
  int n_mcol;
  const int* mcol;
  const unsigned long long* reach;  // per var: frontier work a change causes (light, heavy rows)
  const int* col_mark;              // per CSC entry: row task holding it (see problem_build)
  unsigned long long h_reach;       // Σ over heavy rows of their reach (caps the heavy parts)
};

constexpr int kTile      = 128;   // entries per tile / per gathered chunk (4 per lane)
constexpr int kPiece     = 1024;  // gather / candidate piece of a long row (divides kSumSegment)
constexpr int kFoldChunk = 256;   // staging chunk of the streamed fold (8 per lane)
constexpr int kCandSplit = 2048;  // long rows above: candidates by parallel pieces
constexpr int kHeavyFold = 1024;  // rows above: buffered fold (contribution pieces + stream)

// Aggregates of one 128-entry chunk of a heavy row (infinite contributors, gating maxima).
struct ChunkInfo {
  double gtw, gpm;
  int imn, imx;
};
#ifndef BP_PACK_NNZ
#define BP_PACK_NNZ 32
#endif
#ifndef BP_PACK_TILE
#define BP_PACK_TILE 128
#endif
constexpr int kPackNnz   = BP_PACK_NNZ;   // full rounds: rows up to this length go to packed tiles
// The full-round task lists assume the SELL / medium boundary is the short-row boundary
// (problem_build skips rows <= kShortNnz before listing rows > kPackNnz as fold tasks): with
// BP_PACK_NNZ=16, rows of 17-32 entries were in no list and a C2 propagate ended after 23 rounds
// instead of 24. Pinned at compile time.
static_assert(kPackNnz == kShortNnz, "BP_PACK_NNZ must equal kShortNnz (the validated configuration)");
constexpr int kPackTile  = BP_PACK_TILE;  // packed row tiles: <= 32 rows and <= this many entries

// Per heavy-row piece: round-to-nearest sums and absolute sums of its min / max contributions
// (any order), its reach maxima and infinite-contributor counts -- the inputs of the row-level
// quietness certificate that lets a full round skip a heavy row's sequential chains (heavy_fold).
struct PieceAgg {
  double smin, amin, smax, amax;
  double gtw, gpm;
  int imn, imx;
};

struct SegPart {
  double min, max;
  double tmax, pmax;  // row-level candidate gating: max |a|(w + 1), max |a|max(|lo|,|up|)
  int nmin, nmax;
};

}  // namespace bp
