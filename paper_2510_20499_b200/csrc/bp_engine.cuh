// Host-side engine objects shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "bp_device.cuh"

namespace bp {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define BP_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      throw ::bp::cuda_error(std::string(#x) + ": " + cudaGetErrorString(e_) + " (" +       \
                             __FILE__ + ":" + std::to_string(__LINE__) + ")");              \
  } while (0)

// Owning device allocation.
template <class T>
struct DBuf {
  T* p       = nullptr;
  size_t n   = 0;
  DBuf()     = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { reset(); }
  void reset()
  {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count)
  {
    reset();
    n = count;
    if (count) BP_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void upload(const T* src, size_t count)
  {
    alloc(count);
    if (count) BP_CUDA(cudaMemcpy(p, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  }
  void upload(const std::vector<T>& v) { upload(v.data(), v.size()); }
};

// Per-round frontier/counter block (double-buffered by round parity).
struct ParCtl {
  int n_drow_s, n_dpiece, n_dfold, n_drow_all;  // staged together (stage_rows)
  int n_dvar_s, n_dvar_m;                       // staged together (stage_vars)
  int n_changed, n_crossed, any_rows;
  int cur_a, cur_b, cur_c, cur_vm, cur_vs;
  int cur_x1, cur_x2, n_xtask, stop;
  int n_ctask, cur_x3, cur_x4, xabort;  // xabort: a frontier expansion stopped early (full next)
  int cur_p, cur_s, cur_g, pad4;        // full rounds: heavy-row pieces, long SELL slices, medium-row groups
  unsigned long long colnnz, roww, colw, reach, hreach;
};

constexpr int kMaxMultiCursors = 8;

struct Ctl {
  ParCtl par[2];
  int status, rounds, crossed, any_change;
  int fixpoint;  // 1 if the loop ended at a fixpoint (no change / no dirty row): certifies the bounds
  // hand-off of a full round's row phase to k_rows_full (engine state kept across launches)
  int need_full;              // the engine exited to have round `rounds` run its F2 externally
  unsigned stamp_base;        // stamp base of the running propagate (for the hand-off launches)
  // Dirty-filtered full rounds: 0 = the handed-over round is a true full round;
  // otherwise only rows with row_stamp == df_stamp (rows of the vars changed last round) are
  // recomputed and publish candidates, the candidate slots of unchanged vars persisting.
  unsigned df_stamp;
  int df_cnt[4];  // dirty lists of a dirty-filtered round: slices, medium-row groups, heavy pieces,
                  // and the dirty rows of SELL slices
  int stale;      // some heavy row's activity record is stale (certified quiet, chain skipped)
  int n_touch;    // variables whose slot a dirty-filtered round's rows published into (touched)
  unsigned long long t0;      // globaltimer at the start of the propagate (time limit, stats)
  int pad[2];
  // full rounds: per parity, kMaxMultiCursors work cursors for the medium-row groups, each on its
  // own 128-byte line (zeroed with the rest of Ctl per call, the next parity's per round)
  alignas(128) int mcur[2 * kMaxMultiCursors * 32];
};

// Mutable per-problem workspace (one propagate at a time per problem; calls serialized).
struct DevState {
  double2* bounds;
  RowRec* rec;
  double2* aux;
  // heavy rows' contribution streams (DevProblem::long_off): per piece, its non-zero min / max
  // contributions compacted in entry order at off + first entry of the piece; counts in pcnt
  double* gmin;
  double* gmax;
  int2* pcnt;
  PieceAgg* pagg;   // per piece: the quietness-certificate aggregates
  unsigned* sfold;  // per heavy segment (at its first piece): stamp of its last exact fold
  CandSlot* slot;     // fused full round: per-var candidate slots
  // Candidate-slot state, kept across calls (outside Ctl, which callers zero per call): 0 = all
  // empty, 1 = valid for the current bounds (left by a full or dirty-filtered round's finalize:
  // every unchanged var's slot holds its exact fold), 2 = stale (cleared before the next true full
  // round).
  int* slot_state;
  unsigned* ready;    // per row: stamp of the round whose activity is published
  unsigned char* rquiet;  // per row: 1 if no entry can publish a candidate (set before `ready`)
  ChunkInfo* cinfo;       // heavy rows: per 128-entry chunk of the row
  unsigned* pstamp;       // per heavy-row piece: stamp of the round whose contributions are in gmin/gmax
  unsigned* piece_dirty;  // per heavy-row piece: stamp of the dirty-filtered round that recomputes it
  double2* ckpt;          // per heavy-row piece: (min, max) running sums of its segment before it
  unsigned* task_stamp;   // per SELL slice / medium-row group: stamp of the dirty-filtered round
  int n_task;             // SELL slices + medium-row groups
  unsigned char* row_flag;  // per light row: low byte of the dirty-filtered round's mark
  int* df_slice;          // dirty lists (phase_df_lists)
  int* df_group;
  int* df_piece;
  int* df_rows;           // dirty rows of SELL slices (appended by the marking, deduplicated by sell_stamp)
  unsigned* sell_stamp;   // per row: stamp of the marking that listed it (its own array: the frontier
                          // expansion stamps row_stamp with the same round stamp)
  unsigned* vtouch;       // per var: dirty-filtered round stamp of its first publish (touched list)
  int* touched;           // the touched variables of the running dirty-filtered round
  SegPart* seg_part;
  int* seg_done;
  unsigned* row_stamp;
  unsigned* var_stamp;
  int* drow_s[2];
  int2* dpiece[2];  // (row, piece) gather tasks of dirty long rows
  int2* dfold[2];   // (row, segment) fold tasks of dirty long rows
  int2* xtask[2];   // (row, kTile-entry chunk) var-expansion tasks of dirty long rows
  int* dvar_s[2];
  int* dvar_m[2];
  int* changed;
  int2* ctask;      // (var, kTile-entry column chunk) row-expansion tasks of the changed vars
  Ctl* ctl;
  unsigned long long* dbg;  // optional debug counters (BP_DEBUG=1)
};

enum Mode { MODE_PROPAGATE = 0, MODE_ACTIVITY = 1, MODE_TIGHTEN = 2 };

struct Problem {
  int device = 0;
  int n = 0, m = 0;
  long long nnz = 0;
  // host copies kept for classification of caller-supplied lists
  std::vector<int> h_row_start, h_col_start;
  std::vector<int> h_hpiece;  // first contribution piece of each heavy row (-1 otherwise)
  // device arrays: the matrix twice
  DBuf<int> row_start, row_col, row_ci, col_start, col_row;
  DBuf<double> row_val, col_val;
  DBuf<double2> cons;
  DBuf<uint8_t> is_int;
  // partition tables (see DevProblem)
  DBuf<int> srow, sr_ptr, sr_ci, sr_tile;
  DBuf<double> sr_val;
  DBuf<uint8_t> sr_own;
  DBuf<int> long_off, hpiece;
  DBuf<ChunkInfo> cinfo;
  DBuf<unsigned> pstamp, piece_dirty;
  DBuf<double2> ckpt;
  DBuf<int> col_mark;
  DBuf<unsigned> task_stamp;
  DBuf<int> df_lists;
  DBuf<int> df_rows;
  DBuf<unsigned> sell_stamp;
  DBuf<unsigned> vtouch;
  DBuf<int> touched;
  DBuf<int> sell_pos;
  DBuf<unsigned char> row_flag;
  int n_task = 0;
  DBuf<int2> piece_task, fold_task, cpiece_task;
  DBuf<int> scol, sc_ptr, sc_row, sc_tile;
  DBuf<double> sc_val;
  DBuf<uint8_t> sc_own;
  DBuf<int> seg_base, mcol;
  DBuf<unsigned long long> reach;
  unsigned long long h_reach = 0;
  int n_srow_long = 0;
  int n_srow = 0, n_srtile = 0, n_scol = 0, n_sctile = 0, n_mcol = 0, n_part = 0;
  int n_piece = 0, n_fold = 0, n_cpiece = 0, n_fold_heavy = 0;
  long long n_long_entries = 0;
  // workspace
  DBuf<double2> bounds;
  DBuf<RowRec> rec;
  DBuf<double2> aux;
  DBuf<double2> gbuf;  // storage of gmin / gmax (n_long_entries doubles each)
  DBuf<int2> pcnt;
  DBuf<PieceAgg> pagg;
  DBuf<unsigned> sfold;
  DBuf<CandSlot> slot;
  DBuf<int> slot_state;
  DBuf<unsigned> ready;
  DBuf<unsigned char> rquiet;
  DBuf<SegPart> seg_part;
  DBuf<int> seg_done;
  DBuf<unsigned> row_stamp, var_stamp;
  DBuf<int> lists_i;  // backing store for int lists
  DBuf<int2> lists_i2;
  DBuf<Ctl> ctl;
  DBuf<unsigned long long> dbg;
  DevState st{};
  unsigned stamp_base = 1;
  int grid_blocks = 0;
  int f2_blocks   = 0;  // k_rows_full grid (its own occupancy)
  int sell_blocks = 0;  // k_rows_sell grid (its own occupancy)
  std::shared_ptr<void> probe_ws;  // probing scratch (device + pinned host), kept across calls
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // bracket every engine launch on its stream
  double last_kernel_ms = 0.0;
  double total_kernel_ms = 0.0;
  long long n_launch = 0;
  std::mutex mu;

  DevProblem dev() const;
};

void problem_build(Problem& P, int n, int m, const int* row_start, const int* row_col,
                   const double* row_val, const int* col_start, const int* col_row,
                   const double* col_val, const double* var_lower, const double* var_upper,
                   const uint8_t* is_integer, const double* cons_lower, const double* cons_upper);

struct RunResult {
  int status, rounds, crossed, fixpoint;
};

// flags: ENGINE_FORCE_FRONTIER never substitutes a full round for a large frontier (the exact
// reference trajectory of dirty sets, used to count its work); stats (device, kStatCols per round)
// receives per-round work counts when non-null.
// ENGINE_START_FRONTIER: the bounds are a certified fixpoint except for the variables staged in
// par[0]'s changed list (stage_changed); round 1 starts from their frontier.
enum { ENGINE_FORCE_FRONTIER = 1, ENGINE_START_FRONTIER = 2 };
// full, |R|, row nnz visits, |V|, col nnz visits, |changed|, then phase-end times (ns since
// kernel start): activity, tightening, row expansion, var expansion, gather; one spare
constexpr int kStatCols = 12;
RunResult run_engine(Problem& P, Mode mode, bool full, const Limits& lim, cudaStream_t s,
                     int flags = 0, long long* d_stats = nullptr);

// Stage caller row/var lists into the parity-1 frontier buffers (host-classified).
void stage_rows(Problem& P, const int* rows, int nrows, cudaStream_t s);
void stage_vars(Problem& P, const int* vars, int nvars, cudaStream_t s);
// Stage the changed-variable list of a frontier start (ENGINE_START_FRONTIER).
void stage_changed(Problem& P, const int* vars, int nvars, cudaStream_t s);

extern std::atomic<long long> g_kernel_launches;  // host threads may drive problems concurrently

}  // namespace bp
