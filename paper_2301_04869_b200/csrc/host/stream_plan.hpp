// Static step program of the streamed Schur reduction (kernels/reduce_stream.cu).
//
// The per-scenario work of one column tile of K_hat (reduce_group's tile loop,
// kkt.cpp:385-462) is a fixed sequence of *steps*: the level-scheduled
// triangular sweeps of G_x (L, U, U', L'), the dense separator tail, the
// K_xu' T / G_u' Y accumulations and the K~_xx T product.  Every step's data
// (a 32-byte header, its item list, its column indices and its values) is
// laid out contiguously so that a producer warp can stage it into a shared
// memory ring with one or two bulk (TMA) copies ahead of the consumers.  The
// program, the ring placement and the producer's wait distances are computed
// here once per solve; they are the same for every scenario and every tile.
#pragma once

#include <vector>

#include "common.hpp"
#include "plan.hpp"

namespace bipm {

// step kinds (header word 0)
enum StepKind : int {
  kStepScatter = 0,   // X = P G_u V (tile columns), acc += K_uu V
  kStepSweep = 1,     // one level (or part) of a triangular sweep
  kStepDense = 2,     // rows of the dense tail product X_T <- W X_T
  kStepAcc = 3,       // acc -= (K_xu' or G_u') X over a range of control rows
  kStepSpmv = 4,      // S = -(K~_xx X) over a range of state rows
  kStepCopyBack = 5,  // X = S + K_xu V
  kStepDenseG = 6,    // X_T <- W X_T with W read from global memory (L2), one step
  kStepSweepW = 7,    // warp-local levels of a sweep: each warp its own elimination subtrees
  kStepScatterY = 8,  // X = (y_N, X_T) tile columns (presolved forward half, ReachPlan)
  kStepAccTail = 9,   // acc -= X_T' Z_T (all controls, the tile's columns; DMMA, X_T from L2)
  kStepStoreTail = 10,  // Z_T (tail rows of the panel) -> global, for the batch-sum GEMM
};
// kFlagBarrier: consumers synchronise after the step; kFlagPre: before it
enum StepFlag : int { kFlagDiag = 1, kFlagCommit = 2, kFlagBarrier = 4, kFlagPre = 8 };

// Step pattern block: a 64-byte header (16 ints)
//   {kind, flags, n_items, n_col, aux0, aux1, vcount, par, lg, n_units, warp0, n_lev, 0...}
// [warp-local sweeps: a directory of 2 ints per consumer warp = its level
// record range] then n_lev int4 level records (sweep steps), n_items int4 items and n_col
// 16-bit column entries (panel rows; the kernel forms the panel word).  All-warp steps (dense, spmv): a unit is (item, group of up to
// 8 panel columns) served by 2^lg lanes, chunks of 32 >> lg units dealt to
// the 16 consumer warps round robin from warp0.  Sweep steps: aux0 = T, the
// team of the lowest T warps running them; level record = (unit begin, unit
// end, lg, team barrier after it).
constexpr int kStepHeaderInts = 16;
// panel columns per work unit (the kernel's Panel<K>::CW = min(K, this))
constexpr int kStreamUnitCols = 4;  // measured: 8 -> 30.4 ms, 4 -> 28.5 ms, 2 -> 28.9 ms (1354/256)

// Shared-memory panel layout of the K right-hand-side columns: row r is K
// doubles (K*8 bytes) split in 16-byte chunks, chunk c stored at position
// c ^ sw(r) so that lanes gathering different rows spread over the banks.
// word(r) = r*K*8 + 16*sw(r); element (r, c) lives at byte
// (word(r) ^ ((c >> 1) << 4)) + 8 (c & 1)   (K = 1: r*8).
inline int panel_swizzle(int r, int K) {
  return K >= 16 ? (r & 7) : K == 8 ? ((r >> 1) & 3) : K == 4 ? ((r >> 2) & 1) : 0;
}
inline int panel_word(int r, int K) { return r * K * 8 + 16 * panel_swizzle(r, K); }

// row stride of the reduction's padded copy of W, W' (kArrDense): rows start
// on 128-byte lines so the dense step loads 32-byte vectors, 4 lanes per line
inline int dense_ld(int tl) { return (tl + 15) & ~15; }

// value arrays a step can read ([M][stride] scenario-major on the device)
enum ValArray : int {
  kArrSweep = 0,  // sweep-ordered factor values (VS), written by the refactor
  kArrDense = 1,  // W, W' dense tail inverses, rows padded to dense_ld(tl)
  kArrKxx = 2,    // condensed K_xx (CSR slot order)
  kArrKxuT = 3,   // K_xu values in column (control) order
  kArrGuT = 4,    // G_u values in column (control) order
  kArrSigma = 5,  // sigma_x
  kArrYN = 6,     // y_N (ReachPlan, column-major by control)
  kNumValArrays = 7
};

// producer record of one step (12 ints)
struct StepIssue {
  int pat_off;     // int offset of the step's pattern block in `pat`
  int pat_bytes;   // header + items + columns
  int ring_off;    // byte offset of the step in the ring
  int val_arr, val_off, val_count;  // values: array, offset within a scenario, count
  int x_arr, x_off, x_count;        // extra values (sigma_x segment)
  int val_ring, x_ring;             // byte offsets in the ring
  int wait_delta;  // wait until step (j - wait_delta) has been consumed (0: none)
};

struct StreamProgram {
  int K = 1, consumers = 512, ring_bytes = 0, steps = 0;
  std::vector<int> pat;          // pattern blocks (16-byte aligned)
  std::vector<StepIssue> issue;  // per step
  std::vector<int> ring_off;     // per step (consumer lookup)
  // per step: (last control << 4) | pre/post barrier flags of an accumulation
  // step, 0x7ffffff << 4 otherwise.  A column tile starting at j0 assembles
  // only K_hat's lower triangle (u >= j0 + c), so it skips -- neither loads
  // nor runs -- every accumulation step whose controls all lie below j0,
  // keeping the step's barriers
  std::vector<int> skip;
  std::vector<idx> vs_src;       // VS position -> factor slot (F), -1: padding
  idx nnz_vs = 0;
  std::vector<idx> kxu_t_slot, gu_t_slot;  // column-order gathers of K_xu, G_u values
  long long stride[kNumValArrays] = {0, 0, 0, 0, 0, 0, 0};
  int nq = 0;                    // accumulator registers per consumer thread
  int max_step_bytes = 0;
  // statistics
  int n_sweep_steps = 0, n_dense_steps = 0, n_acc_steps = 0, n_spmv_steps = 0;
};

// Subtree-to-warp mapping of the non-tail elimination forest (the sweeps'
// warp-local part): group[row] = consumer warp owning the row, -1 for rows
// left to the team levels (the split nodes above the subtrees, the tail).
// Every subtree is closed under the L / U' (descendants) and U / L'
// (ancestors inside it) dependencies.  nwarps = 0: no warp-local part.
std::vector<int> subtree_groups(const LuPlan& L, int nwarps);

// Forward half of X = G_x^{-1} P G_u solved once per scenario for all n_u
// columns (kernels/reach_gemm.cu), ahead of the streamed reduction:
//   y_N = L_NN^{-1} (P G_u)_N     sparse: column u is nonzero only on the
//                                 reach of its G_u rows in the graph of L
//   y_T = (P G_u)_T - L_TN y_N    the tail rows (dense, ldy per column)
//   X_T = W y_T                   one batched DMMA GEMM (W = (L_TT U_TT)^{-1})
// A column tile of the reduction then starts from (y_N, X_T) instead of
// running the L sweep over all rows and the first dense product per tile:
// the reach of one G_u column is a few etree paths (1354: 63 rows of 2140 per
// 8-column tile), and W is read once per scenario instead of once per tile.
struct ReachPlan {
  idx n_u = 0, t0 = 0, tl = 0, ldy = 0;
  idx nnz_yn = 0;                // y_N entries per scenario (column-major by u)
  std::vector<idx> yn_ptr;       // [n_u + 1]
  std::vector<idx> yn_row;       // permuted state row (< t0) of each entry
  // per column u, ops [op_ptr[u], op_ptr[u+1]) in dependency order:
  // {dest, G_u slot or -1, entry begin, entry end}; dest >= 0: y_N entry
  // yn_ptr[u] + dest, dest < 0: tail row -1 - dest (y_T); entries
  // {source y_N entry (local to the column), factor slot of L}
  std::vector<idx> op_ptr, ops, ent;
  // pattern of y_T: column u is nonzero only on the tail rows its ops write
  // (1354: 27 of 307), so X_T = W y_T is a sparse-dense product
  std::vector<idx> yt_ptr, yt_row;  // [n_u + 1], tail-local rows (ascending)
  long long fmas = 0;            // entries per scenario (work measure)
};
ReachPlan build_reach_plan(const LuPlan& L, const Csr& gu, idx n_u);

// reach != nullptr: the program starts from (y_N, X_T) (ReachPlan) -- a
// scatter of the tile's columns of both, no L sweep, no first dense product.
// adjoint_identity (with reach): the adjoint half ends after the U' sweep.
// With y^ = L^{-1} P G_u and z^ = U^{-T} S,
//   G_u' G_x^{-T} S = y^' z^ = y_N' z_N + X_T' z_T
// (y^_T' U_TT^{-T} = (U_TT^{-1} L_TT^{-1} y_T)' = X_T'), so the W' product,
// the L' sweep and the G_u' Y accumulation become a sparse accumulation over
// y_N's pattern and one dense n_u x tl product against X_T -- inside the tile
// (kStepAccTail), or with defer_tail, Z_T stored (kStepStoreTail) and
// sum_s X_T' Z_T formed by one batch-sum GEMM after the tiles (reach_gemm.cu).
StreamProgram build_stream_program(const LuPlan& L, const Csr& gu, const Csr& kxx, const Csr& kxu,
                                   idx n_u, int K, int consumers, int ring_bytes,
                                   int lookahead_max, const ReachPlan* reach = nullptr,
                                   bool adjoint_identity = false, bool defer_tail = true);

}  // namespace bipm
