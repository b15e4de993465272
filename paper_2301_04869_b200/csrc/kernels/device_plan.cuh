// Device views of the host plans (plain pointers, passed by value).
#pragma once

#include <cstdint>

namespace bipm {

// One triangular sweep (host: SweepPlan in host/plan.hpp).
struct DevSweep {
  const int* col;
  const int* items;       // int4 per item: row, begin, end, 0
  const int* lvl_ptr;     // item ranges per level
  int n_lvl;
  const int* tail_items;  // int4 per tail row (forward sweeps): row, begin, split, 0
  int n_tail;
};

// Static-pivot LU plan of G_x (host: LuPlan in host/plan.hpp).
struct DevLu {
  int n, nnz_l, nnz_f, n_fwd, n_bwd;
  // pivot-growth guard of the static pivot order: a scenario whose factor
  // entries exceed growth * max|G_x| is flagged (status 2) like a singular
  // block (engine.cu; the reference pivots per scenario, linalg.cpp:76-87)
  double growth;
  const int *perm, *iperm;
  const int *l_ptr, *l_col;               // L strict lower, slot == position
  const int *u_ptr, *u_col, *u_slot;      // U strict upper
  const int *diag;
  const int *ut_ptr, *ut_row, *ut_slot;   // column i of U above the diagonal
  const int *lt_ptr, *lt_row, *lt_slot;   // column i of L below the diagonal
  const int *fwd_ptr, *fwd_rows, *bwd_ptr, *bwd_rows;
  const int *lvl_u_ptr, *lvl_u_slot, *lvl_l_ptr, *lvl_l_slot;
  const int *a_src, *piv_of, *mul_ptr, *mul_l, *mul_u;
  // split refactor: non-tail levels, tail-block partial sums (k < t0)
  int n_nt, n_tail_ent;
  const int *nt_lvl_u_ptr, *nt_lvl_u_slot, *nt_lvl_l_ptr, *nt_lvl_l_slot;
  const int *tail_slot, *tail_mul_ptr, *tail_mul_l, *tail_mul_u;
  int rf_nphase;
  const int* rf_phase_ptr;
  const int4* rf_rec;   // {slot, pair begin, pair end, G_x slot or -1}
  const int* rf_piv;    // pivot slot or -1
  const int2* rf_pair;  // (L position, U slot)
  // solve layouts: transposed factor copy and dense tail blocks
  int t0, tl;
  const int* ft_src;     // [nnz_f]
  const int* dense_src;  // [4 tl tl]
  DevSweep sL, sU, sUt, sLt;
};

// A shared CSR pattern with an optional column-major (transposed) view:
// for column c, entries (row t_row[q], slot t_slot[q]) for q in t_ptr[c]..
struct DevCsr {
  int rows, cols, nnz;
  const int *ptr, *ind;
  const int *t_ptr, *t_row, *t_slot;
};

}  // namespace bipm
