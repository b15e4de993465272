// Device view of the AD program (host/ad_plan.hpp) and the model constants.
#pragma once

namespace bipm {

struct DevGather {
  int n;
  const int *ptr, *src;
  const double* coef;  // may be null: all coefficients 1
};

struct DevAd {
  int M, nbus, nbr, ngen, n_x, n_u, m, n_b, n_d;
  int ref_bus, slack_gen;
  int vv, br, sq, pd, qd, pg, pg2;  // lane offsets
  const int *vmag_in, *pgen_in;
  const int *br_th, *br_v;  // per branch: theta inputs (from, to; -1 at ref), |v| inputs
  double gs_ref;
  const double* brc;  // per branch: gff bff gft bft gtf btf gtt btt
  const int *br_ref, *gen_ref_other;
  const double *pd_v, *qd_v, *status;  // element-major: [nbus][M], [nbus][M], [nbr][M]
  const int *Lf_ptr, *Lf_ind, *Lg_ptr, *Lg_ind, *Lh_ptr, *Lh_ind;
  const double *Lf_val, *Lg_val, *Lh_val;
  int n_dp, n_c, c_bus, c_gen, c_slack, nsd;
  const int *dp_off, *sd;
  DevGather slack_val, slack_grad, w, gx, gu, hx, hu, grad, wxx, wxu, wuu;
};

// Per-call buffers.  Inputs are scenario-major over the engine's M scenarios.
struct AdBuffers {
  const double *X, *u, *Y, *Z;  // [M][n_x], [n_u], [M][n_x], [M][m]
  double obj_w;
  double *Xt, *Yt, *Zt;         // element-major copies of X, Y, Z (scratch)
  double *psi, *dp, *w, *c;     // element-major scratch: [n_b][M], [n_dp][M], [n_b][M], [n_c][M]
  double *f, *g, *h;            // [M], [M][n_x], [M][m]
  double *gx, *gu, *hx, *hu, *wxx, *wxu, *wuu, *grad;  // [M][nnz], grad [M][n_d]
  int* bad;                     // [M] non-finite flags
};

}  // namespace bipm
