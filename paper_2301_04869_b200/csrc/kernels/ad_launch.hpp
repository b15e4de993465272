#pragma once

#include <cuda_runtime.h>

#include "ad_kernels.cuh"

namespace bipm {

// eval_bundle_range (autodiff.cpp:484-516): f, g, h, G_x, G_u, H_x, H_u,
// W_xx, W_xu, W_uu and grad_lag for every owned scenario.
void launch_ad_bundle(const DevAd& A, const AdBuffers& b, cudaStream_t st);
// batch_eval (autodiff.cpp:256-281): f, g, h only (line-search trials).
void launch_ad_values(const DevAd& A, const AdBuffers& b, cudaStream_t st);

}  // namespace bipm
