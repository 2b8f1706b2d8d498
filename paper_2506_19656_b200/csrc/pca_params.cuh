// Band-PCA model passed by value in the kernel parameter block, so the
// per-pixel projections read it as uniform constant-bank operands.
#pragma once
#include "common.cuh"

namespace cvb {

struct PcaParams {
  int C;  // input channels
  int K;  // kept components
  double mean[kMaxC];
  double W[kMaxC * kMaxC];  // [K][kMaxC] (row stride kMaxC)
};

// pc_j = sum_c (x_c - mean_c) * W[j][c], fixed order with explicit fma so
// every kernel that projects produces bit-identical components
// (transform.py:199 computes the same product with BLAS).
__device__ __forceinline__ double project_one(const double *d, const PcaParams &p, int j) {
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < kMaxC; ++c)
    if (c < p.C) acc = __fma_rn(d[c], p.W[j * kMaxC + c], acc);
  return acc;
}

int make_pca_params(PcaParams &p, const double *mean, const double *comps, int K, int C);

}  // namespace cvb
