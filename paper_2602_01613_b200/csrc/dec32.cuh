// dec32.cuh — small-M fp32 merged-cut forward on CUDA cores (dec32.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace tnl {

constexpr int kDec32MaxCut = 256;

// y (M x rows, ldy) = (x (M x K, ldx) . B_in^T) . A_out^T, fp32, M <= 32, r_cut <= kDec32MaxCut.
// t: zero-at-rest fp32 accumulator (>= 32 * r_cut floats), counter: zero-at-rest.
int launch_dec32(const float* bin, int64_t ldb, const float* aout, int64_t lda, int rows, int r_cut, int K,
                 const float* x, int64_t ldx, int M, float* y, int64_t ldy, float* t, unsigned int* counter,
                 cudaStream_t st);

}  // namespace tnl
