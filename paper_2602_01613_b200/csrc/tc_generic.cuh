// tc_generic.cuh — strided batched contraction step on the tcgen05 tensor cores (tc_generic.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tnl {

// One side (M rows or N columns) of the step: up to three sub-dims, outermost first; `so` is the
// operand's element stride along each sub-dim, `sc` the output's.
struct TcgSide {
  int32_t nd;
  int64_t size[3];
  int64_t so[3];
  int64_t sc[3];
};

//   C[z][m][n] (+)= sum_k A[z][m][k] * B[z][n][k]
struct TcgArgs {
  const __nv_bfloat16* A;
  const __nv_bfloat16* B;
  void* C;  // bf16, or fp32 (c_f32), optionally accumulating
  int32_t c_f32, accumulate;
  int32_t a_vec, b_vec;  // operand rows K-contiguous and 16-byte aligned (vector gathers)
  int64_t M, N, K;
  int64_t ka, kb;  // K strides of A and B
  TcgSide m, n;
  int64_t z1, z2;  // batch (grid.z = z1 * z2) and its strides
  int64_t za1, za2, zb1, zb2, zc1, zc2;
  // split-K (set by launch_tc_generic when the step has few output tiles and a long K): fp32
  // partials into acc32 (dense [z][M][N], zero at rest; >= z1*z2*M*N floats, which is below
  // 74 * 128 * 64 whenever a step splits), then one pass to C
  float* acc32;
  int32_t splits, cps;
};

size_t tc_generic_smem();
int launch_tc_generic(const TcgArgs& a, cudaStream_t st);

}  // namespace tnl
