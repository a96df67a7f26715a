// generic.cuh — CUDA-core strided batched contraction step (exact FFMA, fp32 accumulate).
//
// One step of a TN contraction chain:
//   C[b1][b2][i][j] = sum_p A[b1][b2][i][p] * B[b1][b2][p][j]
// with an independent element stride for every index of every operand. Every
// pairwise contraction of the reference (np.tensordot in tensor_core.py:109,130
// and tn_decompositions.py:358) maps onto one such step once the plan has
// permuted the cores into a convenient layout (see tnl_api.cu build_*_steps).
#pragma once
#include <cstdint>

namespace tnl {

enum DType : int32_t { DT_F32 = 0, DT_BF16 = 1 };

struct GStep {
  int64_t b1, b2, I, J, P;
  const void* A;
  int64_t sa1, sa2, sai, sap;
  const void* B;
  int64_t sb1, sb2, sbp, sbj;
  void* C;
  int64_t sc1, sc2, sci, scj;
  int32_t a_dt, b_dt, c_dt;
  int32_t accumulate;  // C += result (fp32 C only)
};

// Folds batch dims into I where the strides allow (keeps GEMV-shaped steps
// from wasting 64x64 tiles), then launches. Returns cudaError_t as int.
int launch_generic_step(const GStep& s, cudaStream_t stream);

// Plan building runs with split-K disabled (fixed summation order), so a plan's panels do not
// depend on its row range: output-sharded plans reproduce the full plan's rows bit for bit.
void set_generic_deterministic(bool on);

}  // namespace tnl
