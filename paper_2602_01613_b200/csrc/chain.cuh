// chain.cuh — core-by-core TT/TR input chain on tcgen05 (two input modes).
//
// For a TT/TR layer whose input side has two modes (n_a, n_b) — cores
// C (b, n_a, c) and D (c, n_b, alpha) — the cut state per token is
//   t1[m, j_a, (alpha, c)] = sum_{j_b} x[m, j_a, j_b] D[c, j_b, alpha]          (MMA1)
//   T [m, (alpha, b)]     += sum_{c}   t1[m, j_a, (alpha, c)] C[b, j_a, c]      (MMA2)
// summed over j_a (TT: alpha = 1; TR: alpha = closure r0).
// Per 128-token tile the kernel streams j_a: TMA brings x[:, j_a, :] (SW32
// chunks of 16 along j_b) and C[:, j_a, :]; MMA1 accumulates t1 in TMEM;
// the epilogue warps round t1 to bf16 into a 128B-swizzled smem operand;
// MMA2 (one per closure index alpha) accumulates T in a second TMEM region.
// t1 never leaves the SM; only T (M x r_cut) is written (bf16, or fp32
// reductions when j_a is split across CTAs).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tnl {

struct ChainArgs {
  int32_t M;          // tokens
  int32_t n_a, n_b;   // input modes (j_a outer, j_b inner): cols = n_a * n_b
  int32_t r0;         // closure (alpha) size, 1 for TT
  int32_t c, c_pad;   // bond between C and D (c_pad in {16, 32, 64})
  int32_t b, b_pad;   // cut bond (left bond of C), b_pad multiple of 16
  int32_t ja_per_split;
  // output: T[m][alpha*b + bb]
  void* out;
  int64_t s_m, s_k;   // element strides of (token, kappa)
  int32_t out_f32_atomic;  // 0: bf16 store, 1: fp32 reductions
};

// x map: bf16 (cols inner, M outer), box {16, 128}, 32B swizzle
// d map: Dp [(alpha, c_pad)][n_b] bf16, box {16, r0*c_pad}, 32B swizzle
// c map: Cp [n_a * b_pad][c_pad] bf16, box {c_pad, b_pad}, swizzle = 2*c_pad bytes
int launch_chain_in2(const CUtensorMap& x, const CUtensorMap& d, const CUtensorMap& c,
                     const ChainArgs& a, int splits, cudaStream_t st);

}  // namespace tnl
