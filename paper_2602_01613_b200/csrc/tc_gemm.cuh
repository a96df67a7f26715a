// tc_gemm.cuh — tcgen05/TMEM/TMA GEMM step: D[i][j] = sum_k A[i][k] * B[j][k].
//
// A ("M side", 128-row tiles) and B ("N side", BN-row tiles) are bf16 K-major
// matrices described by 2-D TMA tensor maps (128B swizzle, 64-element K boxes).
// D accumulates in fp32 in TMEM and is written to out[i*ldo_i + j*ldo_j] as
// bf16, fp32, or fp32 atomic adds (split-K). Used for every dense contraction
// step of the bf16 plans: merged-cut (X.B_in^T, T.A_out^T), the Tucker-2 chain
// (X.U1, T1.G^T, T2.U0^T) and dense layers; in "swap-AB" form (A = weight
// panel, B = activations) for small-M decode.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tnl {

enum TcOutMode : int32_t { TC_OUT_BF16 = 0, TC_OUT_F32_ATOMIC = 1, TC_OUT_F32 = 2 };

struct TcGemmArgs {
  int32_t M, N, K;
  int32_t kb_per_split;  // K blocks (of 64) per blockIdx.z
  void* out;
  int64_t ldo_i, ldo_j;
  int32_t out_mode;
  // bf16 epilogue of the persistent / pair kernels (decoder-stack folds, tnl_fwd_opts):
  int32_t reduce_add = 0;        // out += D (TMA bulk reduce-add at L2) instead of out = D
  const float* ss_in = nullptr;  // D row i scaled by rsqrt(ss_in[i] / rms_n + rms_eps) (folded RMSNorm)
  int32_t rms_n = 0;
  float rms_eps = 0.f;
  // ss_fused (with ss_in set to any non-null marker): the kernel computes sum_k A[i][k]^2 itself
  // from the A tiles streaming through shared memory (full K per tile, no split-K) — the epilogue
  // warps read each stage's own row before releasing it — instead of reading ss_in
  int32_t ss_fused = 0;
};

// sum of squares of row `lrow` of a 128 x 64 bf16 SW128 tile in shared memory
__device__ __forceinline__ float tile_row_sumsq(uint32_t tile_saddr, int lrow) {
  const uint32_t rowp = tile_saddr + (lrow >> 3) * 1024 + (lrow & 7) * 128;
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(rowp + ((c ^ (lrow & 7)) << 4)));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float lo = __uint_as_float(w[t] << 16), hi = __uint_as_float(w[t] & 0xffff0000u);
      s = fmaf(lo, lo, fmaf(hi, hi, s));
    }
  }
  return s;
}

// Epilogue helper shared by the persistent and pair kernels (bf16 output mode): the folded-RMSNorm
// scale of output row `row`.
__device__ __forceinline__ float row_rms_scale(const TcGemmArgs& a, int row) {
  if (!a.ss_in || row >= a.M) return 1.f;
  return rsqrtf(__ldcg(a.ss_in + row) / (float)a.rms_n + a.rms_eps);
}

// dual_gemm.cu: h (M x N) = silu(T[:, :kg] A_g^T) * (T[:, u_off : u_off + ku] A_u^T), bf16.
struct DualArgs {
  int32_t M, N;      // tokens, intermediate width (multiple of 64)
  int32_t kg, ku;    // contraction lengths (cut ranks, zero-padded by TMA to 64)
  int32_t u_off;     // column of T where the up block starts
};
// t: T map (box {64, 128}); g / u: A_g / A_u maps (box {64, 64}: each CTA of a pair loads half the
// rows of an output tile); h: output map (box {64, 128}, SW128). 2x1 clusters over token tiles.
int launch_dual_silu(const CUtensorMap& t, const CUtensorMap& g, const CUtensorMap& u, const CUtensorMap& h,
                     const DualArgs& a, cudaStream_t st);
bool dual_silu_ok(const DualArgs& a);  // kg + ku <= 512 (resident T tile), N % 64 == 0

// Encodes a 2-D bf16 K-major tensor map: `rows` rows of `k` elements with a
// row pitch of `ld` elements, boxes of 64 (K) x box_rows. Returns 0 on success.
int make_tmap_bf16(CUtensorMap* map, const void* base, int64_t k, int64_t rows, int64_t ld,
                   int box_rows);

// General 2-D map: `outer` rows of `inner` elements (bf16 or fp32), row pitch `ld`
// elements, box (box_inner x box_outer), swizzle 0 / 32 / 64 / 128 bytes.
int make_tmap_2d(CUtensorMap* map, const void* base, bool f32, int64_t inner, int64_t outer,
                 int64_t ld, int box_inner, int box_outer, int swizzle_bytes);

// bn in {16,32,64,128,256}; splits >= 1 (grid.z). Returns cudaError_t as int.
int launch_tc_gemm(const CUtensorMap& a, const CUtensorMap& b, const TcGemmArgs& args, int bn,
                   int splits, bool pdl, cudaStream_t stream);

// Persistent variant (prefill): grid = min(tiles, max_ctas); bn in {64,128,256}.
// out_mode TC_OUT_BF16 stores through TMA map `c` (out: M x N bf16, box {64, 128},
// 128B swizzle); TC_OUT_F32_ATOMIC reduces into args.out (row-major fp32, ldo_i).
int launch_tc_gemm_persistent(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                              const TcGemmArgs& args, int bn, int splits, int max_ctas, bool pdl,
                              cudaStream_t st);

// Split-K over a 2-CTA cluster (tc_gemm_splitk2.cu): out (M x N bf16, N <= 64, N % 8 == 0) =
// A (M x K) . B (N x K)^T; CTA 1 ships its K-half partial to CTA 0 over DSMEM (no fp32 buffer, no
// memset, no conversion pass). a: box {64, 128}; b: box {64, 64}.
int launch_tc_gemm_splitk2(const CUtensorMap& a, const CUtensorMap& b, __nv_bfloat16* out, int64_t ldo, int M, int N,
                           int K, cudaStream_t st);

// CTA-pair variant (tc_gemm_pair.cu): 256 x bn tiles over 2x1 clusters, bn in {128, 256};
// `b` must be a map with box {64, bn / 2} (each CTA loads half of the B tile).
int launch_tc_gemm_pair(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const TcGemmArgs& args,
                        int bn, int splits, cudaStream_t st);

}  // namespace tnl
