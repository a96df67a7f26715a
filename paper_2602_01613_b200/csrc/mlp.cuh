// mlp.cuh — fused middle of a TN Qwen3 MLP block (see mlp.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace tnl {

struct MlpArgs {
  int32_t M;           // tokens
  int32_t inter;       // intermediate width (gate/up rows == down cols), multiple of 64
  int32_t rg, ru, rd;  // padded cut ranks (multiples of 64; rg, ru <= 128, rd <= 256)
  int32_t chunks_per_slice;
  int32_t tiles2;      // CTA-pair kernel: token-pair tiles ((M/128 + 1) / 2)
  int64_t per_pair;    // CTA-pair kernel, balanced mode (> 0): chunk-units per pair of the flattened
                       // (token pair, chunk) sequence; 0: slice mode (chunks_per_slice, grid.y slices)
  float* td;           // fp32 [M][ld_td] partial-sum target (zeroed by the caller)
  int64_t ld_td;
  unsigned long long* trace;  // optional: CTA 0 per-chunk %globaltimer stamps [chunk][4]
};

// t : T_gu bf16 (M x (rg+ru)), box {64, 128} SW128 (k-blocks: rg/64 of T_g then ru/64 of T_u)
// ag: A_g bf16 (inter x rg), box {64, 64} SW128;  au: A_u (inter x ru), box {64, 64} SW128
// bd: B_d bf16 (rd x inter), box {64, rd} SW128
int launch_mlp_mid(const CUtensorMap& t, const CUtensorMap& ag, const CUtensorMap& au,
                   const CUtensorMap& bd, const MlpArgs& a, int slices, cudaStream_t st);
size_t mlp_mid_smem(const MlpArgs& a);
// CTA-pair variant (cta_group::2, 2x1 clusters over token tiles): ag/au box {64, 32}, bd box {64, rd/2}
bool mlp_pair_ok(const MlpArgs& a);
int launch_mlp_mid_pair(const CUtensorMap& t, const CUtensorMap& ag, const CUtensorMap& au,
                        const CUtensorMap& bd, const MlpArgs& a, int slices, cudaStream_t st);

}  // namespace tnl
