// decode_cluster.cuh — cluster-resident decode chain (decode_cluster.cu, tnl_chain_*).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tnl {

constexpr int CHAIN_CS = 16;  // CTAs per cluster: each owns D/16 rows of every layer

struct CChainArgs {
  const uint8_t* arena;   // [CHAIN_CS][per_cta_bytes]: every CTA's weight blocks in consumption order
  int64_t per_cta_bytes;
  const uint8_t* rq;      // per layer r_pad / 64 (1..4), device
  int32_t n;              // layers (<= 256)
  int32_t rpc;            // rows per CTA = D / 16 (multiple of 64, <= 384)
  int32_t tokens;         // M <= 32
  int32_t nslot;          // ring slots (set by the launcher)
  const __nv_bfloat16* x;  // [tokens][ldx]
  int64_t ldx;
  __nv_bfloat16* y;        // [tokens][ldy]
  int64_t ldy;
  int32_t debug;           // 1: stream weights only (no dependencies, no MMAs) — measurement aid
  long long* trace;        // optional: [16 CTAs][256 layers][8] clock64 stamps (debug)
};

// one arena block: rows x 64 bf16 from src (row-major, ld elements) at (row0, col0) -> SW128
// smem image at arena + dst (rows x 128 B)
struct CChainBlock {
  const __nv_bfloat16* src;
  int64_t ld;
  int32_t row0, col0, rows, pad;
  int64_t dst;
};

int launch_chain(const CChainArgs& a, cudaStream_t st);
int launch_chain_repack(const CChainBlock* blocks_dev, int64_t nblocks, uint8_t* arena, cudaStream_t st);
// clusters of the chain kernel that can be co-resident (0: not launchable on this device)
int chain_max_active_clusters(int rpc, int tokens);

}  // namespace tnl
