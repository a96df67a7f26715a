// tc_gemm_splitk2.cu — split-K over a CTA pair for the narrow first prefill step.
//
//   T (M x N) = X (M x K) . W (N x K)^T      N = the cut rank (<= 64), K = the layer width
//
// With M/128 token tiles (64 at M = 8192) a tile per CTA leaves half the SMs idle, and the
// classic split-K fix costs a zeroing memset of an fp32 buffer, fp32 atomics, and a separate
// conversion pass (three extra launches' worth of latency on the critical path). Here the two
// CTAs of a 2x1 cluster take the two K halves of one tile: CTA 1 ships its fp32 partial (128 x N)
// into CTA 0's shared memory with st.async (distributed shared memory, mbarrier complete_tx),
// CTA 0 adds it to its own accumulator (fixed order: deterministic) and writes the bf16 tile.
//
// Roles: warp 0 TMA producer (STAGES-deep ring), warp 1 MMA issuer (one TMEM accumulator),
// warps 2-5 epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tnl {

namespace {

#ifndef TNL_SK2_STAGES
#define TNL_SK2_STAGES 7
#endif
constexpr int BM = 128, BK = 64, BN = 64, STAGES = TNL_SK2_STAGES;
constexpr uint32_t A_STAGE = BM * BK * 2, B_STAGE = BN * BK * 2;
constexpr uint32_t RBUF = BM * BN * 4;  // CTA 1's fp32 partial, [row][BN]
constexpr size_t SMEM = 1024 + (size_t)STAGES * (A_STAGE + B_STAGE) + RBUF + 256;

__device__ __forceinline__ void st_async16(uint32_t addr, float4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar)
               : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    splitk2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   __nv_bfloat16* __restrict__ out, int64_t ldo, int M, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * A_STAGE;
  float* rbuf = reinterpret_cast<float*>(sB + STAGES * B_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(rbuf) + RBUF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* rfull = tfull + 1;  // CTA 0: the peer's partial landed (tx bytes)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + 1);

  const uint32_t rank = cluster_ctarank();
  const int tile = blockIdx.x >> 1;
  const int tkb = (K + BK - 1) / BK, half = (tkb + 1) / 2;
  const int kb0 = rank ? half : 0, kb1 = rank ? tkb : half;
  const uint32_t warp = warp_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(rfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<64>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers exist before any st.async
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {
      for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
        tma_load_2d(sA + s * A_STAGE, &tmA, &full[s], kb * BK, tile * BM);
        tma_load_2d(sB + s * B_STAGE, &tmB, &full[s], kb * BK, 0);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        const uint64_t ad = smem_desc_sw128(smem_u32(sA + s * A_STAGE));
        const uint64_t bd = smem_desc_sw128(smem_u32(sB + s * B_STAGE));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) mma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
      }
      mma_commit(tfull);
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3;
    const int lrow = q * 32 + lane_id();
    const int row = tile * BM + lrow;
    const uint32_t d = tmem + ((q * 32) << 16);
    if (rank == 0 && threadIdx.x == 64) mbar_arrive_expect_tx(rfull, RBUF);
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (rank == 1) {
      // ship this K half's partial row into CTA 0's receive buffer
      const uint32_t dst = mapa_shared(rbuf, 0) + lrow * BN * 4;
      const uint32_t bar = mapa_shared(rfull, 0);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(d + c, v);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          st_async16(dst + (c + 4 * j) * 4, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]), bar);
      }
    } else {
      mbar_wait_cluster(rfull, 0);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(d + c, v);
        const uint32_t src = smem_u32(rbuf) + (lrow * BN + c) * 4;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 p = lds128f(src + 16 * j);
          v[4 * j] += p.x;
          v[4 * j + 1] += p.y;
          v[4 * j + 2] += p.z;
          v[4 * j + 3] += p.w;
        }
        if (row < M && c < N) {
          uint4* o = reinterpret_cast<uint4*>(out + (int64_t)row * ldo + c);
          o[0] = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                            pack_bf16x2(v[6], v[7]));
          if (c + 8 < N)
            o[1] = make_uint4(pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]), pack_bf16x2(v[12], v[13]),
                              pack_bf16x2(v[14], v[15]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // CTA 0 has consumed the partial before either CTA leaves
  if (warp == 1) tmem_dealloc<64>(tmem);
}

}  // namespace

int launch_tc_gemm_splitk2(const CUtensorMap& a, const CUtensorMap& b, __nv_bfloat16* out, int64_t ldo, int M, int N,
                           int K, cudaStream_t st) {
  if (N > BN || N % 8 || M <= 0) return (int)cudaErrorInvalidValue;
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(splitk2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  const int tiles = (M + BM - 1) / BM;
  return (int)launch_pdl(splitk2_kernel, dim3(2 * tiles), dim3(192), SMEM, st, a, b, out, ldo, M, N, K);
}

}  // namespace tnl
