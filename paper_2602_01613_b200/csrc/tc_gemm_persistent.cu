// tc_gemm_persistent.cu — persistent warp-specialised tcgen05 GEMM for the prefill steps.
//
//   D[i][j] = sum_k A[i][k] * B[j][k]      A: activations (M side), B: weights (N side)
//
// One CTA per SM loops over output tiles (n fastest so concurrently running
// CTAs share the activation tile in L2). Roles: warp 0 = TMA producer over a
// STAGES-deep smem ring that runs across tile boundaries; warp 1 = MMA issuer
// (tcgen05.mma kind::f16, 128 x BN x 16) into one of TWO TMEM accumulators, so
// the epilogue of tile t overlaps the MMAs of tile t+1; warps 2-5 = epilogue:
// tcgen05.ld -> bf16 -> 128B-swizzled smem staging -> TMA store (64-column
// chunks, two staging buffers in flight), or fp32 vector reductions for split-K.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tnl {

namespace {

constexpr int BM = 128, BK = 64;
constexpr uint32_t A_STAGE = BM * BK * 2;
constexpr uint32_t C_CHUNK = BM * 64 * 2;  // 128 rows x 64 bf16 staging chunk (16 KB)

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int BN, int STAGES>
struct PSmem {
  static constexpr uint32_t B_STAGE = BN * BK * 2;
  static constexpr size_t bytes = 1024 + (size_t)STAGES * (A_STAGE + B_STAGE) + 2 * C_CHUNK + 256;
};

template <int BN, int STAGES, bool SCALE>
__global__ void __launch_bounds__(192, 1)
    tc_gemm_persistent_kernel(const __grid_constant__ CUtensorMap tmA,
                              const __grid_constant__ CUtensorMap tmB,
                              const __grid_constant__ CUtensorMap tmC, const TcGemmArgs args,
                              int tiles_m, int tiles_n, int splits) {
  constexpr uint32_t B_STAGE = PSmem<BN, STAGES>::B_STAGE;
  constexpr uint32_t ACC_COLS = BN;  // two accumulators: [0, BN) and [BN, 2BN)
  constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * A_STAGE;
  uint8_t* sC = sB + STAGES * B_STAGE;  // 2 x 16 KB, 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + 2 * C_CHUNK);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int total_kb = (args.K + BK - 1) / BK;
  const int kb_per = args.kb_per_split;
  const int num_tiles = tiles_m * tiles_n * splits;
  const uint32_t warp = warp_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (args.out_mode == TC_OUT_BF16) tma_prefetch_desc(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SCALE && args.ss_fused ? 5 : 1);  // + 4 epilogue warps reading the A rows
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  auto decode_tile = [&](int t, int& tm, int& tn, int& sp) {
    tn = t % tiles_n;
    const int r = t / tiles_n;
    tm = r % tiles_m;
    sp = r / tiles_m;
  };

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int tm, tn, sp;
        decode_tile(t, tm, tn, sp);
        const int kb0 = sp * kb_per, kb1 = min(total_kb, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
          tma_load_2d(sA + s * A_STAGE, &tmA, &full[s], kb * BK, tm * BM);
          tma_load_2d(sB + s * B_STAGE, &tmB, &full[s], kb * BK, tn * BN);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        int tm, tn, sp;
        decode_tile(t, tm, tn, sp);
        const int kb0 = sp * kb_per, kb1 = min(total_kb, kb0 + kb_per);
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * ACC_COLS;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint64_t adesc = smem_desc_sw128(smem_u32(sA + s * A_STAGE));
          const uint64_t bdesc = smem_desc_sw128(smem_u32(sB + s * B_STAGE));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_ss(d, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3;
    const int et = threadIdx.x - 64;
    int lt = 0, chunk_ct = 0, it_e = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      int tm, tn, sp;
      decode_tile(t, tm, tn, sp);
      const int acc = lt & 1;
      float fused_ss = 0.f;
      if (SCALE && args.ss_fused) {  // the tile's full K streams through the ring: sum this row's squares
        const int kb0 = sp * kb_per, kb1 = min(total_kb, kb0 + kb_per);
        const int lr = (warp & 3) * 32 + lane_id();
        for (int kb = kb0; kb < kb1; ++kb, ++it_e) {
          const int s = it_e % STAGES;
          mbar_wait(&full[s], (it_e / STAGES) & 1);
          fused_ss += tile_row_sumsq(smem_u32(sA + s * A_STAGE), lr);
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&empty[s]);
        }
      }
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * ACC_COLS + ((q * 32) << 16);
      const int lrow = q * 32 + lane_id();
      const int row = tm * BM + lrow;
      if (args.out_mode == TC_OUT_BF16) {
        const float rscale = !SCALE ? 1.f
                             : args.ss_fused ? rsqrtf(fused_ss / (float)args.rms_n + args.rms_eps)
                                             : row_rms_scale(args, row);
        for (int c0 = 0; c0 < BN; c0 += 64) {
          // Dead chunk (ragged N): no TMEM read, no smem write, no store; the staging ring only
          // advances on committed stores so wait_read_le1 always guards the buffer being reused.
          if (tn * BN + c0 >= args.N) {
            if (c0 + 64 >= BN) {
              tc_fence_before();
              __syncwarp();
              if (lane_id() == 0) mbar_arrive(&tempty[acc]);
            }
            continue;
          }
          uint8_t* stage = sC + (chunk_ct & 1) * C_CHUNK;
          // the TMA store that used this staging buffer two chunks ago must have read it
          if (et == 0) tma_store_wait_read_le1();
          named_bar_sync(1, 128);
          uint32_t raw[64];  // the chunk's 64 columns: two loads in flight, one wait
          tmem_ld32_nowait(d + c0, raw);
          tmem_ld32_nowait(d + c0 + 32, raw + 32);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 64; c += 16) {
            float v[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(raw[c + e]);
            if constexpr (SCALE) {  // folded RMSNorm of the step's input rows
#pragma unroll
              for (int e = 0; e < 16; ++e) v[e] *= rscale;
            }
            uint4 p0, p1;
            p0.x = pack_bf16x2(v[0], v[1]);
            p0.y = pack_bf16x2(v[2], v[3]);
            p0.z = pack_bf16x2(v[4], v[5]);
            p0.w = pack_bf16x2(v[6], v[7]);
            p1.x = pack_bf16x2(v[8], v[9]);
            p1.y = pack_bf16x2(v[10], v[11]);
            p1.z = pack_bf16x2(v[12], v[13]);
            p1.w = pack_bf16x2(v[14], v[15]);
            const int ch = c / 8;  // 16-byte chunk index within the 128-byte row
            uint8_t* rowp = stage + (lrow >> 3) * 1024 + (lrow & 7) * 128;
            sts128(smem_u32(rowp) + (((ch) ^ (lrow & 7)) << 4), p0);
            sts128(smem_u32(rowp) + (((ch + 1) ^ (lrow & 7)) << 4), p1);
          }
          if (c0 + 64 >= BN) {  // all TMEM reads of this accumulator are done
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&tempty[acc]);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (et == 0) {
            const int col = tn * BN + c0;
            if (args.reduce_add)
              tma_reduce_add_2d(&tmC, stage, col, tm * BM);
            else
              tma_store_2d(&tmC, stage, col, tm * BM);
            tma_store_commit();
          }
          ++chunk_ct;
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16(d + c, v);
          const int col0 = tn * BN + c;
          if (row < args.M && col0 < args.N) {
            const int n = min(16, args.N - col0);
            float* o = static_cast<float*>(args.out) + (int64_t)row * args.ldo_i + col0;
            if (n == 16) {
#pragma unroll
              for (int e = 0; e < 16; e += 4) red_add_v4(o + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (e < n) atomicAdd(o + e, v[e]);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&tempty[acc]);
      }
    }
    if (et == 0) tma_store_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

template <int BN, int STAGES, bool SCALE>
int launch_p(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const TcGemmArgs& args,
             int splits, int max_ctas, bool pdl, cudaStream_t st) {
  constexpr size_t smem = PSmem<BN, STAGES>::bytes;
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_persistent_kernel<BN, STAGES, SCALE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  const int tiles_m = (args.M + BM - 1) / BM, tiles_n = (args.N + BN - 1) / BN;
  const int tiles = tiles_m * tiles_n * splits;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles < max_ctas ? tiles : max_ctas, 1, 1);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_persistent_kernel<BN, STAGES, SCALE>, a, b, c, args, tiles_m,
                                     tiles_n, splits);
  count_launch();
  return (int)e;
}

}  // namespace

int launch_tc_gemm_persistent(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                              const TcGemmArgs& args, int bn, int splits, int max_ctas, bool pdl,
                              cudaStream_t st) {
  switch (bn) {
    case 64:
      return (args.ss_in || args.ss_fused) ? launch_p<64, 8, true>(a, b, c, args, splits, max_ctas, pdl, st) : launch_p<64, 8, false>(a, b, c, args, splits, max_ctas, pdl, st);
    case 128:
#ifndef P128_STAGES
#define P128_STAGES 6  // 6 x 32 KB ring (225 KB with the staging): q / o first steps 66.7 -> 65.6 us
#endif
      return (args.ss_in || args.ss_fused) ? launch_p<128, P128_STAGES, true>(a, b, c, args, splits, max_ctas, pdl, st) : launch_p<128, P128_STAGES, false>(a, b, c, args, splits, max_ctas, pdl, st);
    case 256:
      return (args.ss_in || args.ss_fused) ? launch_p<256, 3, true>(a, b, c, args, splits, max_ctas, pdl, st) : launch_p<256, 3, false>(a, b, c, args, splits, max_ctas, pdl, st);
    default:
      return (int)cudaErrorInvalidValue;
  }
}

}  // namespace tnl
