// tc_gemm_pair.cu — persistent CTA-pair (cta_group::2) variant of the prefill GEMM step.
//
//   D[i][j] = sum_k A[i][k] * B[j][k]      A: activations (M side), B: weights (N side)
//
// Same roles as tc_gemm_persistent.cu (warp 0 TMA ring across tiles, warp 1 MMA issuer into two
// TMEM accumulators, warps 2-5 epilogue), but the two CTAs of a 2x1 cluster compute a 256 x BN
// tile with M=256 tcgen05.mma.cta_group::2 instructions: each CTA loads its own 128 A rows and
// only HALF of the B tile (BN/2 rows). For the rank-256 cut steps (B = a 256 x K panel re-read
// by every 128-token tile, or an output panel re-read by every token tile) the per-token weight
// traffic from L2 halves and one MMA instruction covers both SMs. The leader CTA issues the MMAs
// and owns the full / tempty barriers; MMA completions are multicast to both CTAs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tnl {

namespace {

constexpr int PBM = 128, PBK = 64;
constexpr uint32_t P_A_STAGE = PBM * PBK * 2;
constexpr uint32_t P_C_CHUNK = PBM * 64 * 2;
#ifndef P_NC
#define P_NC 3  // 3 staging buffers: gate r64 prefill 94.4 -> 92.9 us vs 2
#endif

__device__ __forceinline__ void pbar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int BN, int STAGES>
struct PairSmem {
  static constexpr uint32_t B_STAGE = (BN / 2) * PBK * 2;  // this CTA's half of the B tile
  static constexpr int NC = P_NC;  // output staging buffers (TMA stores in flight per CTA)
  static constexpr size_t bytes = 1024 + (size_t)STAGES * (P_A_STAGE + B_STAGE) + NC * P_C_CHUNK + 256;
};

template <int BN, int STAGES, bool SCALE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    tc_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, const TcGemmArgs args, int tiles_m2, int tiles_n,
                        int splits) {
  constexpr uint32_t B_STAGE = PairSmem<BN, STAGES>::B_STAGE;
  constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * P_A_STAGE;
  uint8_t* sC = sB + STAGES * B_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + P_NC * P_C_CHUNK);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2] leader: 4 epilogue warps x 2 CTAs
  uint64_t* afull = tempty + 2;      // [STAGES] ss_fused: stage consumed by the MMAs (multicast commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(afull + STAGES);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int total_kb = (args.K + PBK - 1) / PBK;
  const int kb_per = args.kb_per_split;
  const int num_tiles = tiles_m2 * tiles_n * splits;
  const uint32_t warp = warp_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (args.out_mode == TC_OUT_BF16) tma_prefetch_desc(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SCALE && args.ss_fused ? 5 : 1);  // + 4 epilogue warps reading the A rows
      mbar_init(&afull[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  auto decode_tile = [&](int t, int& tm, int& tn, int& sp) {
    tn = t % tiles_n;
    const int r = t / tiles_n;
    tm = (r % tiles_m2) * 2 + (int)rank;  // this CTA's 128-row tile of the pair's 256 rows
    sp = r / tiles_m2;
  };

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int t = cluster; t < num_tiles; t += nclusters) {
        int tm, tn, sp;
        decode_tile(t, tm, tn, sp);
        const int kb0 = sp * kb_per, kb1 = min(total_kb, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * (P_A_STAGE + B_STAGE));
          tma_load_2d_pair(sA + s * P_A_STAGE, &tmA, &full[s], kb * PBK, tm * PBM);
          tma_load_2d_pair(sB + s * B_STAGE, &tmB, &full[s], kb * PBK, tn * BN + (int)rank * (BN / 2));
        }
      }
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(2 * PBM, BN);
      int it = 0, lt = 0;
      for (int t = cluster; t < num_tiles; t += nclusters, ++lt) {
        int tm, tn, sp;
        decode_tile(t, tm, tn, sp);
        const int kb0 = sp * kb_per, kb1 = min(total_kb, kb0 + kb_per);
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint64_t adesc = smem_desc_sw128(smem_u32(sA + s * P_A_STAGE));
          const uint64_t bdesc = smem_desc_sw128(smem_u32(sB + s * B_STAGE));
#pragma unroll
          for (int k = 0; k < PBK / 16; ++k)
            mma_bf16_ss_pair(d, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          mma_commit_pair(&empty[s], 3);
          if (SCALE && args.ss_fused) mma_commit_pair(&afull[s], 3);
        }
        mma_commit_pair(&tfull[acc], 3);
      }
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3;
    const int et = threadIdx.x - 64;
    int lt = 0, chunk_ct = 0, it_e = 0;
    for (int t = cluster; t < num_tiles; t += nclusters, ++lt) {
      int tm, tn, sp;
      decode_tile(t, tm, tn, sp);
      const int acc = lt & 1;
      float fused_ss = 0.f;
      if (SCALE && args.ss_fused) {  // this CTA's 128 A rows of every k-block: sum this row's squares
        const int kb0 = sp * kb_per, kb1 = min(total_kb, kb0 + kb_per);
        const int lr = (warp & 3) * 32 + lane_id();
        for (int kb = kb0; kb < kb1; ++kb, ++it_e) {
          const int s = it_e % STAGES;
          // only the leader sees the full barriers: wait for the MMA commit of this stage, multicast to
          // both CTAs (the A rows are in our smem; the slot is not refilled before our empty arrival)
          mbar_wait(&afull[s], (it_e / STAGES) & 1);
          fused_ss += tile_row_sumsq(smem_u32(sA + s * P_A_STAGE), lr);
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&empty[s]);
        }
      }
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * BN + ((q * 32) << 16);
      const int lrow = q * 32 + lane_id();
      const int row = tm * PBM + lrow;
      if (args.out_mode == TC_OUT_BF16) {
        const float rscale = !SCALE ? 1.f
                             : args.ss_fused ? rsqrtf(fused_ss / (float)args.rms_n + args.rms_eps)
                                             : row_rms_scale(args, row);
        for (int c0 = 0; c0 < BN; c0 += 64) {
          // Dead chunk (ragged N, or a CTA whose half tile lies past M): skip it entirely so the
          // staging ring advances only on committed stores (wait_read_le<P_NC-1> guards reuse).
          if (tn * BN + c0 >= args.N || tm * PBM >= args.M) {
            if (c0 + 64 >= BN) {
              tc_fence_before();
              __syncwarp();
              if (lane_id() == 0) mbar_arrive_remote(mapa_shared(&tempty[acc], 0));
            }
            continue;
          }
          uint8_t* stage = sC + (chunk_ct % P_NC) * P_C_CHUNK;
          if (et == 0) tma_store_wait_read_le<P_NC - 1>();
          pbar(1, 128);
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
            const int ch = c / 8;
            uint8_t* rowp = stage + (lrow >> 3) * 1024 + (lrow & 7) * 128;
            sts128(smem_u32(rowp) + (((ch) ^ (lrow & 7)) << 4), p0);
            sts128(smem_u32(rowp) + (((ch + 1) ^ (lrow & 7)) << 4), p1);
          }
          if (c0 + 64 >= BN) {
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive_remote(mapa_shared(&tempty[acc], 0));
          }
          fence_proxy_async_smem();
          pbar(1, 128);
          if (et == 0) {
            const int col = tn * BN + c0;
            if (args.reduce_add)
              tma_reduce_add_2d(&tmC, stage, col, tm * PBM);
            else
              tma_store_2d(&tmC, stage, col, tm * PBM);
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
        if (lane_id() == 0) mbar_arrive_remote(mapa_shared(&tempty[acc], 0));
      }
    }
    if (et == 0) tma_store_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_pair<TMEM_COLS>(tmem);
}

template <int BN, int STAGES, bool SCALE>
int launch_pair(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const TcGemmArgs& args,
                int splits, cudaStream_t st) {
  constexpr size_t smem = PairSmem<BN, STAGES>::bytes;
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_pair_kernel<BN, STAGES, SCALE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  const int tiles_m2 = (args.M + 2 * PBM - 1) / (2 * PBM), tiles_n = (args.N + BN - 1) / BN;
  const int tiles = tiles_m2 * tiles_n * splits;
  const int clusters = tiles < 74 ? tiles : 74;  // 148 SMs = 74 CTA pairs
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters, 1, 1);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_pair_kernel<BN, STAGES, SCALE>, a, b, c, args, tiles_m2, tiles_n, splits);
  count_launch();
  return (int)e;
}

}  // namespace

int launch_tc_gemm_pair(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const TcGemmArgs& args,
                        int bn, int splits, cudaStream_t st) {
  switch (bn) {
    case 128:
#ifndef PAIR128_STAGES
#define PAIR128_STAGES 7  // 7 x 24 KB ring: the N-split first steps (q 64.0, o 66.2 us)
#endif
      return (args.ss_in || args.ss_fused) ? launch_pair<128, PAIR128_STAGES, true>(a, b, c, args, splits, st) : launch_pair<128, PAIR128_STAGES, false>(a, b, c, args, splits, st);
    case 256:
      return (args.ss_in || args.ss_fused) ? launch_pair<256, 5, true>(a, b, c, args, splits, st) : launch_pair<256, 5, false>(a, b, c, args, splits, st);
    default:
      return (int)cudaErrorInvalidValue;
  }
}

}  // namespace tnl
