// chain.cu — tcgen05 core-by-core input chain for two-mode TT/TR input sides (see chain.cuh).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "chain.cuh"
#include "common.cuh"
#include "ptx.cuh"

namespace tnl {

namespace {

constexpr uint32_t T1_CHUNK = 128 * 64 * 2;  // 128 tokens x 64 bf16, SW128 (16 KB)
constexpr uint32_t XCHUNK = 128 * 16 * 2;    // 128 tokens x 16 bf16, SW32 (4 KB)

// K-major smem descriptor with an explicit swizzle: layout 6 = 32B, 4 = 64B, 2 = 128B;
// SBO = 8 rows x row bytes.
__device__ __forceinline__ uint64_t smem_desc_sw(uint32_t saddr, uint32_t layout, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

struct ChainLayout {
  uint32_t d_bytes, t1_bytes, x_bytes, c_bytes, c_tx, stage_bytes;
  int stages;
  size_t total;
};

__host__ __device__ inline ChainLayout chain_layout(const ChainArgs& a) {
  ChainLayout L;
  const uint32_t n1 = a.r0 * a.c_pad;
  L.d_bytes = ((n1 * a.n_b * 2 + 1023) / 1024) * 1024;
  L.t1_bytes = ((n1 + 63) / 64) * T1_CHUNK;
  L.x_bytes = (a.n_b / 16) * XCHUNK;
  L.c_tx = a.b_pad * a.c_pad * 2;
  L.c_bytes = ((L.c_tx + 1023) / 1024) * 1024;
  L.stage_bytes = L.x_bytes + L.c_bytes;
  const size_t fixed = 1024 + L.d_bytes + L.t1_bytes + 256;
  int s = 4;
  while (s > 1 && fixed + (size_t)s * L.stage_bytes > 227 * 1024) --s;
  L.stages = s;
  L.total = fixed + (size_t)s * L.stage_bytes;
  return L;
}

__global__ void __launch_bounds__(192, 1)
    chain_in2_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmD,
                     const __grid_constant__ CUtensorMap tmC, const ChainArgs a) {
  const ChainLayout L = chain_layout(a);
  const int S = L.stages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sD = smem;
  uint8_t* sT1 = sD + L.d_bytes;
  uint8_t* sStage = sT1 + L.t1_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + (size_t)S * L.stage_bytes);
  uint64_t* full = bars;          // [S]
  uint64_t* empty = bars + 4;     // [S]
  uint64_t* dfull = bars + 8;
  uint64_t* d1_full = bars + 9;
  uint64_t* d1_free = bars + 10;
  uint64_t* t1_full = bars + 11;
  uint64_t* t1_free = bars + 12;
  uint64_t* d2_done = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int n1 = a.r0 * a.c_pad;
  const int nq = a.n_b / 16;  // j_b chunks of 16
  const int tile_m = blockIdx.x;
  const int ja0 = blockIdx.y * a.ja_per_split;
  const int nja = min(a.n_a, ja0 + a.ja_per_split) - ja0;
  const uint32_t warp = warp_id();
  // B-operand (C_j) swizzle by its row bytes
  const uint32_t c_layout = a.c_pad == 16 ? 6u : (a.c_pad == 32 ? 4u : 2u);
  const uint32_t c_sbo = 8u * a.c_pad * 2u;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmD);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(dfull, 1);
    mbar_init(d1_full, 1);
    mbar_init(d1_free, 4);
    mbar_init(t1_full, 4);
    mbar_init(t1_free, 1);
    mbar_init(d2_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tD1 = tmem, tD2 = tmem + 256;
  pdl_launch_dependents();

  if (nja > 0) {
    if (warp == 0) {
      if (elect_one()) {
        // cores first: they do not depend on the previous kernel
        mbar_arrive_expect_tx(dfull, n1 * a.n_b * 2);
        for (int q = 0; q < nq; ++q) tma_load_2d(sD + q * (n1 * 32), &tmD, dfull, q * 16, 0);
        const int npre = min(nja, S);
        for (int i = 0; i < npre; ++i) {
          uint8_t* st = sStage + i * L.stage_bytes;
          mbar_arrive_expect_tx(&full[i], L.x_bytes + L.c_tx);
          tma_load_2d(st + L.x_bytes, &tmC, &full[i], 0, (ja0 + i) * a.b_pad);
        }
        pdl_wait();
        for (int i = 0; i < npre; ++i) {
          uint8_t* st = sStage + i * L.stage_bytes;
          for (int q = 0; q < nq; ++q)
            tma_load_2d(st + q * XCHUNK, &tmX, &full[i], (ja0 + i) * a.n_b + q * 16, tile_m * 128);
        }
        for (int i = npre; i < nja; ++i) {
          const int s = i % S;
          uint8_t* st = sStage + s * L.stage_bytes;
          mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], L.x_bytes + L.c_tx);
          tma_load_2d(st + L.x_bytes, &tmC, &full[s], 0, (ja0 + i) * a.b_pad);
          for (int q = 0; q < nq; ++q)
            tma_load_2d(st + q * XCHUNK, &tmX, &full[s], (ja0 + i) * a.n_b + q * 16, tile_m * 128);
        }
      }
    } else if (warp == 1) {
      if (elect_one()) {
        const uint32_t idesc1 = idesc_bf16_f32(128, n1);
        const uint32_t idesc2 = idesc_bf16_f32(128, a.b_pad);
        mbar_wait(dfull, 0);
        auto mma1 = [&](int i) {
          const int s = i % S;
          mbar_wait(&full[s], (i / S) & 1);
          tc_fence_after();
          uint8_t* st = sStage + s * L.stage_bytes;
          for (int q = 0; q < nq; ++q) {
            const uint64_t ad = smem_desc_sw(smem_u32(st + q * XCHUNK), 6u, 256u);
            const uint64_t bd = smem_desc_sw(smem_u32(sD + q * (n1 * 32)), 6u, 256u);
            mma_bf16_ss(tD1, ad, bd, idesc1, q > 0 ? 1u : 0u);
          }
          mma_commit(d1_full);
        };
        mma1(0);
        for (int i = 0; i < nja; ++i) {
          if (i + 1 < nja) {
            mbar_wait(d1_free, i & 1);  // epilogue has read D1(i)
            tc_fence_after();
            mma1(i + 1);
          }
          mbar_wait(t1_full, i & 1);  // bf16 t1(i) is in smem
          tc_fence_after();
          const int s = i % S;
          const uint32_t cbase = smem_u32(sStage + s * L.stage_bytes + L.x_bytes);
          for (int al = 0; al < a.r0; ++al) {
            const int col = al * a.c_pad;
            const uint64_t ad0 = smem_desc_sw(smem_u32(sT1 + (col / 64) * T1_CHUNK), 2u, 1024u) + ((col % 64) * 2 >> 4);
            const uint64_t bd0 = smem_desc_sw(cbase, c_layout, c_sbo);
            for (int k = 0; k < a.c_pad / 16; ++k)
              mma_bf16_ss(tD2 + al * a.b_pad, ad0 + 2 * k, bd0 + 2 * k, idesc2, (i > 0 || k > 0) ? 1u : 0u);
          }
          mma_commit(t1_free);
          mma_commit(&empty[s]);
        }
        mma_commit(d2_done);
      }
      __syncwarp();
    } else {
      const uint32_t q = warp & 3;
      const int lrow = q * 32 + lane_id();
      const uint32_t lane_base = (q * 32) << 16;
      pdl_wait();
      for (int i = 0; i < nja; ++i) {
        mbar_wait(d1_full, i & 1);
        tc_fence_after();
        if (i > 0) mbar_wait(t1_free, (i - 1) & 1);  // MMA2(i-1) finished reading t1
        uint8_t* rowp_base = sT1 + (lrow >> 3) * 1024 + (lrow & 7) * 128;
        for (int cc = 0; cc < n1; cc += 32) {
          float v[32];
          tmem_ld16(tD1 + lane_base + cc, v);
          tmem_ld16(tD1 + lane_base + cc + 16, v + 16);
          uint8_t* rowp = rowp_base + (cc / 64) * T1_CHUNK;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 p;
            p.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
            p.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
            p.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
            p.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
            const int ch = ((cc % 64) / 8) + j;
            sts128(smem_u32(rowp) + ((ch ^ (lrow & 7)) << 4), p);
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0) {
          mbar_arrive(d1_free);
          mbar_arrive(t1_full);
        }
      }
      // cut state T[m][alpha*b + bb]
      mbar_wait(d2_done, 0);
      tc_fence_after();
      const int m = tile_m * 128 + lrow;
      const bool ok = m < a.M;
      // vector path: unit cut stride and a bond that fills whole 16-column groups -> one 16-byte
      // bf16 store / four red.global.add.v4.f32 per 16 values (rows start 32-byte aligned: s_m is
      // the padded cut width, a multiple of 16)
      const bool vec = a.s_k == 1 && a.b % 16 == 0 && a.s_m % 16 == 0;
      for (int al = 0; al < a.r0; ++al) {
        for (int bb = 0; bb < a.b_pad; bb += 16) {
          float v[16];
          tmem_ld16(tD2 + lane_base + al * a.b_pad + bb, v);
          if (!ok) continue;
          if (vec) {
            const int64_t k = (int64_t)al * a.b + bb;
            if (a.out_f32_atomic) {
              float* o = static_cast<float*>(a.out) + (int64_t)m * a.s_m + k;
#pragma unroll
              for (int e = 0; e < 16; e += 4) red_add_v4(o + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
            } else {
              uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.out) + (int64_t)m * a.s_m + k);
              o[0] = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                                pack_bf16x2(v[6], v[7]));
              o[1] = make_uint4(pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]), pack_bf16x2(v[12], v[13]),
                                pack_bf16x2(v[14], v[15]));
            }
            continue;
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            if (bb + e >= a.b) continue;
            const int64_t k = (int64_t)al * a.b + bb + e;
            if (a.out_f32_atomic)
              atomicAdd(static_cast<float*>(a.out) + (int64_t)m * a.s_m + k * a.s_k, v[e]);
            else
              static_cast<__nv_bfloat16*>(a.out)[(int64_t)m * a.s_m + k * a.s_k] = __float2bfloat16_rn(v[e]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

int launch_chain_in2(const CUtensorMap& x, const CUtensorMap& d, const CUtensorMap& c, const ChainArgs& a,
                     int splits, cudaStream_t st) {
  const ChainLayout L = chain_layout(a);
  if (L.total > 227 * 1024 || a.r0 * a.c_pad > 256 || a.r0 * a.b_pad > 256 || a.n_b % 16) return (int)cudaErrorInvalidValue;
  static int attr_smem = 0;
  if ((int)L.total > attr_smem) {
    cudaError_t e = cudaFuncSetAttribute(chain_in2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return (int)e;
    attr_smem = 227 * 1024;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.M + 127) / 128, splits, 1);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, chain_in2_kernel, x, d, c, a);
  count_launch();
  return (int)e;
}

}  // namespace tnl
