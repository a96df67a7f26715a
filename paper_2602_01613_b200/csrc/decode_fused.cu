// decode_fused.cu — one kernel per layer boundary for a decode stack:
// phase B of layer l fused with phase A of layer l+1 (merged-cut plans).
//
// CTA i owns output rows [128 i, 128 i + 128) of layer l. Those rows are
// exactly the K-slice [128 i, 128 i + 128) that layer l+1's phase A contracts,
// so y_l never leaves the SM:
//   D_B (128 rows x M) = A_out^l[rows] . T_l            T_l from the fp32 accumulator
//   x   = bf16(D_B)^T   -> SW128 smem operand [M tokens][128 k]
//   D_A (kappa x M)     = B_in^{l+1}[:, rows] . x        -> fp32 reductions into T_{l+1}
// One kernel boundary per layer instead of two, no activation round trip
// through HBM/L2. T_l / T_{l+1} alternate between two zero-at-rest
// accumulators; the last CTA to finish reading T_l re-zeroes it.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "decode.cuh"
#include "ptx.cuh"

namespace tnl {

namespace {

constexpr int FT = 320, FEPI = 256;  // threads: TMA warp, MMA warp, 8 epilogue warps
constexpr uint32_t WBLK = 128 * 64 * 2;  // one 128-row x 64-k bf16 weight block (16 KB)

__device__ __forceinline__ void nbar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
}

// Shared memory, laid out by the boundary's actual block counts (kbB A_out / T blocks, nT B_in
// tiles): A_out blocks | B_in blocks (later the D_A transpose stage) | x operand | T operand | bars
struct FSmem {
  static constexpr uint32_t T_BLK = 64 * 128;  // bf16 T operand block, MN-major [64 kappa][128 B]
  static constexpr uint32_t X_BLK = 64 * 128;  // bf16 x operand block, MN-major [64 k][128 B]
  static size_t bytes(int kbB, int nT) {
    return 1024 + (size_t)kbB * WBLK + (size_t)nT * 2 * WBLK + 2 * X_BLK + (size_t)kbB * T_BLK + 256;
  }
  // large gated boundary (gate + up cut > 256): B_in reuses the gate's A blocks once the gate MMAs
  // have completed, so only the A_out blocks, x and T take space
  static size_t bytes_large(int kbB) { return 1024 + (size_t)kbB * WBLK + 2 * X_BLK + (size_t)kbB * T_BLK + 256; }
};

template <int BN, bool GATED, int KMAX>
__global__ void __launch_bounds__(FT, 1)
    dec_fused_kernel(const __grid_constant__ CUtensorMap tmWo, const __grid_constant__ CUtensorMap tmT,
                     const __grid_constant__ CUtensorMap tmWi, const FusedArgs a) {
  using SM = FSmem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int kbB = (a.kB + 63) / 64;
  // kappa split (plain boundaries, a.ksplit == 2): two CTAs per row tile, each computing phase B
  // for the tile and phase A for one 128-row half of kappa' (half the partial-T egress per CTA)
  const int ks = a.ksplit > 1 ? a.ksplit : 1;
  const int nT = ks > 1 ? 1 : (a.nA + 127) / 128;
  const int t0 = ks > 1 ? (int)(blockIdx.x % ks) : 0;  // first kappa' tile of this CTA
  constexpr bool LARGE = KMAX > 4;        // B_in aliases the gate's A blocks (loaded after their MMAs)
  uint8_t* sWo = smem;                    // kbB blocks
  uint8_t* sWi = LARGE ? sWo : sWo + kbB * WBLK;  // nT x 2 blocks (then the D_A transpose stage)
  uint8_t* sX = LARGE ? sWo + kbB * WBLK : sWi + nT * 2 * WBLK;  // x operand: 2 blocks
  uint8_t* sT = sX + 2 * SM::X_BLK;       // kbB bf16 T blocks
  uint64_t* bars = reinterpret_cast<uint64_t*>(sT + kbB * SM::T_BLK);
  uint64_t* wfull = bars;
  uint64_t* stg = bars + 1;  // [4]
  uint64_t* tfull = bars + 18;  // [8]: T block kb converted (one arrive per epilogue warp)
  uint64_t* bdone = bars + 6;
  uint64_t* xfull = bars + 7;
  uint64_t* adone = bars + 8;
  uint64_t* flagbar = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  uint64_t* gdone = bars + 16;   // LARGE: the gate's phase-B MMAs have completed (its A blocks are free)
  uint64_t* wfull2 = bars + 17;  // LARGE: B_in landed
  uint32_t* last_flag = tmem_slot + 1;

  const int tile = blockIdx.x / ks;
  unsigned long long* tr = a.trace ? a.trace + 16 * blockIdx.x : nullptr;
#ifdef TNL_TRACE_CLOCK  // SM-local cycle stamps (diagnostic builds)
#define TRACE(ev) \
  if (tr) tr[ev] = clock64();
#else
#define TRACE(ev) \
  if (tr) tr[ev] = globaltimer();
#endif
  if (threadIdx.x == 0) TRACE(0);
  const uint32_t warp = warp_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmWo);
    tma_prefetch_desc(&tmT);
    tma_prefetch_desc(&tmWi);
    mbar_init(wfull, 1);
    for (int s = 0; s < 4; ++s) mbar_init(&stg[s], 1);
    for (int kb = 0; kb < KMAX; ++kb) mbar_init(&tfull[kb], FEPI / 32);
    mbar_init(bdone, 1);
    mbar_init(xfull, 1);
    mbar_init(adone, 1);
    mbar_init(flagbar, 1);
    mbar_init(gdone, 1);
    mbar_init(wfull2, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDB = tmem, tDA = tmem + BN;  // D_A: nT blocks of BN columns
  const uint32_t tDU = tmem + 192;             // gated boundary: the up projection's D_B (BN <= 64)
  const int kg = GATED ? a.kg : 0;
  pdl_launch_dependents();
  if (threadIdx.x == 0) TRACE(1);

  if (warp == 0) {
    if (elect_one()) {
      // both layers' weights first (independent of the previous kernel)
      mbar_arrive_expect_tx(wfull, (kbB + (LARGE ? 0 : 2 * nT)) * WBLK);
      // L2 policy of the weight stream (TNL_DEC_WPOL at build time, A/B): 0 evict_first (default:
      // keeps the accumulators and activations resident), 2 evict_last (the concurrent token
      // groups re-read each layer's panels from L2 instead of HBM)
#if defined(TNL_DEC_WPOL) && TNL_DEC_WPOL == 2
      const uint64_t pol = policy_evict_last();
#elif defined(TNL_DEC_WPOL) && TNL_DEC_WPOL == 1
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#else
      const uint64_t pol = policy_evict_first();
#endif
      for (int kb = 0; kb < kbB; ++kb)
        tma_load_2d_hint(sWo + kb * WBLK, &tmWo, wfull, kb * 64, tile * 128, pol);
      if (!LARGE)
        for (int t = 0; t < nT; ++t)
          for (int h = 0; h < 2; ++h)
            tma_load_2d_hint(sWi + (t * 2 + h) * WBLK, &tmWi, wfull, tile * 128 + h * 64, (t0 + t) * 128, pol);
      TRACE(2);
      pdl_wait();
      TRACE(3);
      if constexpr (LARGE) {  // B_in into the gate's A blocks once the gate MMAs have read them
        mbar_wait(gdone, 0);
        mbar_arrive_expect_tx(wfull2, 2 * nT * WBLK);
        for (int t = 0; t < nT; ++t)
          for (int h = 0; h < 2; ++h)
            tma_load_2d_hint(sWi + (t * 2 + h) * WBLK, &tmWi, wfull2, tile * 128 + h * 64, t * 128, pol);
      }
    }
    __syncwarp();
    // T_{l-1} was read only by the previous kernel, which has completed: zero this CTA's slice
    if (a.t_zero) {
      pdl_wait();
      const int64_t n4 = a.zero_elems / 4, per = (n4 + gridDim.x - 1) / gridDim.x;
      float4* z = reinterpret_cast<float4*>(a.t_zero);
      const int64_t e0 = (int64_t)blockIdx.x * per, e1 = min(n4, e0 + per);
      for (int64_t e = e0 + lane_id(); e < e1; e += 32) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32_bmn(128, BN);  // T and x operands are MN-major
      mbar_wait(wfull, 0);
      for (int kb = 0; kb < kbB; ++kb) {  // block kb as soon as it is converted
        mbar_wait(&tfull[kb], 0);
        if (kb == kbB - 1) TRACE(15);
        tc_fence_after();
        const uint64_t ad = smem_desc_sw128(smem_u32(sWo + kb * WBLK));
        const uint64_t bd = smem_desc_sw128(smem_u32(sT + kb * SM::T_BLK));
        const bool up = GATED && kb >= kg;
        const uint32_t d = up ? tDU : tDB;
        const int kk = up ? kb - kg : kb;
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_bf16_ss(d, ad + 2 * k, bd + 128 * k, idesc, (kk | k) != 0);
        if (LARGE && kb == kg - 1) mma_commit(gdone);
      }
      mma_commit(bdone);
      mbar_wait(xfull, 0);
      if constexpr (LARGE) mbar_wait(wfull2, 0);
      tc_fence_after();
      for (int t = 0; t < nT; ++t)
        for (int h = 0; h < 2; ++h) {
          const uint64_t ad = smem_desc_sw128(smem_u32(sWi + (t * 2 + h) * WBLK));
          const uint64_t bd = smem_desc_sw128(smem_u32(sX + h * SM::X_BLK));
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_bf16_ss(tDA + t * BN, ad + 2 * k, bd + 128 * k, idesc, (h | k) != 0);
        }
      mma_commit(adone);
    }
    __syncwarp();
  } else {
    const int et = threadIdx.x - 64;
    pdl_wait();
    if (et == 0) TRACE(11);
    // T_l: fp32 [64 kappa][BN tokens] -> bf16 MN-major SW128 [64 kappa][128 B] per k-block
    // (the accumulator's kappa-major layout is the MMA's MN-major B operand: no transpose).
    // Read straight from L2 by all epilogue threads: every 16-byte load of every block is in
    // flight at once (a TMA box per block lands at ~14 B/cycle, one after the other), then one
    // proxy fence publishes all converted blocks. One float4 = 4 tokens of one kappa row; a warp
    // reads 512 contiguous bytes and writes 8-byte halves of the swizzled 16-byte chunks.
    constexpr int QPR = BN / 4;                  // float4 quads per kappa row
    constexpr int ITEMS = 64 * QPR;              // per k-block
    constexpr int PER = ITEMS >= FEPI ? ITEMS / FEPI : 1;
    {
      float4 v[KMAX][PER];
#pragma unroll
      for (int kb = 0; kb < KMAX; ++kb)
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int e = et + u * FEPI;
          const int kap = kb * 64 + e / QPR, quad = e % QPR;
          v[kb][u] = make_float4(0.f, 0.f, 0.f, 0.f);
#ifndef TNL_DIAG_NOTLOAD  // timing diagnostic only: skip the T_l read (wrong results)
          if (kb < kbB && e < ITEMS && kap < a.kB) v[kb][u] = ldg128_cg(a.t_in + (int64_t)kap * 64 + quad * 4);
#endif
        }
      if (et == 0) TRACE(12);
#pragma unroll
      for (int kb = 0; kb < KMAX; ++kb) {
        if (kb >= kbB) break;
        const uint32_t dst = smem_u32(sT) + kb * SM::T_BLK;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int e = et + u * FEPI;
          if (e < ITEMS) {
            const int kap = e / QPR, quad = e % QPR;
            uint2 p;
            p.x = pack_bf16x2(v[kb][u].x, v[kb][u].y);
            p.y = pack_bf16x2(v[kb][u].z, v[kb][u].w);
            sts64(dst + sw128(kap, quad >> 1) + (quad & 1) * 8, p);
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane_id() == 0)
        for (int kb = 0; kb < kbB; ++kb) mbar_arrive(&tfull[kb]);
      if (et == 0) TRACE(14);
    }
    if (et == 0) TRACE(5);

    const uint32_t q = warp & 3;
    const int lrow = q * 32 + lane_id();
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const int c_begin = ((warp - 2) >> 2) * HALF;
    // y_l tile -> x operand of layer l+1 (row = token, k = this CTA's row lrow)
    mbar_wait(bdone, 0);
    tc_fence_after();
    if (et == 0) TRACE(6);
    {
      // x operand of layer l+1, MN-major: K index = this CTA's row lrow, 128-byte row of tokens
#pragma unroll 1
      for (int c = c_begin; c < c_begin + HALF && c < BN; c += 16) {
        float v[16];
        tmem_ld16(tDB + ((q * 32) << 16) + c, v);
        if constexpr (GATED) {  // h = silu(g) * u = g * u * sigmoid(g), fp32
          float w[16];
          tmem_ld16(tDU + ((q * 32) << 16) + c, w);
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = v[e] * w[e] * __frcp_rn(1.f + __expf(-v[e]));
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint4 p;
          p.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
          p.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
          p.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
          p.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
          sts128(smem_u32(sX) + sw128(lrow, c / 8 + j), p);
        }
      }
    }
    tc_fence_before();
    fence_proxy_async_smem();
    nbar(1, FEPI);
    if (et == 0) mbar_arrive(xfull);
    if (et == 0) TRACE(7);
    // D_A -> fp32 reductions into T_{l+1} (kappa-major [kappa][64]). A thread holds one kappa
    // row, so reducing straight from TMEM makes every 16-byte red its own L2 transaction (32
    // per warp instruction); the partial is transposed through smem first (over the B_in blocks,
    // free once adone fired; float4 slots XOR-swizzled by kappa & 7) so that each warp then
    // reduces two contiguous 256-byte rows per instruction.
    mbar_wait(adone, 0);
    tc_fence_after();
    if (et == 0) TRACE(8);
    constexpr int SLOTS = BN / 4;  // float4 slots per kappa row
    const uint32_t stage = smem_u32(sWi);
    auto slot_addr = [&](int kap, int sl) {
      return stage + (uint32_t)(kap * SLOTS + (sl ^ (kap & 7 & (SLOTS - 1)))) * 16u;
    };
    for (int t = 0; t < nT; ++t) {
      const int kap = t * 128 + lrow;  // local row of this CTA's kappa' range
#pragma unroll 1
      for (int c = c_begin; c < c_begin + HALF && c < BN; c += 16) {
        float v[16];
        tmem_ld16(tDA + t * BN + ((q * 32) << 16) + c, v);
        if (t0 * 128 + kap >= a.nA) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 p;
          p.x = __float_as_uint(v[4 * j]);
          p.y = __float_as_uint(v[4 * j + 1]);
          p.z = __float_as_uint(v[4 * j + 2]);
          p.w = __float_as_uint(v[4 * j + 3]);
          sts128(slot_addr(kap, c / 4 + j), p);
        }
      }
    }
    nbar(1, FEPI);
    {
      const int tok_slots = (a.tokens + 3) / 4 < SLOTS ? (a.tokens + 3) / 4 : SLOTS;
      const int rows_here = min(a.nA - t0 * 128, nT * 128);
      float* t_out = a.t_out + (int64_t)t0 * 128 * 64;
      for (int e = et; e < rows_here * SLOTS; e += FEPI) {
        const int kap = e / SLOTS, sl = e % SLOTS;
        if (sl >= tok_slots) continue;
        const float4 v = lds128f(slot_addr(kap, sl));
#ifdef TNL_DIAG_NORED  // timing diagnostic only: plain stores instead of reductions (wrong results)
        *reinterpret_cast<float4*>(t_out + (int64_t)kap * 64 + sl * 4) = v;
#else
        red_add_v4(t_out + (int64_t)kap * 64 + sl * 4, v.x, v.y, v.z, v.w);
#endif
      }
    }
    if (et == 0) TRACE(9);

  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
  if (threadIdx.x == 32) TRACE(10);
#undef TRACE
}

template <int BN, bool GATED, int KMAX>
int launch_fused(const CUtensorMap& wo, const CUtensorMap& t, const CUtensorMap& wi, const FusedArgs& a,
                 int grid, cudaStream_t st) {
  // plain boundaries (decode stacks: 40-64 CTAs) reserve the full layout, one CTA per SM; the gated
  // MLP boundary (inter/128 = 200 CTAs at Qwen3 shapes) takes only what its ranks need, so two
  // CTAs share an SM and the grid runs in one wave
  const size_t smem = KMAX > 4 ? FSmem::bytes_large((a.kB + 63) / 64)
                     : GATED ? FSmem::bytes((a.kB + 63) / 64, (a.nA + 127) / 128) : FSmem::bytes(4, 2);
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(dec_fused_kernel<BN, GATED, KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(KMAX > 4 ? FSmem::bytes_large(KMAX) : FSmem::bytes(4, 2)));
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(FT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dec_fused_kernel<BN, GATED, KMAX>, wo, t, wi, a);
  count_launch();
  return (int)e;
}

}  // namespace

int launch_dec_fused(const CUtensorMap& wo, const CUtensorMap& t, const CUtensorMap& wi, const FusedArgs& a,
                     int grid, cudaStream_t st) {
  if (a.nA > 256 || a.rows % 128) return (int)cudaErrorInvalidValue;
  if (a.kB > 256) {
    // large gated boundary: B_in (2 * nT blocks) must fit in the gate's A blocks
    if (!a.kg || a.kB > 512 || a.kg < 2 * ((a.nA + 127) / 128)) return (int)cudaErrorInvalidValue;
    if (a.tokens <= 16) return launch_fused<16, true, 8>(wo, t, wi, a, grid, st);
    if (a.tokens <= 32) return launch_fused<32, true, 8>(wo, t, wi, a, grid, st);
    return launch_fused<64, true, 8>(wo, t, wi, a, grid, st);
  }
  if (a.kg) {
    if (a.tokens <= 16) return launch_fused<16, true, 4>(wo, t, wi, a, grid, st);
    if (a.tokens <= 32) return launch_fused<32, true, 4>(wo, t, wi, a, grid, st);
    return launch_fused<64, true, 4>(wo, t, wi, a, grid, st);
  }
  if (a.tokens <= 16) return launch_fused<16, false, 4>(wo, t, wi, a, grid, st);
  if (a.tokens <= 32) return launch_fused<32, false, 4>(wo, t, wi, a, grid, st);
  return launch_fused<64, false, 4>(wo, t, wi, a, grid, st);
}

}  // namespace tnl
