// decode_pair.cu — the decode-stack boundary kernel (decode_fused.cu) over a CTA pair.
//
// Same boundary as dec_fused_kernel: phase B of layer l (y = A_out^l T_l) fused with phase A of
// layer l+1 (T_{l+1} += B_in^{l+1}[:, rows] y), but two CTAs of a 2x1 cluster own 256 consecutive
// rows and issue M=256 tcgen05.mma.cta_group::2 instructions for both phases:
//   phase B: A = A_out rows (128 per CTA), B = T_l split by TOKENS (each CTA converts only its
//            half of the tokens: half the fp32 T_l bytes read per CTA);
//   phase A: A = B_in^{l+1} split by KAPPA (each CTA holds 128 kappa rows for all 256 K rows of
//            the pair), B = y split by tokens (each CTA sends the other half of its y rows to the
//            peer over DSMEM, 8 KB at 64 tokens); the K reduction over the pair's 256 rows
//            happens inside the MMA, so each CTA reduces 128 kappa rows into T_{l+1} instead of
//            256: half the fp32 reduction bytes leaving each SM, half the L2 atomics per layer.
// The measured critical path of the one-CTA kernel is the T_l read and the partial-T egress
// (profiles/r02: skipping the reductions' atomicity changes nothing, their bytes do).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "decode.cuh"
#include "ptx.cuh"

namespace tnl {

namespace {

constexpr int PT = 320, PEPI = 256;      // TMA warp, MMA warp, 8 epilogue warps
constexpr uint32_t PWBLK = 128 * 64 * 2;  // 128 rows x 64 k bf16 weight block (16 KB)

__device__ __forceinline__ void pnbar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// byte offset of bf16 element (row r, k) in a K-major SW128 block (128-byte rows, 8-row atoms)
__device__ __forceinline__ uint32_t sw128_elem(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2);
}
__device__ __forceinline__ void sts16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void bulk_to_peer(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                             uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(src_cta), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ float ldg_cg(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

template <int BN>
struct PSmem {
  static constexpr int H = BN / 2;                    // tokens per CTA in the B operands
  static constexpr uint32_t HB = H * 128;             // one K-major 64-k block of H token rows
  static constexpr size_t bytes = 1024 + 4 * PWBLK    // A_out blocks (kB <= 256)
                                  + 4 * PWBLK         // B_in blocks (then the D_A transpose stage)
                                  + 4 * HB            // T operand (this CTA's tokens)
                                  + 4 * HB            // x operand (this CTA's tokens, all 256 K)
                                  + 2 * HB            // x staging for the peer's tokens
                                  + 256;
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PT, 1)
    dec_fused_pair_kernel(const __grid_constant__ CUtensorMap tmWo, const __grid_constant__ CUtensorMap tmWi,
                          const FusedArgs a) {
  using SM = PSmem<BN>;
  constexpr int H = SM::H;
  constexpr uint32_t HB = SM::HB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sWo = smem;
  uint8_t* sWi = sWo + 4 * PWBLK;
  uint8_t* sT = sWi + 4 * PWBLK;
  uint8_t* sX = sT + 4 * HB;
  uint8_t* sXs = sX + 4 * HB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sXs + 2 * HB);
  uint64_t* wfull = bars;      // leader: every weight block of both CTAs landed
  uint64_t* tfull = bars + 1;  // leader: T converted in both CTAs (8 warps x 2)
  uint64_t* bdone = bars + 2;  // phase-B MMAs complete (multicast)
  uint64_t* xfull = bars + 3;  // this CTA's x operand complete (local part + the peer's bulk copy)
  uint64_t* xpeer = bars + 4;  // leader: the peer's x operand complete
  uint64_t* adone = bars + 5;  // phase-A MMAs complete (multicast)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const uint32_t rank = cluster_ctarank();
  const uint32_t peer = rank ^ 1u;
  const bool leader = rank == 0;
  const int tile = blockIdx.x;            // this CTA's 128 rows of layer l
  const int pair_row0 = (tile >> 1) * 256;
  const int kbB = (a.kB + 63) / 64;
  const bool a_live = 128 * (int)rank < a.nA;  // this CTA's kappa half has rows of B_in^{l+1}
  unsigned long long* tr = a.trace ? a.trace + 16 * blockIdx.x : nullptr;
#define PTRACE(ev) \
  if (tr) tr[ev] = globaltimer();
  if (threadIdx.x == 0) PTRACE(0);
  const uint32_t warp = warp_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmWo);
    tma_prefetch_desc(&tmWi);
    mbar_init(wfull, 1);
    mbar_init(tfull, 2 * (PEPI / 32));
    mbar_init(bdone, 1);
    mbar_init(xfull, 1);
    mbar_init(xpeer, 1);
    mbar_init(adone, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDB = tmem, tDA = tmem + 64;
  pdl_launch_dependents();
  if (threadIdx.x == 0) PTRACE(1);

  if (warp == 0) {
    if (elect_one()) {
      if (leader) {
        const int live = (a.nA > 0 ? 1 : 0) + (a.nA > 128 ? 1 : 0);
        mbar_arrive_expect_tx(wfull, (uint32_t)(2 * kbB + 4 * live) * PWBLK);
      }
      for (int kb = 0; kb < kbB; ++kb) tma_load_2d_pair(sWo + kb * PWBLK, &tmWo, wfull, kb * 64, tile * 128);
      if (a_live)
        for (int kb = 0; kb < 4; ++kb)
          tma_load_2d_pair(sWi + kb * PWBLK, &tmWi, wfull, pair_row0 + kb * 64, 128 * (int)rank);
      PTRACE(2);
    }
    __syncwarp();
    if (a.t_zero) {  // T_{l-1} was read only by the previous kernel, which has completed
      pdl_wait();
      const int64_t n4 = a.zero_elems / 4, per = (n4 + gridDim.x - 1) / gridDim.x;
      float4* z = reinterpret_cast<float4*>(a.t_zero);
      const int64_t e0 = (int64_t)blockIdx.x * per, e1 = min(n4, e0 + per);
      for (int64_t e = e0 + lane_id(); e < e1; e += 32) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, BN);
      mbar_wait(wfull, 0);
      mbar_wait_cluster(tfull, 0);
      tc_fence_after();
      for (int kb = 0; kb < kbB; ++kb) {
        const uint64_t ad = smem_desc_sw128(smem_u32(sWo + kb * PWBLK));
        const uint64_t bd = smem_desc_sw128(smem_u32(sT + kb * HB));
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_bf16_ss_pair(tDB, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
      }
      mma_commit_pair(bdone, 3);
      mbar_wait(xfull, 0);
      mbar_wait_cluster(xpeer, 0);
      tc_fence_after();
      for (int kb = 0; kb < 4; ++kb) {
        const uint64_t ad = smem_desc_sw128(smem_u32(sWi + kb * PWBLK));
        const uint64_t bd = smem_desc_sw128(smem_u32(sX + kb * HB));
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_bf16_ss_pair(tDA, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
      }
      mma_commit_pair(adone, 3);
    }
    __syncwarp();
  } else {
    const int et = threadIdx.x - 64;
    pdl_wait();
    if (et == 0) PTRACE(3);
    // T_l (fp32, kappa-major [kappa][64]) -> this CTA's tokens, K-major bf16 [token][kappa]: a
    // thread packs 8 consecutive kappa of one token (8 loads, each a 128-byte warp-coalesced row
    // segment across the lanes' tokens) into one 16-byte chunk.
    {
      constexpr int ITEMS = 8 * H;  // (token, 8-kappa chunk) per 64-kappa block
      constexpr int PER = ITEMS >= PEPI ? ITEMS / PEPI : 1;
      const int tok0 = (int)rank * H;
      float v[4][PER][8];
#pragma unroll
      for (int kb = 0; kb < 4; ++kb)
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int e = et + u * PEPI;
          const int tok = e % H, ch = e / H;
          const int kap0 = kb * 64 + ch * 8;
          const bool ok = kb < kbB && e < ITEMS && tok0 + tok < a.tokens;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            v[kb][u][j] = ok && kap0 + j < a.kB ? ldg_cg(a.t_in + (int64_t)(kap0 + j) * 64 + tok0 + tok) : 0.f;
        }
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        if (kb >= kbB) break;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int e = et + u * PEPI;
          if (e < ITEMS) {
            const int tok = e % H, ch = e / H;
            uint4 p;
            p.x = pack_bf16x2(v[kb][u][0], v[kb][u][1]);
            p.y = pack_bf16x2(v[kb][u][2], v[kb][u][3]);
            p.z = pack_bf16x2(v[kb][u][4], v[kb][u][5]);
            p.w = pack_bf16x2(v[kb][u][6], v[kb][u][7]);
            sts128(smem_u32(sT + kb * HB) + (uint32_t)((tok >> 3) * 1024 + (tok & 7) * 128 + ((ch ^ (tok & 7)) << 4)), p);
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive_cluster(mapa_shared(tfull, 0));
    }
    if (et == 0) PTRACE(5);

    const uint32_t q = warp & 3;
    const int lrow = q * 32 + lane_id();
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const int c_begin = ((warp - 2) >> 2) * HALF;
    mbar_wait(bdone, 0);
    tc_fence_after();
    if (et == 0) PTRACE(6);
    {
      // y row lrow of this CTA = K index 128 rank + lrow of the pair: tokens of this CTA's half go
      // into the local x operand (k-block 2 rank + lrow / 64), the peer's tokens into the staging
      // block that is bulk-copied to the same k-blocks of the peer's x operand.
      const int kb_loc = (lrow >> 6), kcol = lrow & 63;
      const uint32_t own = smem_u32(sX) + (uint32_t)(2 * rank + kb_loc) * HB;
      const uint32_t stg = smem_u32(sXs) + (uint32_t)kb_loc * HB;
#pragma unroll 1
      for (int c = c_begin; c < c_begin + HALF && c < BN; c += 16) {
        float v[16];
        tmem_ld16(tDB + ((q * 32) << 16) + c, v);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int t = c + e;
          const bool mine = (t / H) == (int)rank;
          const uint32_t dst = (mine ? own : stg) + sw128_elem(t % H, kcol);
          sts16(dst, __bfloat16_as_ushort(__float2bfloat16_rn(v[e])));
        }
      }
    }
    tc_fence_before();
    fence_proxy_async_smem();
    pnbar(1, PEPI);
    if (et == 0) {
      mbar_arrive_expect_tx(xfull, 2 * HB);  // the peer's rows of our tokens
      bulk_to_peer(mapa_shared(sX, peer) + 2 * rank * HB, smem_u32(sXs), 2 * HB, mapa_shared(xfull, peer));
      PTRACE(7);
      if (!leader) {
        mbar_wait(xfull, 0);
        mbar_arrive_cluster(mapa_shared(xpeer, 0));
      }
    }
    // D_A (this CTA's 128 kappa rows) -> fp32 reductions into T_{l+1}, transposed through smem
    // (over the B_in blocks, free once adone fired) so each warp reduces contiguous rows
    mbar_wait(adone, 0);
    tc_fence_after();
    if (et == 0) PTRACE(8);
    constexpr int SLOTS = BN / 4;
    const uint32_t stage = smem_u32(sWi);
    auto slot_addr = [&](int kap, int sl) {
      return stage + (uint32_t)(kap * SLOTS + (sl ^ (kap & 7 & (SLOTS - 1)))) * 16u;
    };
    const int kap_base = 128 * (int)rank;
#pragma unroll 1
    for (int c = c_begin; c < c_begin + HALF && c < BN; c += 16) {
      float v[16];
      tmem_ld16(tDA + ((q * 32) << 16) + c, v);
      if (kap_base + lrow >= a.nA) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 p;
        p.x = __float_as_uint(v[4 * j]);
        p.y = __float_as_uint(v[4 * j + 1]);
        p.z = __float_as_uint(v[4 * j + 2]);
        p.w = __float_as_uint(v[4 * j + 3]);
        sts128(slot_addr(lrow, c / 4 + j), p);
      }
    }
    pnbar(1, PEPI);
    {
      const int tok_slots = (a.tokens + 3) / 4 < SLOTS ? (a.tokens + 3) / 4 : SLOTS;
      const int rows = min(128, a.nA - kap_base);
      for (int e = et; e < rows * SLOTS; e += PEPI) {
        const int kap = e / SLOTS, sl = e % SLOTS;
        if (sl >= tok_slots) continue;
        const float4 v = lds128f(slot_addr(kap, sl));
        red_add_v4(a.t_out + (int64_t)(kap_base + kap) * 64 + sl * 4, v.x, v.y, v.z, v.w);
      }
    }
    if (et == 0) PTRACE(9);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's MMAs / bulk copy no longer touch this CTA's TMEM and smem
  if (warp == 1) tmem_dealloc_pair<128>(tmem);
  if (threadIdx.x == 32) PTRACE(10);
#undef PTRACE
}

template <int BN>
int launch_pair(const CUtensorMap& wo, const CUtensorMap& wi, const FusedArgs& a, int grid, cudaStream_t st) {
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(dec_fused_pair_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)PSmem<BN>::bytes);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(PT, 1, 1);
  cfg.dynamicSmemBytes = PSmem<BN>::bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dec_fused_pair_kernel<BN>, wo, wi, a);
  count_launch();
  return (int)e;
}

}  // namespace

bool dec_fused_pair_ok(const FusedArgs& a) {
  return !a.kg && a.kB <= 256 && a.nA <= 256 && a.rows % 256 == 0 && a.tokens >= 1 && a.tokens <= 64 &&
         !a.flag_wait && !a.flag_signal;
}

int launch_dec_fused_pair(const CUtensorMap& wo, const CUtensorMap& wi, const FusedArgs& a, int grid,
                          cudaStream_t st) {
  if (!dec_fused_pair_ok(a) || grid % 2) return (int)cudaErrorInvalidValue;
  if (a.tokens <= 16) return launch_pair<16>(wo, wi, a, grid, st);
  if (a.tokens <= 32) return launch_pair<32>(wo, wi, a, grid, st);
  return launch_pair<64>(wo, wi, a, grid, st);
}

}  // namespace tnl
