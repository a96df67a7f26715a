// decode.cu — small-M kernels of the merged-cut plan (see decode.cuh).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "decode.cuh"
#include "ptx.cuh"

namespace tnl {

namespace {

constexpr int BM = 128, BK = 64;
constexpr uint32_t A_STAGE = BM * BK * 2;

template <int BN>
constexpr uint32_t tmem_cols() {
  return BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
}

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// SW128 K-major: byte offset of 16-byte chunk c (8 bf16) of row r inside a stage tile
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
}

template <int BN, int STAGES, bool ACT_F32>
struct DecSmem {
  // bf16 activation operand: x K-major [BN tokens][64 k] (phase A, TMA) or T MN-major
  // [64 kappa][128 B] (phase B: the kappa-major accumulator converted without a transpose)
  static constexpr uint32_t B_STAGE = ACT_F32 ? 64 * 128 : BN * BK * 2;
  static constexpr uint32_t F_STAGE = ACT_F32 ? BK * BN * 4 : 0;  // fp32 staging [64 k][BN tokens]
  static constexpr uint32_t Y_BYTES = ACT_F32 ? BN * BM * 2 : 0;  // y tile [BN tokens][128 rows]
  static constexpr size_t bytes = 1024 + (size_t)STAGES * (A_STAGE + B_STAGE + F_STAGE) + Y_BYTES + 512;
};

// 2 non-epilogue warps (TMA, MMA) + 8 epilogue warps: two warps per TMEM lane
// quarter split the token columns, halving the per-thread reduction / store count.
constexpr int DEC_THREADS = 320, DEC_EPI = 256;

template <int BN, int STAGES, bool ACT_F32>
__global__ void __launch_bounds__(DEC_THREADS, 1)
    dec_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
               const __grid_constant__ CUtensorMap tmY, const DecArgs a) {
  using SM = DecSmem<BN, STAGES, ACT_F32>;
  constexpr uint32_t B_STAGE = SM::B_STAGE, F_STAGE = SM::F_STAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  float* sF = reinterpret_cast<float*>(sB + STAGES * B_STAGE);
  __nv_bfloat16* sY = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(sF) + STAGES * F_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sY) + SM::Y_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* stg = empty + STAGES;
  uint64_t* done = stg + STAGES;
  uint64_t* flagbar = done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(flagbar + 1);
  uint32_t* last_flag = tmem_slot + 1;

  const int tile_m = blockIdx.x;
  const int total_kb = (a.K + BK - 1) / BK;
  const int kb0 = blockIdx.z * a.kb_per_split;
  const int kb1 = min(total_kb, kb0 + a.kb_per_split);
  const int nkb = kb1 - kb0;
  const uint32_t warp = warp_id();
  unsigned long long* tr = a.trace ? a.trace + 16 * (blockIdx.x + gridDim.x * blockIdx.z) : nullptr;
#define TRACE(ev) \
  if (tr) tr[ev] = globaltimer();
  if (threadIdx.x == 0) TRACE(0);

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    if (ACT_F32) tma_prefetch_desc(&tmY);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], (ACT_F32 || a.x_host) ? 2 : 1);
      mbar_init(&empty[s], 1);
      mbar_init(&stg[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(flagbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<tmem_cols<BN>()>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();
  if (threadIdx.x == 0) TRACE(1);

  if (warp == 0) {
    if (elect_one()) {
      const int npre = min(nkb, STAGES);
      const uint32_t tx = A_STAGE + ((ACT_F32 || a.x_host) ? 0u : B_STAGE);
      for (int i = 0; i < npre; ++i) {  // weights do not depend on the previous kernel
        mbar_arrive_expect_tx(&full[i], tx);
        tma_load_2d_hint(sA + i * A_STAGE, &tmW, &full[i], (kb0 + i) * BK, tile_m * BM,
                         policy_evict_first());
      }
      TRACE(2);
      pdl_wait();
      TRACE(3);
      if (!ACT_F32 && !a.x_host)  // (phase B / host x: the epilogue warps fill the operand stages)
        for (int i = 0; i < npre; ++i) tma_load_2d(sB + i * B_STAGE, &tmX, &full[i], (kb0 + i) * BK, 0);
      for (int i = npre; i < nkb; ++i) {  // (phase A only: ACT_F32 keeps nkb <= STAGES)
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], tx);
        tma_load_2d_hint(sA + s * A_STAGE, &tmW, &full[s], (kb0 + i) * BK, tile_m * BM,
                         policy_evict_first());
        tma_load_2d(sB + s * B_STAGE, &tmX, &full[s], (kb0 + i) * BK, 0);
      }
    }
    __syncwarp();
    if (a.zero_prev) {  // a buffer only the previous kernel read: zero this CTA's slice
      pdl_wait();
      const int64_t ncta = (int64_t)gridDim.x * gridDim.y * gridDim.z;
      const int64_t cta = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z);
      const int64_t n4 = a.zero_prev_elems / 4, per = (n4 + ncta - 1) / ncta;
      float4* z = reinterpret_cast<float4*>(a.zero_prev);
      const int64_t e0 = cta * per, e1 = min(n4, e0 + per);
      for (int64_t e = e0 + lane_id(); e < e1; e += 32) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = ACT_F32 ? idesc_bf16_f32_bmn(BM, BN) : idesc_bf16_f32(BM, BN);
      constexpr uint32_t bstep = ACT_F32 ? 128 : 2;  // descriptor advance per K=16
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (i / STAGES) & 1);
        tc_fence_after();
        if (i == 0) TRACE(4);
        const uint64_t adesc = smem_desc_sw128(smem_u32(sA + s * A_STAGE));
        const uint64_t bdesc = smem_desc_sw128(smem_u32(sB + s * B_STAGE));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) mma_bf16_ss(tmem, adesc + 2 * k, bdesc + bstep * k, idesc, (i | k) != 0);
        mma_commit(&empty[s]);
      }
      mma_commit(done);
      TRACE(5);
    }
    __syncwarp();
  } else {
    const int et = threadIdx.x - 64;  // 0..255
    pdl_wait();
    if constexpr (!ACT_F32) {
      if (a.x_host) {
        // zero-copy H2D: this CTA's K slice of x, [BN tokens][64 k] per stage (SW128 K-major), read
        // from pinned host memory with every 16-byte request in flight at once (nkb <= STAGES)
        constexpr int ITEMS = BN * 8;  // (token, 16-byte chunk) per stage
        constexpr int PER = (ITEMS + DEC_EPI - 1) / DEC_EPI;
        uint4 v[4][PER];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int e = et + u * DEC_EPI;
            const int tok = e >> 3, ch = e & 7;
            v[i][u] = make_uint4(0u, 0u, 0u, 0u);
            if (i < nkb && e < ITEMS && tok < a.tokens) {
              const uint4* src = reinterpret_cast<const uint4*>(a.x_host + (int64_t)tok * a.ldx_host + (kb0 + i) * BK) + ch;
              asm volatile("ld.global.cv.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v[i][u].x), "=r"(v[i][u].y), "=r"(v[i][u].z), "=r"(v[i][u].w)
                           : "l"(src));
            }
          }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i >= nkb) break;
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int e = et + u * DEC_EPI;
            if (e < ITEMS) {
              const int tok = e >> 3, ch = e & 7;
              sts128(smem_u32(sB + i * B_STAGE) + sw128_off(tok, ch), v[i][u]);
            }
          }
        }
        fence_proxy_async_smem();
        named_bar(1, DEC_EPI);
        if (et == 0)
          for (int i = 0; i < nkb; ++i) mbar_arrive(&full[i]);
      }
    }
    if (et == 0) TRACE(6);
    if constexpr (ACT_F32) {
      // fp32 accumulator [64 kappa][BN tokens] per k-block -> bf16 MN-major SW128 operand
      // [64 kappa][128 B] (no transpose). All 16-byte L2 loads of all blocks are in flight at
      // once (instead of one TMA box per block landing after the other), one proxy fence.
      constexpr int QPR = BN / 4;
      constexpr int ITEMS = 64 * QPR;  // (kappa, 4-token quad) per block
      constexpr int PER = ITEMS >= DEC_EPI ? ITEMS / DEC_EPI : 1;
      static_assert(STAGES >= 4, "phase B holds every k-block of the accumulator");
      float4 v[4][PER];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int e = et + u * DEC_EPI;
          const int kap = (kb0 + i) * BK + e / QPR, quad = e % QPR;
          v[i][u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (i < nkb && e < ITEMS && kap < a.K) v[i][u] = ldg128_cg(a.act_f32 + (int64_t)kap * a.act_ld + quad * 4);
        }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i >= nkb) break;
        const uint32_t dst = smem_u32(sB) + i * B_STAGE;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int e = et + u * DEC_EPI;
          if (e < ITEMS) {
            const int kap = e / QPR, quad = e % QPR;
            uint2 p;
            p.x = pack_bf16x2(v[i][u].x, v[i][u].y);
            p.y = pack_bf16x2(v[i][u].z, v[i][u].w);
            sts64(dst + sw128_off(kap, quad >> 1) + (quad & 1) * 8, p);
          }
        }
      }
      fence_proxy_async_smem();
      named_bar(1, DEC_EPI);
      if (et == 0) {
        for (int i = 0; i < nkb; ++i) mbar_arrive(&full[i]);
        if (a.counter) {
          // every accumulator read of this CTA has completed (the values were consumed above):
          // count it; the last CTA re-zeroes the accumulator at the very end
          __threadfence();
          const unsigned total = gridDim.x * gridDim.y * gridDim.z;
          *last_flag = (atomicAdd(a.counter, 1u) == total - 1) ? 1u : 0u;
        }
      }
      if (et == 0) TRACE(7);
    }
    mbar_wait(done, 0);
    tc_fence_after();
    if (et == 0) TRACE(8);
    const uint32_t q = warp & 3;
    const int lrow = q * 32 + lane_id();
    const int row = tile_m * BM + lrow;
    const bool row_ok = row < a.M_rows;
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const int c_begin = ((warp - 2) >> 2) * HALF;
#pragma unroll 1
    for (int c = c_begin; c < c_begin + HALF && c < BN; c += 16) {
      float v[16];
      tmem_ld16(tmem + ((q * 32) << 16) + c, v);
      if constexpr (ACT_F32) {
        // y tile staged [token][row] for one TMA store
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const __nv_bfloat16 h = __float2bfloat16_rn(v[e]);
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(smem_u32(sY + (c + e) * BM + lrow)),
                       "h"(*reinterpret_cast<const unsigned short*>(&h))
                       : "memory");
        }
      } else {
        if (!row_ok || c >= a.tokens) continue;
        const int n = min(16, a.tokens - c);
        // kappa-major accumulator: this thread's 16 token values are contiguous
        float* o = static_cast<float*>(a.out) + (int64_t)row * a.ldo_i + c;
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
    if constexpr (ACT_F32) {
      fence_proxy_async_smem();
      named_bar(1, DEC_EPI);
      if (a.y_host) {
        // zero-copy D2H: the staged y tile [BN tokens][128 rows] straight to pinned host memory
        for (int e = et; e < a.tokens * (BM / 8); e += DEC_EPI) {
          const int tok = e / (BM / 8), ch = e % (BM / 8);
          const int row0 = tile_m * BM + ch * 8;
          if (row0 < a.M_rows)
            *reinterpret_cast<uint4*>(a.y_host + (int64_t)tok * a.ldy_host + row0) =
                lds128(smem_u32(sY) + (tok * BM + ch * 8) * 2);
        }
        __threadfence_system();
      } else if (et == 0) {
        tma_store_2d(&tmY, sY, tile_m * BM, 0);
        tma_store_commit();
      }
      if (a.counter) {  // last_flag was written by et 0 before the named barrier above
        if (*last_flag) {
          float4* z = reinterpret_cast<float4*>(const_cast<float*>(a.act_f32));
          for (int64_t e = et; e < a.zero_elems / 4; e += DEC_EPI) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (et == 0) atomicExch(a.counter, 0u);
        }
      }
      if (et == 0) tma_store_wait_all();
    }
  }
  if (threadIdx.x == 64) TRACE(9);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<tmem_cols<BN>()>(tmem);
  if (threadIdx.x == 32) TRACE(10);
#undef TRACE
}

template <int BN, int STAGES, bool ACT_F32>
int launch_dec(const CUtensorMap& w, const CUtensorMap& x, const CUtensorMap& y, const DecArgs& a,
               int splits, cudaStream_t st) {
  constexpr size_t smem = DecSmem<BN, STAGES, ACT_F32>::bytes;
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(dec_kernel<BN, STAGES, ACT_F32>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.M_rows + BM - 1) / BM, 1, splits);
  cfg.blockDim = dim3(DEC_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dec_kernel<BN, STAGES, ACT_F32>, w, x, y, a);
  count_launch();
  return (int)e;
}

// ---------------------------------------------------------------------------
// CUDA-core GEMV variants (tokens <= 8): one warp per weight row, the whole
// contraction in the warp (16-byte vector loads, warp-shuffle reduction), so
// no split-K reduction and no atomics. A CTA's weight rows are contiguous and
// arrive by one bulk TMA copy issued before griddepcontrol.wait; the
// activations follow after the wait. T is plain fp32 [tokens][ldt].
// ---------------------------------------------------------------------------
constexpr int GV_MAXT = 8;
constexpr int GV_ROWS_A = 8;   // phase A: rows (warps) per CTA
constexpr int GV_ROWS_B = 32;  // phase B: rows per CTA (4 per warp)

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// T[m][row] = sum_k W[row][k] x[m][k]   (W rows contiguous, ldw == K)
__global__ void __launch_bounds__(256) gemv_a_kernel(const __nv_bfloat16* __restrict__ w, int rows, int K,
                                                     const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                     int tokens, float* t, int64_t ldt) {
  extern __shared__ __align__(128) uint8_t gsm[];
  __nv_bfloat16* ws = reinterpret_cast<__nv_bfloat16*>(gsm);                 // [8][K]
  __nv_bfloat16* xs = ws + GV_ROWS_A * K;                                    // [tokens][K]
  __shared__ __align__(8) uint64_t bar;
  const int row0 = blockIdx.x * GV_ROWS_A;
  const int nrows = min(GV_ROWS_A, rows - row0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)(nrows * K * 2));
    bulk_g2s(ws, w + (int64_t)row0 * K, (uint32_t)(nrows * K * 2), &bar);
  }
  pdl_wait();
  for (int e = threadIdx.x; e < tokens * (K / 8); e += 256) {
    const int m = e / (K / 8), c = e % (K / 8);
    reinterpret_cast<uint4*>(xs + (int64_t)m * K)[c] = __ldcg(reinterpret_cast<const uint4*>(x + (int64_t)m * ldx) + c);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int wid = warp_id(), lane = lane_id();
  if (wid >= nrows) return;
  float acc[GV_MAXT];
#pragma unroll
  for (int m = 0; m < GV_MAXT; ++m) acc[m] = 0.f;
  const uint4* wr = reinterpret_cast<const uint4*>(ws + (int64_t)wid * K);
  for (int c = lane; c < K / 8; c += 32) {
    float wf[8];
    bf16x8_to_f32(wr[c], wf);
#pragma unroll
    for (int m = 0; m < GV_MAXT; ++m) {
      if (m >= tokens) break;
      float xf[8];
      bf16x8_to_f32(reinterpret_cast<const uint4*>(xs + (int64_t)m * K)[c], xf);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[m] = fmaf(wf[i], xf[i], acc[m]);
    }
  }
#pragma unroll
  for (int m = 0; m < GV_MAXT; ++m) {
    if (m >= tokens) break;
    float v = acc[m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) t[(int64_t)m * ldt + row0 + wid] = v;
  }
}

// y[m][row] = sum_k W[row][k] bf16(T[m][k])   (W rows contiguous, ldw == K, K % 8 == 0)
__global__ void __launch_bounds__(256) gemv_b_kernel(const __nv_bfloat16* __restrict__ w, int rows, int K,
                                                     const float* __restrict__ t, int64_t ldt, int tokens,
                                                     __nv_bfloat16* y, int64_t ldy) {
  extern __shared__ __align__(128) uint8_t gsm[];
  __nv_bfloat16* ws = reinterpret_cast<__nv_bfloat16*>(gsm);   // [32][K]
  float* ts = reinterpret_cast<float*>(ws + GV_ROWS_B * K);     // [tokens][K]
  __shared__ __align__(8) uint64_t bar;
  const int row0 = blockIdx.x * GV_ROWS_B;
  const int nrows = min(GV_ROWS_B, rows - row0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)(nrows * K * 2));
    bulk_g2s(ws, w + (int64_t)row0 * K, (uint32_t)(nrows * K * 2), &bar);
  }
  pdl_wait();
  for (int e = threadIdx.x; e < tokens * K / 4; e += 256) {
    const int m = e / (K / 4), c = e % (K / 4);
    reinterpret_cast<float4*>(ts + (int64_t)m * K)[c] = __ldcg(reinterpret_cast<const float4*>(t + (int64_t)m * ldt) + c);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int wid = warp_id(), lane = lane_id();
  for (int rr = 0; rr < GV_ROWS_B / 8; ++rr) {
    const int lr = wid * (GV_ROWS_B / 8) + rr;
    if (lr >= nrows) break;
    float acc[GV_MAXT];
#pragma unroll
    for (int m = 0; m < GV_MAXT; ++m) acc[m] = 0.f;
    const uint4* wr = reinterpret_cast<const uint4*>(ws + (int64_t)lr * K);
    for (int c = lane; c < K / 8; c += 32) {
      float wf[8];
      bf16x8_to_f32(wr[c], wf);
#pragma unroll
      for (int m = 0; m < GV_MAXT; ++m) {
        if (m >= tokens) break;
        const float4* tp = reinterpret_cast<const float4*>(ts + (int64_t)m * K + c * 8);
        const float4 a0 = tp[0], a1 = tp[1];
        // T is rounded to bf16 exactly as the tensor-core path rounds its operand
        acc[m] = fmaf(wf[0], __bfloat162float(__float2bfloat16_rn(a0.x)), acc[m]);
        acc[m] = fmaf(wf[1], __bfloat162float(__float2bfloat16_rn(a0.y)), acc[m]);
        acc[m] = fmaf(wf[2], __bfloat162float(__float2bfloat16_rn(a0.z)), acc[m]);
        acc[m] = fmaf(wf[3], __bfloat162float(__float2bfloat16_rn(a0.w)), acc[m]);
        acc[m] = fmaf(wf[4], __bfloat162float(__float2bfloat16_rn(a1.x)), acc[m]);
        acc[m] = fmaf(wf[5], __bfloat162float(__float2bfloat16_rn(a1.y)), acc[m]);
        acc[m] = fmaf(wf[6], __bfloat162float(__float2bfloat16_rn(a1.z)), acc[m]);
        acc[m] = fmaf(wf[7], __bfloat162float(__float2bfloat16_rn(a1.w)), acc[m]);
      }
    }
#pragma unroll
    for (int m = 0; m < GV_MAXT; ++m) {
      if (m >= tokens) break;
      float v = acc[m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) y[(int64_t)m * ldy + row0 + lr] = __float2bfloat16_rn(v);
    }
  }
}

template <typename K, typename... Args>
int launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  count_launch();
  return (int)e;
}

}  // namespace

int launch_dec_a(const CUtensorMap& w, const CUtensorMap& x, const DecArgs& a, int splits, cudaStream_t st) {
  if (a.tokens <= 16) return launch_dec<16, 4, false>(w, x, w, a, splits, st);
  if (a.tokens <= 32) return launch_dec<32, 4, false>(w, x, w, a, splits, st);
  return launch_dec<64, 4, false>(w, x, w, a, splits, st);
}

int launch_dec_b(const CUtensorMap& w, const CUtensorMap& t, const CUtensorMap& y, const DecArgs& a,
                 cudaStream_t st) {
  // K = r_pad <= 256 -> <= 4 k-blocks, all resident (no ring reuse in the fp32-operand path)
  if (a.K > 4 * BK) return (int)cudaErrorInvalidValue;
  if (a.tokens <= 16) return launch_dec<16, 4, true>(w, t, y, a, 1, st);
  if (a.tokens <= 32) return launch_dec<32, 4, true>(w, t, y, a, 1, st);
  return launch_dec<64, 4, true>(w, t, y, a, 1, st);
}

int launch_gemv_a(const __nv_bfloat16* w, int64_t ldw, int rows, int K, const __nv_bfloat16* x, int64_t ldx,
                  int tokens, float* t, int64_t ldt, cudaStream_t st) {
  if (tokens > GV_MAXT || K % 8 || ldw != K || (ldx % 8)) return (int)cudaErrorInvalidValue;
  const size_t smem = (size_t)(GV_ROWS_A + tokens) * K * 2;
  if (smem > 220 * 1024) return (int)cudaErrorInvalidValue;
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(gemv_a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return (int)e;
    attr = 220 * 1024;
  }
  return launch_pdl(gemv_a_kernel, dim3((rows + GV_ROWS_A - 1) / GV_ROWS_A), dim3(256), smem, st, w, rows, K, x,
                    ldx, tokens, t, ldt);
}

int launch_gemv_b(const __nv_bfloat16* w, int64_t ldw, int rows, int K, const float* t, int64_t ldt, int tokens,
                  __nv_bfloat16* y, int64_t ldy, cudaStream_t st) {
  if (tokens > GV_MAXT || K % 8 || ldw != K) return (int)cudaErrorInvalidValue;
  const size_t smem = (size_t)GV_ROWS_B * K * 2 + (size_t)tokens * K * 4;
  if (smem > 220 * 1024) return (int)cudaErrorInvalidValue;
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(gemv_b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return (int)e;
    attr = 220 * 1024;
  }
  return launch_pdl(gemv_b_kernel, dim3((rows + GV_ROWS_B - 1) / GV_ROWS_B), dim3(256), smem, st, w, rows, K, t,
                    ldt, tokens, y, ldy);
}

}  // namespace tnl
