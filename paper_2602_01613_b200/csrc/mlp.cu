// mlp.cu — fused middle of a TN-compressed Qwen3 MLP block.
//
//   y = down( silu(gate(x)) * up(x) ),  gate/up/down merged-cut TN layers.
// With the cut panels (gate: B_g, A_g; up: B_u, A_u; down: B_d, A_d) the block is
//   T_g = x B_g^T, T_u = x B_u^T                 (one GEMM over the concatenated B_g|B_u)
//   h   = silu(T_g A_g^T) * (T_u A_u^T)          (M x 25600 — the expensive intermediate)
//   T_d = h B_d^T                                 (contracts the 25600 intermediate)
//   y   = T_d A_d^T
// The kernels here fuse the middle two lines: per (128-token tile, slice of the intermediate)
// they stream 64-column chunks of A_g, A_u, B_d through an smem ring; G and U land in TMEM
// accumulators, epilogue warps apply SiLU*mul (one MUFU tanh per element) and hand the bf16 h
// chunk to the next MMA, which folds it into the T_d accumulator (TMEM). h never touches HBM;
// only the (M x r_d) partial T_d of each slice is reduced into global memory (fp32 vector reds).
//
// Three variants, chosen by the host (launch_mlp_mid / launch_mlp_mid_pair):
//   mlp_mid_pair_kernel  2x1 CTA pairs, cta_group::2 M=256 MMAs, T in TMEM, h via an smem ring,
//                        separate G/U and D issuer warps (default; see its comment block)
//   mlp_mid_ts_kernel    one CTA, T and h in TMEM (TS-mode MMAs)   — pair layout does not fit
//   mlp_mid_kernel       one CTA, everything from smem (SS MMAs)   — TS layout does not fit
// Measured on cfg3 (5120 -> 25600 -> 5120, TT r64, M = 8192): block 0.163 ms (pair) vs 0.170
// (TS) vs 0.26 (SS, first version) vs 0.51 unfused vs 4.6 dense cuBLAS; the pair kernel sits
// between two floors of similar size — the SFU (8192 tanh per chunk and CTA, 8 cycles per warp
// instruction) and the tensor pipe (>= ~44 cycles per tcgen05.mma at N <= 64,
// tools/ubench/mma*.cu).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "mlp.cuh"
#include "ptx.cuh"

namespace tnl {

namespace {

constexpr int CH = 64;                        // intermediate columns per chunk
constexpr uint32_t TBLK = 128 * 64 * 2;       // 128-row x 64-k bf16 block (16 KB)
constexpr uint32_t WBLK = 64 * 64 * 2;        // 64-row x 64-k bf16 weight block (8 KB)

__device__ __forceinline__ void nbar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct MlpLayout {
  int kg, ku, kd;  // k-blocks of r_g, r_u; r_d/64 row blocks of B_d chunk
  uint32_t stage, ag_off, au_off, bd_off;
  int stages;
  int nb;   // G/U TMEM accumulator pairs (and h smem buffers) in flight
  int lag;  // the T_d MMA of chunk i-lag is issued after the G/U MMAs of chunk i
  size_t t_bytes, total;
};

__host__ __device__ inline MlpLayout mlp_layout(const MlpArgs& a) {
  MlpLayout L;
  L.kg = a.rg / 64;
  L.ku = a.ru / 64;
  L.kd = a.rd / 64;
  L.ag_off = 0;
  L.au_off = L.kg * WBLK;
  L.bd_off = L.au_off + L.ku * WBLK;
  L.stage = L.bd_off + (uint32_t)a.rd * 128;  // B_d chunk: rd rows x 64 k (128 B rows)
  L.stage = (L.stage + 1023) / 1024 * 1024;
  L.t_bytes = (size_t)(L.kg + L.ku) * TBLK;
  L.nb = (3 * 128 + a.rd <= 512) ? 3 : 2;  // TMEM: nb x (G|U 128 cols) + T_d (rd cols)
  size_t fixed = 1024 + L.t_bytes + (size_t)L.nb * TBLK /*h*/ + 256;
  L.stages = 4;
  while (L.stages > 2 && fixed + (size_t)L.stages * L.stage > 227 * 1024) --L.stages;
  if (fixed + (size_t)L.stages * L.stage > 227 * 1024 && L.nb == 3) {
    L.nb = 2;
    fixed -= TBLK;
  }
  L.lag = L.nb - 1 < L.stages - 2 ? L.nb - 1 : L.stages - 2;
  if (L.lag < 1) L.lag = 1;
  L.total = fixed + (size_t)L.stages * L.stage;
  return L;
}

// silu(g) = g * sigmoid(g) = g * (0.5 + 0.5 tanh(g/2)): one MUFU op (tanh.approx) per element
// instead of two (ex2 + rcp) — the SFU is the epilogue's bottleneck (8192 elements per chunk).
__device__ __forceinline__ float silu(float g) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * g));
  return g * fmaf(0.5f, t, 0.5f);
}
// silu(g) * u = (g/2 * u) * (1 + tanh(g/2)): FMUL, MUFU, FMUL, FFMA per element
__device__ __forceinline__ float silu_mul(float g, float u) {
  const float a = 0.5f * g;
  float t;
#ifdef TNL_DIAG_NOTANH  // timing diagnostic only (wrong SiLU): no MUFU op
  t = fminf(fmaxf(a, -1.f), 1.f);
#else
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(a));
#endif
  const float b = a * u;
  return fmaf(b, t, b);
}

// warp 0 TMA, warp 1 MMA, warps 2..9 epilogue (two warps per TMEM lane quarter, 32 columns each)
constexpr int MLP_THREADS = 320, MLP_EPI = 256;

__global__ void __launch_bounds__(MLP_THREADS, 1)
    mlp_mid_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmAg,
                   const __grid_constant__ CUtensorMap tmAu, const __grid_constant__ CUtensorMap tmBd,
                   const MlpArgs a) {
  const MlpLayout L = mlp_layout(a);
  const int S = L.stages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sT = smem;                    // [kg blocks of T_g][ku blocks of T_u]
  const int NB = L.nb;
  uint8_t* sH = sT + L.t_bytes;          // NB x 16 KB
  uint8_t* sR = sH + NB * TBLK;          // ring stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(sR + (size_t)S * L.stage);
  uint64_t* full = bars;           // [4]
  uint64_t* empty = bars + 4;      // [4]
  uint64_t* tfull = bars + 8;
  uint64_t* gu_full = bars + 9;    // [3]
  uint64_t* gu_empty = bars + 12;  // [3]
  uint64_t* h_full = bars + 15;    // [3]
  uint64_t* h_empty = bars + 18;   // [3]
  uint64_t* td_done = bars + 21;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);

  const int tile = blockIdx.x;
  const int total_ch = a.inter / CH;
  const int c0 = blockIdx.y * a.chunks_per_slice;
  const int nch = min(total_ch, c0 + a.chunks_per_slice) - c0;
  const uint32_t warp = warp_id();
  const uint32_t stage_tx = (uint32_t)((L.kg + L.ku) * WBLK + a.rd * 128);

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmT);
    tma_prefetch_desc(&tmAg);
    tma_prefetch_desc(&tmAu);
    tma_prefetch_desc(&tmBd);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    for (int b = 0; b < 3; ++b) {
      mbar_init(&gu_full[b], 1);
      mbar_init(&gu_empty[b], 8);
      mbar_init(&h_full[b], 8);
      mbar_init(&h_empty[b], 1);
    }
    mbar_init(td_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tTD = tmem + NB * 128;  // T_d accumulator (rd columns)
  pdl_launch_dependents();

  if (nch > 0) {
    if (warp == 0) {
      if (elect_one()) {
        auto load_stage = [&](int i) {
          const int s = i % S;
          uint8_t* st = sR + (size_t)s * L.stage;
          const int col = (c0 + i) * CH;  // intermediate column of this chunk
          mbar_arrive_expect_tx(&full[s], stage_tx);
          for (int k = 0; k < L.kg; ++k) tma_load_2d(st + L.ag_off + k * WBLK, &tmAg, &full[s], k * 64, col);
          for (int k = 0; k < L.ku; ++k) tma_load_2d(st + L.au_off + k * WBLK, &tmAu, &full[s], k * 64, col);
          tma_load_2d(st + L.bd_off, &tmBd, &full[s], col, 0);
        };
        const int npre = min(nch, S);
        for (int i = 0; i < npre; ++i) load_stage(i);  // weights: before the dependency wait
        pdl_wait();
        mbar_arrive_expect_tx(tfull, (uint32_t)((L.kg + L.ku) * TBLK));
        for (int k = 0; k < L.kg + L.ku; ++k) tma_load_2d(sT + k * TBLK, &tmT, tfull, k * 64, tile * 128);
        for (int i = npre; i < nch; ++i) {
          mbar_wait(&empty[i % S], ((i / S) & 1) ^ 1);
          load_stage(i);
        }
      }
    } else if (warp == 1) {
      if (elect_one()) {
        const uint32_t idesc_gu = idesc_bf16_f32(128, CH);
        const uint32_t idesc_d = idesc_bf16_f32(128, a.rd);
        mbar_wait(tfull, 0);
        tc_fence_after();
        auto mma_d = [&](int j) {  // T_d += h_j . B_d[:, chunk j]^T, then free stage j and h_j
          const int s = j % S;
          mbar_wait(&h_full[j % NB], (j / NB) & 1);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(sH + (j % NB) * TBLK));
          const uint64_t bd = smem_desc_sw128(smem_u32(sR + (size_t)s * L.stage + L.bd_off));
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_bf16_ss(tTD, ad + 2 * k, bd + 2 * k, idesc_d, (j > 0 || k > 0) ? 1u : 0u);
          mma_commit(&h_empty[j % NB]);
          mma_commit(&empty[s]);
        };
        unsigned long long* tr = (a.trace && blockIdx.x == 0 && blockIdx.y == 0) ? a.trace : nullptr;
        for (int i = 0; i < nch; ++i) {
          const int s = i % S;
          const int b = i % NB;
          mbar_wait(&full[s], (i / S) & 1);
          if (tr && i < 256) tr[i * 4 + 0] = globaltimer();
          if (i >= NB) mbar_wait(&gu_empty[b], ((i / NB) & 1) ^ 1);
          tc_fence_after();
          uint8_t* st = sR + (size_t)s * L.stage;
          const uint32_t tG = tmem + b * 128, tU = tG + 64;
          for (int k = 0; k < L.kg; ++k) {
            const uint64_t ad = smem_desc_sw128(smem_u32(sT + k * TBLK));
            const uint64_t bd = smem_desc_sw128(smem_u32(st + L.ag_off + k * WBLK));
#pragma unroll
            for (int q = 0; q < 4; ++q) mma_bf16_ss(tG, ad + 2 * q, bd + 2 * q, idesc_gu, (k | q) != 0);
          }
          for (int k = 0; k < L.ku; ++k) {
            const uint64_t ad = smem_desc_sw128(smem_u32(sT + (L.kg + k) * TBLK));
            const uint64_t bd = smem_desc_sw128(smem_u32(st + L.au_off + k * WBLK));
#pragma unroll
            for (int q = 0; q < 4; ++q) mma_bf16_ss(tU, ad + 2 * q, bd + 2 * q, idesc_gu, (k | q) != 0);
          }
          mma_commit(&gu_full[b]);
          if (tr && i < 256) tr[i * 4 + 1] = globaltimer();
          if (i >= L.lag) mma_d(i - L.lag);
        }
        for (int j = nch - L.lag < 0 ? 0 : nch - L.lag; j < nch; ++j) mma_d(j);
        mma_commit(td_done);
      }
      __syncwarp();
    } else {
      const uint32_t q = warp & 3;
      const int lrow = q * 32 + lane_id();
      const uint32_t lane_base = (q * 32) << 16;
      unsigned long long* tr = (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && warp == 2 && lane_id() == 0) ? a.trace : nullptr;
      for (int i = 0; i < nch; ++i) {
        const int b = i % NB;
        mbar_wait(&gu_full[b], (i / NB) & 1);
        tc_fence_after();
        if (tr && i < 256) tr[i * 4 + 2] = globaltimer();
        if (i >= NB) mbar_wait(&h_empty[b], ((i / NB) & 1) ^ 1);
        if (tr && i < 256) tr[1024 + i * 4 + 2] = globaltimer();
        uint8_t* rowp = sH + b * TBLK + (lrow >> 3) * 1024 + (lrow & 7) * 128;
        const int cb = ((warp - 2) >> 2) * 32;  // this warp's 32 columns of the chunk
        const uint32_t tG = tmem + b * 128 + lane_base + cb, tU = tG + 64;
        uint32_t gr[32], ur[32];
        tmem_ld32_nowait(tG, gr);
        tmem_ld32_nowait(tU, ur);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&gu_empty[b]);  // accumulator pair b may be overwritten
        if (tr && i < 256) tr[1024 + i * 4 + 0] = globaltimer();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 p;
          float h[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            h[e] = silu(__uint_as_float(gr[8 * j + e])) * __uint_as_float(ur[8 * j + e]);
          p.x = pack_bf16x2(h[0], h[1]);
          p.y = pack_bf16x2(h[2], h[3]);
          p.z = pack_bf16x2(h[4], h[5]);
          p.w = pack_bf16x2(h[6], h[7]);
          const int ch = cb / 8 + j;
          sts128(smem_u32(rowp) + ((ch ^ (lrow & 7)) << 4), p);
        }
        if (tr && i < 256) tr[1024 + i * 4 + 1] = globaltimer();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&h_full[b]);
        if (tr && i < 256) tr[i * 4 + 3] = globaltimer();
      }
      // partial T_d (this slice of the intermediate) -> fp32 reductions
      mbar_wait(td_done, 0);
      tc_fence_after();
      const int m = tile * 128 + lrow;
      const int half = a.rd / 2;  // rd is a multiple of 64
#pragma unroll 1
      for (int c = ((warp - 2) >> 2) * half; c < ((warp - 2) >> 2) * half + half; c += 16) {
        float v[16];
        tmem_ld16(tTD + lane_base + c, v);
        if (m >= a.M) continue;
        float* o = a.td + (int64_t)m * a.ld_td + c;
#pragma unroll
        for (int e = 0; e < 16; e += 4) red_add_v4(o + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// TS variant: the T tile and h live in TMEM, so the tensor core reads only the streamed
// weight chunks from shared memory (the SS kernel above re-reads the 128-token T tile from
// smem for every chunk and round-trips h through smem: ~3x the smem traffic per chunk).
//   TMEM columns: [b*128, b*128+128) G|U accumulator pair b (NB of them; after the
//   epilogue, h_b is packed bf16 in columns b*128 + {0..15, 32..47}), then T (32 columns per
//   64-wide k-block, packed bf16 as the MMA's A operand), then T_d (rd columns).
struct MlpTsLayout {
  int kg, ku;
  uint32_t stage, ag_off, au_off, bd_off;
  int stages, nb, lag;
  uint32_t t_col, td_col;
  size_t t_bytes, total;
};

__host__ __device__ inline MlpTsLayout mlp_ts_layout(const MlpArgs& a) {
  MlpTsLayout L;
  L.kg = a.rg / 64;
  L.ku = a.ru / 64;
  L.ag_off = 0;
  L.au_off = L.kg * WBLK;
  L.bd_off = L.au_off + L.ku * WBLK;
  L.stage = (L.bd_off + (uint32_t)a.rd * 128 + 1023) / 1024 * 1024;
  L.t_bytes = (size_t)(L.kg + L.ku) * TBLK;
  const int tcols = (L.kg + L.ku) * 32;
  L.nb = (512 - tcols - a.rd) / 128;
  if (L.nb > 3) L.nb = 3;
  L.t_col = L.nb * 128;
  L.td_col = L.t_col + tcols;
  const size_t fixed = 1024 + L.t_bytes + 256;
  L.stages = 6;
  while (L.stages > 2 && fixed + (size_t)L.stages * L.stage > 227 * 1024) --L.stages;
  L.lag = L.nb - 1 < L.stages - 2 ? L.nb - 1 : L.stages - 2;
  if (L.lag < 1) L.lag = 1;
  L.total = fixed + (size_t)L.stages * L.stage;
  return L;
}

// circular-buffer position: slot index and the mbarrier phase parity of its current use
struct Ring {
  int idx = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++idx == n) {
      idx = 0;
      ph ^= 1;
    }
  }
  __device__ __forceinline__ void next2(int n) {  // two slots ahead (n >= 2)
    idx += 2;
    if (idx >= n) {
      idx -= n;
      ph ^= 1;
    }
  }
};

__global__ void __launch_bounds__(MLP_THREADS, 1)
    mlp_mid_ts_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmAg,
                      const __grid_constant__ CUtensorMap tmAu, const __grid_constant__ CUtensorMap tmBd,
                      const MlpArgs a) {
  const MlpTsLayout L = mlp_ts_layout(a);
  const int S = L.stages, NB = L.nb;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sT = smem;             // T tile staging (TMA -> smem -> TMEM)
  uint8_t* sR = sT + L.t_bytes;   // ring stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(sR + (size_t)S * L.stage);
  uint64_t* full = bars;           // [8]
  uint64_t* empty = bars + 8;      // [8]
  uint64_t* tfull = bars + 16;
  uint64_t* t_tmem = bars + 17;
  uint64_t* gu_full = bars + 18;   // [3]
  uint64_t* gu_empty = bars + 21;  // [3]
  uint64_t* h_full = bars + 24;    // [3]
  uint64_t* td_done = bars + 27;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);

  const int tile = blockIdx.x;
  const int total_ch = a.inter / CH;
  const int c0 = blockIdx.y * a.chunks_per_slice;
  const int nch = min(total_ch, c0 + a.chunks_per_slice) - c0;
  const uint32_t warp = warp_id();
  const uint32_t stage_tx = (uint32_t)((L.kg + L.ku) * WBLK + a.rd * 128);

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmT);
    tma_prefetch_desc(&tmAg);
    tma_prefetch_desc(&tmAu);
    tma_prefetch_desc(&tmBd);
    for (int s = 0; s < 8; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(t_tmem, 8);
    for (int b = 0; b < 3; ++b) {
      mbar_init(&gu_full[b], 1);
      mbar_init(&gu_empty[b], 1);
      mbar_init(&h_full[b], 4);
    }
    mbar_init(td_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tT = tmem + L.t_col, tTD = tmem + L.td_col;
  pdl_launch_dependents();

  if (nch > 0) {
    if (warp == 0) {
      if (elect_one()) {
        Ring r;
        auto load_stage = [&](int i) {
          const int s = r.idx;
          uint8_t* st = sR + (size_t)s * L.stage;
          const int col = (c0 + i) * CH;
          mbar_arrive_expect_tx(&full[s], stage_tx);
          for (int k = 0; k < L.kg; ++k) tma_load_2d(st + L.ag_off + k * WBLK, &tmAg, &full[s], k * 64, col);
          for (int k = 0; k < L.ku; ++k) tma_load_2d(st + L.au_off + k * WBLK, &tmAu, &full[s], k * 64, col);
          tma_load_2d(st + L.bd_off, &tmBd, &full[s], col, 0);
          r.next(S);
        };
        const int npre = min(nch, S);
        for (int i = 0; i < npre; ++i) load_stage(i);  // weights: before the dependency wait
        pdl_wait();
        mbar_arrive_expect_tx(tfull, (uint32_t)((L.kg + L.ku) * TBLK));
        for (int k = 0; k < L.kg + L.ku; ++k) tma_load_2d(sT + k * TBLK, &tmT, tfull, k * 64, tile * 128);
        for (int i = npre; i < nch; ++i) {
          mbar_wait(&empty[r.idx], r.ph ^ 1);
          load_stage(i);
        }
      }
    } else if (warp == 1) {
      if (elect_one()) {
        const uint32_t idesc_gu = idesc_bf16_f32(128, CH);
        const uint32_t idesc_d = idesc_bf16_f32(128, a.rd);
        mbar_wait(t_tmem, 0);
        tc_fence_after();
        Ring rf, rb, js, jb;  // G/U side: stage, pair; T_d side: stage, pair
        auto mma_d = [&](int j) {  // T_d += h_j . B_d[:, chunk j]^T; frees stage j and pair j
          mbar_wait(&h_full[jb.idx], jb.ph);
          tc_fence_after();
          const uint32_t th = tmem + jb.idx * 128;
          const uint64_t bd = smem_desc_sw128(smem_u32(sR + (size_t)js.idx * L.stage + L.bd_off));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_bf16_ts(tTD, th + (k >> 1) * 32 + (k & 1) * 8, bd + 2 * k, idesc_d, (j > 0 || k > 0) ? 1u : 0u);
          mma_commit(&gu_empty[jb.idx]);
          mma_commit(&empty[js.idx]);
          js.next(S);
          jb.next(NB);
        };
        unsigned long long* tr = (a.trace && blockIdx.x == 0 && blockIdx.y == 0) ? a.trace : nullptr;
        for (int i = 0; i < nch; ++i) {
          const int s = rf.idx, b = rb.idx;
          mbar_wait(&full[s], rf.ph);
          if (tr && i < 256) tr[i * 4 + 0] = globaltimer();
          if (i >= NB) mbar_wait(&gu_empty[b], rb.ph ^ 1);
          rf.next(S);
          rb.next(NB);
          tc_fence_after();
          uint8_t* st = sR + (size_t)s * L.stage;
          const uint32_t tG = tmem + b * 128, tU = tG + 64;
          for (int k = 0; k < L.kg; ++k) {
            const uint64_t bd = smem_desc_sw128(smem_u32(st + L.ag_off + k * WBLK));
#pragma unroll
            for (int q = 0; q < 4; ++q) mma_bf16_ts(tG, tT + k * 32 + q * 8, bd + 2 * q, idesc_gu, (k | q) != 0);
          }
          for (int k = 0; k < L.ku; ++k) {
            const uint64_t bd = smem_desc_sw128(smem_u32(st + L.au_off + k * WBLK));
#pragma unroll
            for (int q = 0; q < 4; ++q)
              mma_bf16_ts(tU, tT + (L.kg + k) * 32 + q * 8, bd + 2 * q, idesc_gu, (k | q) != 0);
          }
          mma_commit(&gu_full[b]);
          if (tr && i < 256) tr[i * 4 + 1] = globaltimer();
          if (i >= L.lag) mma_d(i - L.lag);
        }
        for (int j = nch - L.lag < 0 ? 0 : nch - L.lag; j < nch; ++j) mma_d(j);
        mma_commit(td_done);
      }
      __syncwarp();
    } else {
      const uint32_t q = warp & 3, hh = (warp - 2) >> 2;
      const int lrow = q * 32 + lane_id();
      const uint32_t lane_base = (q * 32) << 16;
      // T tile: smem (SW128, k-blocks of 64) -> TMEM (packed bf16 pairs, 32 columns per k-block)
      mbar_wait(tfull, 0);
      for (int kb = hh; kb < L.kg + L.ku; kb += 2) {
        const uint8_t* rowp = sT + kb * TBLK + (lrow >> 3) * 1024 + (lrow & 7) * 128;
        uint32_t r[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 v = lds128(smem_u32(rowp) + ((c ^ (lrow & 7)) << 4));
          r[4 * c] = v.x;
          r[4 * c + 1] = v.y;
          r[4 * c + 2] = v.z;
          r[4 * c + 3] = v.w;
        }
        tmem_st32(tT + lane_base + kb * 32, r);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(t_tmem);
      unsigned long long* tr = (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && (warp == 2 || warp == 6) && lane_id() == 0) ? a.trace : nullptr;
      // the two epilogue warps of a lane quarter take alternate chunks (all 64 columns each),
      // so one warp's SFU work overlaps the other's TMEM round trips and barrier waits
      Ring eb;
      eb.idx = hh;
      for (int i = hh; i < nch; i += 2) {
        const int b = eb.idx;
        mbar_wait(&gu_full[b], eb.ph);
        eb.next2(NB);
        tc_fence_after();
        if (tr && i < 256) tr[i * 4 + 2] = globaltimer();
        const uint32_t tG = tmem + b * 128 + lane_base, tU = tG + 64;
        uint32_t gr[64], ur[64];
        tmem_ld32_nowait(tG, gr);
        tmem_ld32_nowait(tU, ur);
        tmem_ld32_nowait(tG + 32, gr + 32);
        tmem_ld32_nowait(tU + 32, ur + 32);
        tmem_wait_ld();
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t hp[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            hp[e] = pack_bf16x2(silu(__uint_as_float(gr[32 * hf + 2 * e])) * __uint_as_float(ur[32 * hf + 2 * e]),
                                silu(__uint_as_float(gr[32 * hf + 2 * e + 1])) * __uint_as_float(ur[32 * hf + 2 * e + 1]));
          tmem_st16(tG + hf * 32, hp);  // h over already-read G columns
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&h_full[b]);
        if (tr && i < 256) tr[i * 4 + 3] = globaltimer();
      }
      mbar_wait(td_done, 0);
      tc_fence_after();
      const int m = tile * 128 + lrow;
      const int half = a.rd / 2;
#pragma unroll 1
      for (int c = hh * half; c < hh * half + half; c += 16) {
        float v[16];
        tmem_ld16(tTD + lane_base + c, v);
        if (m >= a.M) continue;
        float* o = a.td + (int64_t)m * a.ld_td + c;
#pragma unroll
        for (int e = 0; e < 16; e += 4) red_add_v4(o + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// Pair variant (cta_group::2): the two CTAs of a 2x1 cluster (one TPC) run M=256 MMAs over
// their two 128-token tiles. A tcgen05.mma costs >= ~44 cycles however small N is (measured:
// tools/ubench/mma*.cu), so at N=64 one pair instruction doing both SMs' work halves the
// tensor-pipe time per token; each CTA also streams only HALF of every weight chunk (A_g/A_u:
// 32 of the 64 chunk rows, B_d: r_d/2 rows). T (the G/U A operand) lives in TMEM; h is written
// by the epilogue into a 128B-swizzled smem ring (the D MMA's A operand), so a G/U TMEM pair is
// released as soon as the epilogue has loaded it rather than after the D MMA — the MMA warp's
// waits are then normally already satisfied. The leader (rank 0) issues every MMA and owns
// full / t_tmem / gu_empty / h_full; MMA completions are multicast to both CTAs.
constexpr uint32_t HBLK = 32 * 128;  // 32-row x 64-k bf16 half weight block (4 KB)
// warp 0 TMA, warp 1 G/U MMA issuer, warps 2..9 epilogue, warp 10 D MMA issuer
constexpr int MLP_PAIR_THREADS = 352;

struct MlpPairLayout {
  int kg, ku;
  uint32_t stage, ag_off, au_off, bd_off, stage_tx;  // stage_tx: bytes per CTA
  int stages, nb, nh, lag;
  uint32_t t_col, td_col;
  size_t t_bytes, h_off, total;
};

__host__ __device__ inline MlpPairLayout mlp_pair_layout(const MlpArgs& a) {
  MlpPairLayout L;
  L.kg = a.rg / 64;
  L.ku = a.ru / 64;
  L.ag_off = 0;
  L.au_off = L.kg * HBLK;
  L.bd_off = L.au_off + L.ku * HBLK;
  L.stage_tx = L.bd_off + (uint32_t)(a.rd / 2) * 128;
  L.stage = (L.stage_tx + 1023) / 1024 * 1024;
  L.t_bytes = (size_t)(L.kg + L.ku) * TBLK;
  const int tcols = (L.kg + L.ku) * 32;
  L.nb = (512 - tcols - a.rd) / 128;
  if (L.nb > 3) L.nb = 3;
  L.nh = 3;
  L.t_col = L.nb * 128;
  L.td_col = L.t_col + tcols;
  L.h_off = L.t_bytes;
  const size_t fixed = 1024 + L.t_bytes + (size_t)L.nh * TBLK + 512;
  L.stages = 12;
  while (L.stages > 3 && fixed + (size_t)L.stages * L.stage > 227 * 1024) --L.stages;
  L.lag = 2;
  L.total = fixed + (size_t)L.stages * L.stage;
  return L;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(MLP_PAIR_THREADS, 1)
    mlp_mid_pair_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmAg,
                        const __grid_constant__ CUtensorMap tmAu, const __grid_constant__ CUtensorMap tmBd,
                        const MlpArgs a) {
  const MlpPairLayout L = mlp_pair_layout(a);
  const int S = L.stages, NB = L.nb, NH = L.nh;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sT = smem;                 // own T tile (TMA -> smem -> TMEM)
  uint8_t* sH = smem + L.h_off;       // NH x 16 KB h ring (own 128 rows)
  uint8_t* sR = sH + NH * TBLK;       // weight ring (own halves)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sR + (size_t)S * L.stage);
  uint64_t* full = bars;           // [12] leader: both CTAs' weight bytes
  uint64_t* empty = bars + 12;     // [12] per CTA (multicast commit)
  uint64_t* tfull = bars + 24;     //      per CTA (own T tile)
  uint64_t* t_tmem = bars + 25;    //      leader: T copied into TMEM in both CTAs (16 warps)
  uint64_t* gu_full = bars + 26;   // [3]  per CTA (multicast commit)
  uint64_t* gu_empty = bars + 29;  // [3]  leader: G/U pair loaded by both CTAs' epilogues (8 warps)
  uint64_t* h_full = bars + 32;    // [3]  leader: h chunk written in both CTAs (8 warps)
  uint64_t* h_empty = bars + 35;   // [3]  per CTA (multicast commit of the D MMA)
  uint64_t* td_done = bars + 38;   //      per CTA (multicast commit): an item's T_d complete
  uint64_t* t_copied = bars + 39;  //      per CTA: the item's T read out of sT by the 8 epilogue warps
  uint64_t* t_free = bars + 40;    //      per CTA (multicast commit): the item's G/U MMAs done (TMEM T free)
  uint64_t* td_empty = bars + 41;  //      leader: both CTAs' epilogues read the item's T_d (16 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 42);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int total_ch = a.inter / CH;
  const uint32_t warp = warp_id();
  // Work of this CTA pair: a contiguous range of the (token-pair tile, 64-column chunk) sequence.
  // Slice mode: one token pair, chunk slice blockIdx.y. Balanced mode (a.per_pair > 0): per_pair
  // chunk-units from the flattened sequence, split into items at token-pair boundaries, so every
  // pair of the grid (74 on 148 SMs) does the same amount of work whatever the token count.
  const int pair_id = blockIdx.x >> 1;
  int64_t w_beg, w_end;
  if (a.per_pair > 0) {
    w_beg = (int64_t)pair_id * a.per_pair;
    w_end = min((int64_t)a.tiles2 * total_ch, w_beg + a.per_pair);
  } else {
    w_beg = (int64_t)pair_id * total_ch + (int64_t)blockIdx.y * a.chunks_per_slice;
    w_end = min((int64_t)(pair_id + 1) * total_ch, w_beg + a.chunks_per_slice);
  }
  auto next_item = [&](int64_t& w, int& tile, int& c0, int& nch) -> bool {
    if (w >= w_end) return false;
    const int tp = (int)(w / total_ch);
    c0 = (int)(w % total_ch);
    nch = (int)min(w_end - w, (int64_t)(total_ch - c0));
    tile = 2 * tp + (int)rank;  // this CTA's 128-token tile of the pair
    w += nch;
    return true;
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmT);
    tma_prefetch_desc(&tmAg);
    tma_prefetch_desc(&tmAu);
    tma_prefetch_desc(&tmBd);
    for (int s = 0; s < 12; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // G/U issuer + D issuer
    }
    mbar_init(tfull, 1);
    mbar_init(t_tmem, 16);
    for (int b = 0; b < 3; ++b) {
      mbar_init(&gu_full[b], 1);
      mbar_init(&gu_empty[b], 8);
      mbar_init(&h_full[b], 8);
      mbar_init(&h_empty[b], 1);
    }
    mbar_init(td_done, 1);
    mbar_init(t_copied, 8);
    mbar_init(t_free, 1);
    mbar_init(td_empty, 16);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive / multicast commit
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tT = tmem + L.t_col, tTD = tmem + L.td_col;
  pdl_launch_dependents();

  if (w_beg < w_end) {
    if (warp == 0) {
      if (elect_one()) {
        Ring r;
        const int wrow = (int)rank * 32, drow = (int)rank * (a.rd / 2);
        int gi = 0;  // weight stages issued
        auto load_stage = [&](int chunk) {
          const int s = r.idx;
          if (gi >= S) mbar_wait(&empty[s], r.ph ^ 1);
          uint8_t* st = sR + (size_t)s * L.stage;
          const int col = chunk * CH;
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * L.stage_tx);
          for (int k = 0; k < L.kg; ++k) tma_load_2d_pair(st + L.ag_off + k * HBLK, &tmAg, &full[s], k * 64, col + wrow);
          for (int k = 0; k < L.ku; ++k) tma_load_2d_pair(st + L.au_off + k * HBLK, &tmAu, &full[s], k * 64, col + wrow);
          tma_load_2d_pair(st + L.bd_off, &tmBd, &full[s], col, drow);
          r.next(S);
          ++gi;
        };
        int64_t w = w_beg;
        int tile, c0, nch, k = 0;
        while (next_item(w, tile, c0, nch)) {
          int i = 0;
          if (k == 0) {
            for (; i < min(nch, S); ++i) load_stage(c0 + i);  // weights: before the dependency wait
            pdl_wait();
          } else {
            mbar_wait(t_copied, (k - 1) & 1);  // the previous item's T has left sT
          }
          mbar_arrive_expect_tx(tfull, (uint32_t)((L.kg + L.ku) * TBLK));
          for (int kb = 0; kb < L.kg + L.ku; ++kb) tma_load_2d(sT + kb * TBLK, &tmT, tfull, kb * 64, tile * 128);
          for (; i < nch; ++i) load_stage(c0 + i);
          ++k;
        }
      }
    } else if (warp == 1) {
      // G/U issuer: G_i = T_g A_g[chunk i]^T, U_i = T_u A_u[chunk i]^T into TMEM pair i % NB
      if (leader && elect_one()) {
        const uint32_t idesc_gu = idesc_bf16_f32(256, CH);
        Ring rf, rb;
        int gi = 0;
        int64_t w = w_beg;
        int tile, c0, nch, k = 0;
        while (next_item(w, tile, c0, nch)) {
          mbar_wait(t_tmem, k & 1);
          tc_fence_after();
          for (int i = 0; i < nch; ++i, ++gi) {
            const int s = rf.idx, b = rb.idx;
            mbar_wait(&full[s], rf.ph);
            if (gi >= NB) mbar_wait(&gu_empty[b], rb.ph ^ 1);
            rf.next(S);
            rb.next(NB);
            tc_fence_after();
            uint8_t* st = sR + (size_t)s * L.stage;
            const uint32_t tG = tmem + b * 128, tU = tG + 64;
            for (int kk = 0; kk < L.kg; ++kk) {
              const uint64_t bd = smem_desc_sw128(smem_u32(st + L.ag_off + kk * HBLK));
#pragma unroll
              for (int q = 0; q < 4; ++q) mma_bf16_ts_pair(tG, tT + kk * 32 + q * 8, bd + 2 * q, idesc_gu, (kk | q) != 0);
            }
            for (int kk = 0; kk < L.ku; ++kk) {
              const uint64_t bd = smem_desc_sw128(smem_u32(st + L.au_off + kk * HBLK));
#pragma unroll
              for (int q = 0; q < 4; ++q)
                mma_bf16_ts_pair(tU, tT + (L.kg + kk) * 32 + q * 8, bd + 2 * q, idesc_gu, (kk | q) != 0);
            }
            mma_commit_pair(&gu_full[b], 3);
            mma_commit_pair(&empty[s], 3);
          }
          mma_commit_pair(t_free, 3);  // every G/U MMA of this item has read the TMEM T tile
          ++k;
        }
      }
      __syncwarp();
    } else if (warp == MLP_PAIR_THREADS / 32 - 1) {
      // D issuer: T_d += h_j B_d[:, chunk j]^T (A = h from the smem ring); its own warp (SMSP)
      // so the two MMA chains interleave on the tensor pipe instead of serialising
      if (leader && elect_one()) {
        const uint32_t idesc_d = idesc_bf16_f32(256, a.rd);
        Ring rf, rh;
        int64_t w = w_beg;
        int tile, c0, nch, k = 0;
        while (next_item(w, tile, c0, nch)) {
          if (k > 0) mbar_wait_cluster(td_empty, (k - 1) & 1);  // previous item's T_d read out
          tc_fence_after();
          for (int j = 0; j < nch; ++j) {
            const int s = rf.idx, hb = rh.idx;
            mbar_wait(&full[s], rf.ph);
            mbar_wait(&h_full[hb], rh.ph);
            rf.next(S);
            rh.next(NH);
            tc_fence_after();
            const uint64_t ad = smem_desc_sw128(smem_u32(sH + hb * TBLK));
            const uint64_t bd = smem_desc_sw128(smem_u32(sR + (size_t)s * L.stage + L.bd_off));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ss_pair(tTD, ad + 2 * kk, bd + 2 * kk, idesc_d, (j > 0 || kk > 0) ? 1u : 0u);
            mma_commit_pair(&h_empty[hb], 3);
            mma_commit_pair(&empty[s], 3);
          }
          mma_commit_pair(td_done, 3);
          ++k;
        }
      }
      __syncwarp();
    } else {
      const uint32_t q = warp & 3, hh = (warp - 2) >> 2;
      const int lrow = q * 32 + lane_id();
      const uint32_t lane_base = (q * 32) << 16;
      // the two epilogue warps of a lane quarter take alternate chunks of the CTA's chunk sequence
      Ring eb, ehb;
      eb.idx = hh;
      ehb.idx = hh;
      int g = 0;  // chunks of previous items
      int64_t w = w_beg;
      int tile, c0, nch, k = 0;
      while (next_item(w, tile, c0, nch)) {
        // T tile: smem (SW128, k-blocks of 64) -> TMEM (packed bf16 pairs, 32 columns per k-block)
        mbar_wait(tfull, k & 1);
        if (k > 0) mbar_wait(t_free, (k - 1) & 1);  // the previous item's G/U MMAs no longer read TMEM T
        for (int kb = hh; kb < L.kg + L.ku; kb += 2) {
          const uint8_t* rowp = sT + kb * TBLK + (lrow >> 3) * 1024 + (lrow & 7) * 128;
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = lds128(smem_u32(rowp) + ((c ^ (lrow & 7)) << 4));
            r[4 * c] = v.x;
            r[4 * c + 1] = v.y;
            r[4 * c + 2] = v.z;
            r[4 * c + 3] = v.w;
          }
          tmem_st32(tT + lane_base + kb * 32, r);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) {
          mbar_arrive_remote(mapa_shared(t_tmem, 0));
          mbar_arrive(t_copied);
        }
        for (int i = (int)((hh + g) & 1); i < nch; i += 2) {  // global chunk g + i has parity hh
          const int gg = g + i;
          const int b = eb.idx, hb = ehb.idx;
          const uint32_t hph = ehb.ph;
          mbar_wait(&gu_full[b], eb.ph);
          eb.next2(NB);
          ehb.next2(NH);
          tc_fence_after();
          const uint32_t tG = tmem + b * 128 + lane_base, tU = tG + 64;
          uint32_t gr[64], ur[64];
          tmem_ld32_nowait(tG, gr);
          tmem_ld32_nowait(tU, ur);
          tmem_ld32_nowait(tG + 32, gr + 32);
          tmem_ld32_nowait(tU + 32, ur + 32);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive_remote(mapa_shared(&gu_empty[b], 0));  // pair b reusable
          if (gg >= NH) mbar_wait(&h_empty[hb], hph ^ 1);
          uint8_t* rowp = sH + hb * TBLK + (lrow >> 3) * 1024 + (lrow & 7) * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint4 p;
            p.x = pack_bf16x2(silu_mul(__uint_as_float(gr[8 * c + 0]), __uint_as_float(ur[8 * c + 0])),
                              silu_mul(__uint_as_float(gr[8 * c + 1]), __uint_as_float(ur[8 * c + 1])));
            p.y = pack_bf16x2(silu_mul(__uint_as_float(gr[8 * c + 2]), __uint_as_float(ur[8 * c + 2])),
                              silu_mul(__uint_as_float(gr[8 * c + 3]), __uint_as_float(ur[8 * c + 3])));
            p.z = pack_bf16x2(silu_mul(__uint_as_float(gr[8 * c + 4]), __uint_as_float(ur[8 * c + 4])),
                              silu_mul(__uint_as_float(gr[8 * c + 5]), __uint_as_float(ur[8 * c + 5])));
            p.w = pack_bf16x2(silu_mul(__uint_as_float(gr[8 * c + 6]), __uint_as_float(ur[8 * c + 6])),
                              silu_mul(__uint_as_float(gr[8 * c + 7]), __uint_as_float(ur[8 * c + 7])));
            sts128(smem_u32(rowp) + ((c ^ (lrow & 7)) << 4), p);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive_remote(mapa_shared(&h_full[hb], 0));
        }
        g += nch;
        // this item's T_d partial (the 128 rows of `tile`) -> fp32 reductions; then hand the TMEM
        // accumulator back to the D issuer for the next item
        mbar_wait(td_done, k & 1);
        tc_fence_after();
        const int m = tile * 128 + lrow;
        const int half = a.rd / 2;
#pragma unroll 1
        for (int c = hh * half; c < hh * half + half; c += 16) {
          float v[16];
          tmem_ld16(tTD + lane_base + c, v);
          if (m >= a.M) continue;
          float* o = a.td + (int64_t)m * a.ld_td + c;
#pragma unroll
          for (int e = 0; e < 16; e += 4) red_add_v4(o + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive_remote(mapa_shared(td_empty, 0));
        ++k;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_pair<512>(tmem);
}

}  // namespace

size_t mlp_mid_smem(const MlpArgs& a) {
  const MlpTsLayout Lt = mlp_ts_layout(a);
  return Lt.nb >= 2 ? Lt.total : mlp_layout(a).total;
}

int launch_mlp_mid(const CUtensorMap& t, const CUtensorMap& ag, const CUtensorMap& au, const CUtensorMap& bd,
                   const MlpArgs& a, int slices, cudaStream_t st) {
  const MlpLayout L = mlp_layout(a);
  if (a.rg % 64 || a.ru % 64 || a.rd % 64 || a.rg > 128 || a.ru > 128 || a.rd > 256 || a.inter % CH ||
      L.total > 227 * 1024)
    return (int)cudaErrorInvalidValue;
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(mlp_mid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mlp_mid_ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  const MlpTsLayout Lt = mlp_ts_layout(a);
  static const int ts_env = getenv("TNL_MLP_SS") ? 0 : 1;
  const bool ts = ts_env && Lt.nb >= 2 && Lt.total <= 227 * 1024;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.M + 127) / 128, slices, 1);
  cfg.blockDim = dim3(MLP_THREADS, 1, 1);
  cfg.dynamicSmemBytes = ts ? Lt.total : L.total;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = ts ? cudaLaunchKernelEx(&cfg, mlp_mid_ts_kernel, t, ag, au, bd, a)
                     : cudaLaunchKernelEx(&cfg, mlp_mid_kernel, t, ag, au, bd, a);
  count_launch();
  return (int)e;
}

}  // namespace tnl

namespace tnl {

bool mlp_pair_ok(const MlpArgs& a) {
  static const bool nopair = getenv("TNL_MLP_NOPAIR") != nullptr;  // A/B switch for measurements
  if (nopair) return false;
  const MlpPairLayout L = mlp_pair_layout(a);
  return L.nb >= 2 && L.total <= 227 * 1024 && a.rg % 64 == 0 && a.ru % 64 == 0 && a.rd % 64 == 0 &&
         a.rg <= 128 && a.ru <= 128 && a.rd <= 256 && a.inter % CH == 0;
}

int launch_mlp_mid_pair(const CUtensorMap& t, const CUtensorMap& ag, const CUtensorMap& au, const CUtensorMap& bd,
                        const MlpArgs& a, int slices, cudaStream_t st) {
  if (!mlp_pair_ok(a)) return (int)cudaErrorInvalidValue;
  const MlpPairLayout L = mlp_pair_layout(a);
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(mlp_mid_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  const int tiles = (a.M + 127) / 128;
  cudaLaunchConfig_t cfg = {};
  // balanced mode: a.per_pair chunk-units per CTA pair over the flattened (token pair, chunk) sequence
  const int64_t work = (int64_t)((tiles + 1) / 2) * (a.inter / CH);
  cfg.gridDim = a.per_pair > 0 ? dim3((unsigned)(2 * ((work + a.per_pair - 1) / a.per_pair)), 1, 1)
                               : dim3((tiles + 1) / 2 * 2, slices, 1);
  cfg.blockDim = dim3(MLP_PAIR_THREADS, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, mlp_mid_pair_kernel, t, ag, au, bd, a);
  count_launch();
  return (int)e;
}

}  // namespace tnl
