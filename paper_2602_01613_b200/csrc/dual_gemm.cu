// dual_gemm.cu — gate/up output GEMMs of a TN MLP block fused with SiLU*mul (prefill).
//
//   h[i][j] = silu( sum_k T[i][k] * A_g[j][k] ) * ( sum_k T[i][rg + k] * A_u[j][k] )
//
// T = x [B_g; B_u]^T is the concatenated cut activation (M x (rg + ru), bf16), A_g / A_u the gate
// and up output panels (inter x r_pad). This is the MLP path for rank layouts the on-chip
// middle kernel (mlp.cu) cannot hold (cut ranks > 128, or r_d > 128 with gate/up 128): instead of
// writing g and u (2 x M x inter) and re-reading both for a separate SiLU*mul pass, each output
// tile accumulates G and U side by side in TMEM and the epilogue writes h once.
//
// One CTA per (token tile, slice of output tiles); its T tile stays resident in smem (the
// re-streamed T tile made the first, persistent version L2-bandwidth bound). Warp 0: TMA producer
// (A_g / A_u k-blocks through a 4-deep ring, weights prefetched before the dependency wait);
// warp 1: MMA issuer (128 x 128 x 16) into two double-buffered accumulator pairs (G | U = 256
// columns each, 512 total) so the epilogue of tile t overlaps the MMAs of tile t+1; warps 2-5:
// epilogue tcgen05.ld G and U -> silu(g) * u (one tanh.approx per element) -> bf16 ->
// 128B-swizzled staging -> TMA store.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tnl {

namespace {

constexpr int DBM = 128, DBN = 128, DBK = 64, DSTAGES = 8, DMAXKB = 8;
constexpr int DUAL_THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (two column halves)
constexpr uint32_t D_BLK = DBM * DBK * 2;   // 128 x 64 bf16 block (16 KB): a T k-block or a B stage
constexpr uint32_t D_HBLK = (DBN / 2) * DBK * 2;  // 64 x 64 bf16 half B block (8 KB, this CTA's rows)
constexpr uint32_t D_CHUNK = DBM * 64 * 2;  // 128 rows x 64 bf16 staging chunk
constexpr size_t D_SMEM = 1024 + (size_t)DMAXKB * D_BLK + (size_t)DSTAGES * D_HBLK + 2 * D_CHUNK + 256;

__device__ __forceinline__ void dbar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ float silu_mul(float g, float u) {
  const float a = 0.5f * g;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(a));
  const float b = a * u;
  return fmaf(b, t, b);  // g/2 * u * (1 + tanh(g/2)) = silu(g) * u
}

// grid (tiles_m rounded up to even, slices), 2x1 clusters: the two CTAs of a pair own two
// 128-token T tiles (resident in their smem) and walk the same output tiles
// [s * per, (s + 1) * per) of their rows with M=256 cta_group::2 MMAs; each CTA streams only half
// of every A_g / A_u block (64 of the 128 rows), so the L2->SM weight traffic per token halves —
// the kernel's bound once the T tile stopped being re-streamed. The leader issues the MMAs and
// owns full / tload / tempty; MMA completions are multicast to both CTAs.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(DUAL_THREADS, 1)
    dual_silu_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmG,
                     const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmH,
                     const DualArgs a, int tiles_n, int per, int per_pair) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sT = smem;                    // kg + ku resident T k-blocks (own 128 rows)
  uint8_t* sB = sT + DMAXKB * D_BLK;     // B ring (own 64-row halves, 8 KB per stage)
  uint8_t* sC = sB + DSTAGES * D_HBLK;   // 2 staging chunks
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + 2 * D_CHUNK);
  uint64_t* empty = full + DSTAGES;
  uint64_t* tfull = empty + DSTAGES;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]  leader: 4 epilogue warps x 2 CTAs
  uint64_t* tload = tempty + 2;       //      leader: both CTAs' T tiles
  uint64_t* t_free = tload + 1;       //      per CTA (multicast commit): an item's MMAs done, sT reusable
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_free + 1);

  const int kg = (a.kg + DBK - 1) / DBK, ku = (a.ku + DBK - 1) / DBK, nkb = kg + ku;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const uint32_t warp = warp_id();
  // Work of this CTA pair: a contiguous range of the flattened (token-pair tile, output tile)
  // sequence — one token pair's slice [y * per, (y+1) * per) of output tiles, or (balanced,
  // per_pair > 0) an even share over the whole grid, cut into items at token-pair boundaries
  // (each item reloads the resident T tile).
  const int pair_id = blockIdx.x >> 1, tiles2 = (a.M + 2 * DBM - 1) / (2 * DBM);
  int w_beg, w_end;
  if (per_pair > 0) {
    w_beg = pair_id * per_pair;
    w_end = min(tiles2 * tiles_n, w_beg + per_pair);
  } else {
    w_beg = pair_id * tiles_n + blockIdx.y * per;
    w_end = min((pair_id + 1) * tiles_n, w_beg + per);
  }
  auto next_item = [&](int& w, int& tm, int& tn0, int& tn1) -> bool {
    if (w >= w_end) return false;
    const int tp = w / tiles_n;
    tn0 = w % tiles_n;
    tn1 = min(tiles_n, tn0 + (w_end - w));
    tm = 2 * tp + (int)rank;
    w += tn1 - tn0;
    return true;
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmT);
    tma_prefetch_desc(&tmG);
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmH);
    for (int s = 0; s < DSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 16);  // 8 epilogue warps x 2 CTAs
    }
    mbar_init(tload, 1);
    mbar_init(t_free, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      const int hrow = (int)rank * (DBN / 2);
      auto load_b = [&](int tn, int kb) {
        const int s = it % DSTAGES;
        if (it >= DSTAGES) mbar_wait(&empty[s], ((it / DSTAGES) & 1) ^ 1);
        if (leader) mbar_arrive_expect_tx(&full[s], 2 * D_HBLK);
        const bool up = kb >= kg;
        tma_load_2d_pair(sB + s * D_HBLK, up ? &tmU : &tmG, &full[s], (up ? kb - kg : kb) * DBK, tn * DBN + hrow);
        ++it;
      };
      int w = w_beg, tm, tn0, tn1, k = 0;
      while (next_item(w, tm, tn0, tn1)) {
        const int n = (tn1 - tn0) * nkb;
        const int pre = min(DSTAGES, n);
        for (int i = 0; i < pre; ++i) load_b(tn0 + i / nkb, i % nkb);  // weights before the T wait
        if (k == 0)
          pdl_wait();
        else
          mbar_wait(t_free, (k - 1) & 1);  // the previous item's MMAs no longer read sT
        if (leader) mbar_arrive_expect_tx(tload, 2 * nkb * D_BLK);
        for (int kb = 0; kb < nkb; ++kb)
          tma_load_2d_pair(sT + kb * D_BLK, &tmT, tload, (kb >= kg ? a.u_off + (kb - kg) * DBK : kb * DBK), tm * DBM);
        for (int i = pre; i < n; ++i) load_b(tn0 + i / nkb, i % nkb);
        ++k;
      }
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(2 * DBM, DBN);
      int it = 0, lt = 0;
      int w = w_beg, tm, tn0, tn1, k = 0;
      while (next_item(w, tm, tn0, tn1)) {
      mbar_wait(tload, k & 1);
      tc_fence_after();
      for (int tn = tn0; tn < tn1; ++tn, ++lt) {
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % DSTAGES;
          mbar_wait(&full[s], (it / DSTAGES) & 1);
          tc_fence_after();
          const bool up = kb >= kg;
          const uint32_t d = tmem + acc * 2 * DBN + (up ? DBN : 0);
          const int k0 = up ? kb - kg : kb;
          const uint64_t adesc = smem_desc_sw128(smem_u32(sT + kb * D_BLK));
          const uint64_t bdesc = smem_desc_sw128(smem_u32(sB + s * D_HBLK));
#pragma unroll
          for (int k = 0; k < DBK / 16; ++k)
            mma_bf16_ss_pair(d, adesc + 2 * k, bdesc + 2 * k, idesc, (k0 > 0 || k > 0) ? 1u : 0u);
          mma_commit_pair(&empty[s], 3);
        }
        mma_commit_pair(&tfull[acc], 3);
      }
      mma_commit_pair(t_free, 3);  // every MMA of this item has read the resident T tile
      ++k;
      }
    }
    __syncwarp();
  } else {
    // warps 2-9: lane quarter q, column half hf (64 of the tile's 128 columns, staging buffer hf)
    const uint32_t q = warp & 3, hf = (warp - 2) >> 2;
    const int et = threadIdx.x - 64 - (int)hf * 128;  // 0..127 within the half's group
    const int lrow = q * 32 + lane_id();
    uint8_t* stage = sC + hf * D_CHUNK;
    int lt = 0;
    int w = w_beg, tm, tn0, tn1;
    while (next_item(w, tm, tn0, tn1))
    for (int tn = tn0; tn < tn1; ++tn, ++lt) {
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t dg = tmem + acc * 2 * DBN + ((q * 32) << 16) + hf * 64, du = dg + DBN;
      if (et == 0) tma_store_wait_read();  // this group's previous store has read the staging buffer
      dbar(1 + hf, 128);
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t gr[32], ur[32];
        tmem_ld32_nowait(dg + c, gr);
        tmem_ld32_nowait(du + c, ur);
        tmem_wait_ld();
        if (c == 32) {
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive_remote(mapa_shared(&tempty[acc], 0));
        }
        uint8_t* rowp = stage + (lrow >> 3) * 1024 + (lrow & 7) * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 p;
          p.x = pack_bf16x2(silu_mul(__uint_as_float(gr[8 * j + 0]), __uint_as_float(ur[8 * j + 0])),
                            silu_mul(__uint_as_float(gr[8 * j + 1]), __uint_as_float(ur[8 * j + 1])));
          p.y = pack_bf16x2(silu_mul(__uint_as_float(gr[8 * j + 2]), __uint_as_float(ur[8 * j + 2])),
                            silu_mul(__uint_as_float(gr[8 * j + 3]), __uint_as_float(ur[8 * j + 3])));
          p.z = pack_bf16x2(silu_mul(__uint_as_float(gr[8 * j + 4]), __uint_as_float(ur[8 * j + 4])),
                            silu_mul(__uint_as_float(gr[8 * j + 5]), __uint_as_float(ur[8 * j + 5])));
          p.w = pack_bf16x2(silu_mul(__uint_as_float(gr[8 * j + 6]), __uint_as_float(ur[8 * j + 6])),
                            silu_mul(__uint_as_float(gr[8 * j + 7]), __uint_as_float(ur[8 * j + 7])));
          const int ch = c / 8 + j;  // 16-byte chunk within the 128-byte row
          sts128(smem_u32(rowp) + ((ch ^ (lrow & 7)) << 4), p);
        }
      }
      fence_proxy_async_smem();
      dbar(1 + hf, 128);
      if (et == 0) {
        const int col = tn * DBN + hf * 64;
        if (col < a.N && tm * DBM < a.M) {
          tma_store_2d(&tmH, stage, col, tm * DBM);
          tma_store_commit();
        }
      }
    }
    if (et == 0) tma_store_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_pair<512>(tmem);
}

}  // namespace

bool dual_silu_ok(const DualArgs& a) {
  return (a.kg + DBK - 1) / DBK + (a.ku + DBK - 1) / DBK <= DMAXKB && a.N % 64 == 0;
}

int launch_dual_silu(const CUtensorMap& t, const CUtensorMap& g, const CUtensorMap& u, const CUtensorMap& h,
                     const DualArgs& a, cudaStream_t st) {
  if (!dual_silu_ok(a)) return (int)cudaErrorInvalidValue;
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(dual_silu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)D_SMEM);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  const int tiles_m = ((a.M + DBM - 1) / DBM + 1) / 2 * 2, tiles_n = (a.N + DBN - 1) / DBN;
  // output-tile slices per token tile: waves nearly full (one CTA per SM), ~2 tiles of fixed
  // cost per CTA (T tile load, pipeline fill)
  int slices = 1;
  long best = -1;
  for (int s = 1; s <= tiles_n; ++s) {
    const long waves = ((long)tiles_m * s + 147) / 148, per = (tiles_n + s - 1) / s;
    const long cost = waves * (per + 2);
    if (best < 0 || cost < best) best = cost, slices = s;
  }
  static const int env_slices = getenv("TNL_DUAL_SLICES") ? atoi(getenv("TNL_DUAL_SLICES")) : 0;  // A/B switch
  if (env_slices > 0) slices = env_slices < tiles_n ? env_slices : tiles_n;
  const int per = (tiles_n + slices - 1) / slices;
  slices = (tiles_n + per - 1) / per;
  // balanced: the flattened (token pair, output tile) work split evenly over 74 CTA pairs
  static const bool balance = !(getenv("TNL_DUAL_BALANCE") && atoi(getenv("TNL_DUAL_BALANCE")) == 0);  // A/B
  const int work = tiles_m / 2 * tiles_n;
  const int per_pair = (balance && env_slices <= 0 && work >= 74 * 8) ? (work + 73) / 74 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = per_pair ? dim3(2 * ((work + per_pair - 1) / per_pair), 1, 1) : dim3(tiles_m, slices, 1);
  cfg.blockDim = dim3(DUAL_THREADS, 1, 1);
  cfg.dynamicSmemBytes = D_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dual_silu_kernel, t, g, u, h, a, tiles_n, per, per_pair);
  count_launch();
  return (int)e;
}

}  // namespace tnl
