// tucker_chain.cu — the fused Tucker-2 chain for prefill: y = U0 . G . U1^T . x in ONE kernel.
//
// Reference: reconstruct for Tucker is G x_k U_k (tn_decompositions.py:351-355), so the layer
// applied to x is y[i] = sum_{r0} U0[i, r0] sum_{r1} G[r0, r1] sum_j U1[j, r1] x[j]
// (Tucker-2). The three contractions run back to back on chip per 128-token
// tile; the rank intermediates T1 (x U1) and T2 (T1 G^T) never leave the SM pair:
//
//   stage 1  T1 = X_tile . U1^T            K = cols, accumulated in TMEM (fp32)
//   stage 2  T2 = T1 . G^T                 T1 as a bf16 smem operand, K = R1, TMEM accumulator
//   stage 3  y_tile[:, n] = T2 . U0[n]^T   T2 as a bf16 smem operand, K = R0, 256-row tiles of U0
//
// Parallelism: a 2-CTA cluster per token tile (M = 8192 -> 128 CTAs). Stage 1 is split over the
// rank dimension (CTA r computes T1[:, r*R1/2 : (r+1)*R1/2] over the full K): each CTA converts its
// half to bf16 in the SW128 operand layout and ships it into the partner's operand buffer with one
// bulk async copy over distributed shared memory (cp.async.bulk shared::cluster, mbarrier
// complete_tx) — so both hold the full T1 with no fp32 partials and no HBM round trip. Stage 2 is
// computed by both CTAs (2 * 128 * R0 * R1 flops: negligible); stage 3 splits the output rows
// between them (interleaved 256-row tiles). HBM traffic = x + y (+ the L2-resident factors).
//
// Roles (192 threads): warp 0 TMA producer over one 4-slot ring (x/U1 tiles, then G chunks, then
// U0 chunks), warp 1 tcgen05.mma issuer, warps 2-5 epilogue (one token row per thread).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tnl {

namespace {

constexpr int BM = 128, BK = 64, BN3 = 256, STAGES = 4;
constexpr uint32_t SLOT = 32 * 1024;       // ring slot: x tile (16 KB) + U1 tile (<= 16 KB), or a G / U0 chunk
constexpr uint32_t OPCHUNK = BM * BK * 2;  // one 64-wide K chunk of a 128-row bf16 operand (16 KB)
constexpr uint32_t STG = BM * 64 * 2;      // output staging chunk (128 rows x 64 bf16)
constexpr size_t SMEM = 1024 + (size_t)STAGES * SLOT + 4 * OPCHUNK + 2 * STG + 256;

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Tucker2Args {
  int32_t M, rows, cols;
  int32_t r1p, r0p;  // padded ranks (multiples of 64, <= 256)
  int32_t split;     // 1: stage 1 split over the rank halves across the pair (r1p % 128 == 0)
};

__device__ __forceinline__ void bulk_s2cluster(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                               uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_cluster),
      "r"(src_cta), "r"(bytes), "r"(bar_cluster)
      : "memory");
}

__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// TMEM columns [c0, c0 + ncols) of this thread's row -> bf16 into the SW128 K-major operand buffer
__device__ __forceinline__ void tmem_to_operand(uint32_t taddr, int c0, int ncols, uint8_t* opbuf, int kbase, int lrow) {
  for (int c = 0; c < ncols; c += 32) {
    float v[32];
    tmem_ld16(taddr + c0 + c, v);
    tmem_ld16(taddr + c0 + c + 16, v + 16);
    const int k = kbase + c;
    uint8_t* rowp = opbuf + (k / 64) * OPCHUNK + (lrow >> 3) * 1024 + (lrow & 7) * 128;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 p;
      p.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
      p.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
      p.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
      p.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
      const int ch = ((k % 64) / 8) + j;
      sts128(smem_u32(rowp) + ((ch ^ (lrow & 7)) << 4), p);
    }
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    tucker2_chain_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmU1,
                         const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmU0,
                         const __grid_constant__ CUtensorMap tmY, const Tucker2Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* opbuf = ring + STAGES * SLOT;
  uint8_t* stg = opbuf + 4 * OPCHUNK;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 2 * STG);
  uint64_t* empty = full + STAGES;
  uint64_t* t1_done = empty + STAGES;  // MMA -> epilogue: stage-1 accumulator complete
  uint64_t* t1_ready = t1_done + 1;    // epilogue -> MMA: own T1 part written (4 warps)
  uint64_t* x_full = t1_ready + 1;     // partner's T1 half landed (tx bytes)
  uint64_t* t2_done = x_full + 1;
  uint64_t* t2_ready = t2_done + 1;    // 4 warps
  uint64_t* tfull = t2_ready + 1;      // [2]
  uint64_t* tempty = tfull + 2;        // [2], 4 warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const int tile = blockIdx.x >> 1;
  const int kb_total = (a.cols + BK - 1) / BK;
  const int n1 = a.split ? a.r1p / 2 : a.r1p;  // stage-1 width of this CTA
  const int k1_off = a.split ? (int)rank * n1 : 0;
  const int kc2 = a.r1p / 64, kc3 = a.r0p / 64;
  const int nt_total = (a.rows + BN3 - 1) / BN3;
  const int nt_mine = nt_total > (int)rank ? (nt_total - (int)rank + 1) / 2 : 0;  // tiles rank, rank+2, ...
  const uint32_t warp = warp_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmU1);
    tma_prefetch_desc(&tmG);
    tma_prefetch_desc(&tmU0);
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(t1_done, 1);
    mbar_init(t1_ready, 4);
    mbar_init(x_full, 1);
    mbar_init(t2_done, 1);
    mbar_init(t2_ready, 4);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
    if (a.split) mbar_arrive_expect_tx(x_full, (uint32_t)BM * n1 * 2);  // armed before the peer can send
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers exist before any bulk copy targets them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      auto slot = [&](uint32_t bytes) -> uint8_t* {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], bytes);
        return ring + s * SLOT;
      };
      // stage 1: x tile + this CTA's rows of U1^T
      pdl_wait();  // x is produced by the previous kernel
      for (int kb = 0; kb < kb_total; ++kb, ++it) {
        const int s = it % STAGES;
        uint8_t* sl = slot(OPCHUNK + (uint32_t)n1 * BK * 2);
        tma_load_2d(sl, &tmX, &full[s], kb * BK, tile * BM);
        tma_load_2d(sl + OPCHUNK, &tmU1, &full[s], kb * BK, k1_off);
      }
      // stage 2: G (r0p x r1p) in 64-wide K chunks
      for (int kc = 0; kc < kc2; ++kc, ++it) {
        const int s = it % STAGES;
        uint8_t* sl = slot((uint32_t)a.r0p * BK * 2);
        tma_load_2d(sl, &tmG, &full[s], kc * BK, 0);
      }
      // stage 3: 256-row tiles of U0 (this CTA's interleaved share), 64-wide K chunks
      for (int t = 0; t < nt_mine; ++t) {
        const int nt = (int)rank + 2 * t;
        for (int kc = 0; kc < kc3; ++kc, ++it) {
          const int s = it % STAGES;
          uint8_t* sl = slot(BN3 * BK * 2);
          tma_load_2d(sl, &tmU0, &full[s], kc * BK, nt * BN3);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      int it = 0;
      // stage 1
      {
        const uint32_t idesc = idesc_bf16_f32(BM, n1);
        for (int kb = 0; kb < kb_total; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(ring + s * SLOT));
          const uint64_t bd = smem_desc_sw128(smem_u32(ring + s * SLOT + OPCHUNK));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) mma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(t1_done);
      }
      // stage 2: T2 (TMEM columns [256, 256 + r0p)) = T1 . G^T
      mbar_wait(t1_ready, 0);
      if (a.split) mbar_wait_cluster(x_full, 0);
      tc_fence_after();
      {
        const uint32_t idesc = idesc_bf16_f32(BM, a.r0p);
        for (int kc = 0; kc < kc2; ++kc, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(opbuf + kc * OPCHUNK));
          const uint64_t bd = smem_desc_sw128(smem_u32(ring + s * SLOT));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_ss(tmem + 256, ad + 2 * k, bd + 2 * k, idesc, (kc > 0 || k > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(t2_done);
      }
      // stage 3: y tiles, accumulators alternating between TMEM [0, 256) and [256, 512)
      mbar_wait(t2_ready, 0);
      tc_fence_after();
      {
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN3);
        for (int t = 0; t < nt_mine; ++t) {
          const int acc = t & 1;
          if (t >= 2) mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + acc * BN3;
          for (int kc = 0; kc < kc3; ++kc, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            tc_fence_after();
            const uint64_t ad = smem_desc_sw128(smem_u32(opbuf + kc * OPCHUNK));
            const uint64_t bd = smem_desc_sw128(smem_u32(ring + s * SLOT));
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) mma_bf16_ss(d, ad + 2 * k, bd + 2 * k, idesc, (kc > 0 || k > 0) ? 1u : 0u);
            mma_commit(&empty[s]);
          }
          mma_commit(&tfull[acc]);
        }
      }
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3;
    const int lrow = q * 32 + lane_id();
    const int et = threadIdx.x - 64;
    const uint32_t lane_base = (q * 32) << 16;
    // T1: this CTA's part -> bf16 operand buffer; split: ship it into the partner's buffer too
    mbar_wait(t1_done, 0);
    tc_fence_after();
    tmem_to_operand(tmem + lane_base, 0, n1, opbuf, k1_off, lrow);
    fence_proxy_async_smem();
    tc_fence_before();
    named_bar(1, 128);
    if (a.split && et == 0) {
      const uint32_t off = (uint32_t)(k1_off / 64) * OPCHUNK, bytes = (uint32_t)(n1 / 64) * OPCHUNK;
      bulk_s2cluster(mapa_shared(opbuf, peer) + off, smem_u32(opbuf) + off, bytes, mapa_shared(x_full, peer));
      bulk_commit_wait_read();  // our buffer is rewritten with T2 later
    }
    __syncwarp();
    if (lane_id() == 0) mbar_arrive(t1_ready);
    // T2 -> bf16 operand buffer (stage 2 has finished reading T1)
    mbar_wait(t2_done, 0);
    tc_fence_after();
    if (a.split) {
      named_bar(1, 128);  // the bulk copy out of our buffer has finished reading it
    }
    tmem_to_operand(tmem + lane_base + 256, 0, a.r0p, opbuf, 0, lrow);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncwarp();
    if (lane_id() == 0) mbar_arrive(t2_ready);
    // stage 3 epilogue: TMEM -> bf16 -> SW128 staging -> TMA store (two staging buffers)
    pdl_wait();  // y may still be read by the previous kernel
    int chunk_ct = 0;
    for (int t = 0; t < nt_mine; ++t) {
      const int nt = (int)rank + 2 * t;
      const int acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * BN3 + lane_base;
      for (int c0 = 0; c0 < BN3; c0 += 64) {
        const int col = nt * BN3 + c0;
        if (col >= a.rows) {  // dead chunk of the ragged last tile: no TMEM read, no store
          if (c0 + 64 >= BN3) {
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&tempty[acc]);
          }
          continue;
        }
        uint8_t* stage = stg + (chunk_ct & 1) * STG;
        if (et == 0) tma_store_wait_read_le1();
        named_bar(1, 128);
        tmem_to_operand(d, c0, 64, stage, 0, lrow);
        if (c0 + 64 >= BN3) {
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&tempty[acc]);
        }
        fence_proxy_async_smem();
        named_bar(1, 128);
        if (et == 0) {
          tma_store_2d(&tmY, stage, col, tile * BM);
          tma_store_commit();
        }
        ++chunk_ct;
      }
    }
    if (et == 0) tma_store_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

// r1p in {64, 128, 256}: the stage-1 width of one CTA (r1p, or r1p / 2 when split over the pair)
// must fit the 16 KB U1 half of a ring slot and split into whole 64-wide operand chunks
bool tucker2_chain_ok(int r1p, int r0p) {
  return (r1p == 64 || r1p == 128 || r1p == 256) && r0p % 64 == 0 && r0p >= 64 && r0p <= 256;
}

int launch_tucker2_chain(const CUtensorMap& x, const CUtensorMap& u1, const CUtensorMap& g, const CUtensorMap& u0,
                         const CUtensorMap& y, int M, int rows, int cols, int r1p, int r0p, cudaStream_t st) {
  if (!tucker2_chain_ok(r1p, r0p) || M <= 0) return (int)cudaErrorInvalidValue;
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(tucker2_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  Tucker2Args a;
  a.M = M;
  a.rows = rows;
  a.cols = cols;
  a.r1p = r1p;
  a.r0p = r0p;
  a.split = r1p % 128 == 0 ? 1 : 0;
  const int tiles = (M + BM - 1) / BM;
  return (int)launch_pdl(tucker2_chain_kernel, dim3(2 * tiles), dim3(192), SMEM, st, x, u1, g, u0, y, a);
}

}  // namespace tnl
