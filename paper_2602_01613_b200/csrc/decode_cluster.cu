// decode_cluster.cu — cluster-resident decode of a chain of square merged-cut layers.
//
// The kernel-per-boundary decode (decode_fused.cu) pays, per layer, one grid completion and
// one L2 round trip for the split-K reduction of T (~1.5 us of a ~3.5 us layer). Here ONE
// thread-block cluster of 16 CTAs walks the whole chain for one token group (M <= 32) and the
// reduction never leaves the cluster:
//
//   CTA c owns rows [c R, c R + R) of every layer (R = D / 16), i.e. the K-slice of the next
//   layer's input side. Per layer l:
//     phase A   D_A (r x M) = B_in^l[:, slice_c] . x_c           tcgen05, x MN-major in smem
//     reduce    each D_A row goes to its owner CTA (r/16 rows per CTA) by st.async into the
//               owner's receive buffer (DSMEM, mbarrier complete_tx); the owner sums the 16
//               partials in a fixed order (deterministic) and broadcasts its bf16 T rows to all
//               16 CTAs' T operand (st.async again)
//     phase B   D_B (R x M) = A_out^l[slice_c, :] . T             tcgen05
//               -> bf16 -> x operand of layer l+1 (never leaves the SM) / y for the last layer
//
// Weights do not depend on activations: a producer warp streams every CTA's blocks of every
// layer, in consumption order, through a ring of 16 KB smem slots with 1-D bulk copies (no
// tensor maps — the arena is pre-swizzled into the SW128 smem image at tnl_chain_create), so
// the weight stream runs ahead of the dependency chain by the ring depth. 16 SMs stream a
// weight set at ~2.4 TB/s (measured, tools/ubench/smbw.cu); independent token groups run as
// independent clusters.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "decode_cluster.cuh"
#include "ptx.cuh"

namespace tnl {

namespace {

constexpr int CT = 320, CEPI = 256;
constexpr uint32_t SLOT = 16384;  // ring slot: one 128-row x 64-k bf16 SW128 block
constexpr uint32_t OPB = 8192;    // MN-major operand block: 64 k x 128 B

__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 16-byte store into (possibly) another CTA's shared memory; completion counted on that CTA's
// mbarrier (both addresses are shared::cluster addresses from mapa)
__device__ __forceinline__ void st_async16(uint32_t addr, uint4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(bar)
               : "memory");
}

template <int BN>
struct CSmem {
  static constexpr uint32_t RS = CHAIN_CS * 16 * BN * 4;  // receive buffer [src][<=16 rows][BN] fp32
  static size_t bytes(int nslot, int kbx) {
    return 1024 + (size_t)nslot * SLOT + 4 * OPB + (size_t)kbx * OPB + RS + 256 + 256;
  }
};

template <int BN>
__global__ void __launch_bounds__(CT, 1) chain_kernel(const CChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nslot = a.nslot;
  const int kbx = a.rpc / 64;
  uint8_t* ring = smem;
  uint8_t* sT = ring + nslot * SLOT;
  uint8_t* sX = sT + 4 * OPB;
  float* sRS = reinterpret_cast<float*>(sX + kbx * OPB);
  uint8_t* sRq = reinterpret_cast<uint8_t*>(sRS) + CSmem<BN>::RS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRq + 256);
  uint64_t* full = bars;        // [8]
  uint64_t* empty = bars + 8;   // [8]
  uint64_t* xready = bars + 16;  // x operand written (one arrive per epilogue warp)
  uint64_t* adone = bars + 17;   // phase-A MMAs complete
  uint64_t* bdone = bars + 18;   // phase-B MMAs complete
  uint64_t* tready = bars + 19;  // T operand received from all owners (tx bytes)
  uint64_t* rsfull = bars + 20;  // my rows' partials received from all CTAs (tx bytes)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);

  const uint32_t crank = cluster_ctarank();
  const uint32_t warp = warp_id();
  long long* tr = a.trace ? a.trace + (int64_t)crank * 256 * 16 : nullptr;
  const long long tbase = clock64();
#define CTRACE(l, ev) \
  if (tr) tr[(l) * 16 + (ev)] = clock64() - tbase;
  const int L = a.n;
  const int ntb = (a.rpc + 127) / 128;
  for (int i = threadIdx.x; i < L; i += CT) sRq[i] = a.rq[i];
  if (warp == 0 && elect_one()) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(xready, CEPI / 32);
    mbar_init(adone, 1);
    mbar_init(bdone, 1);
    mbar_init(tready, 1);
    mbar_init(rsfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every CTA's barriers are initialised before any remote st.async
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDB = tmem;        // ntb tiles x BN columns
  const uint32_t tDA = tmem + 128;  // <= 2 tiles x BN columns
  pdl_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {
      // weight stream, in exactly the MMA warp's consumption order: A(0) B(0) A(1) B(1) ...
      const uint8_t* src = a.arena + (int64_t)crank * a.per_cta_bytes;
      uint32_t blk = 0;
      const uint32_t ring_u32 = smem_u32(ring);
      auto push = [&](uint32_t bytes) {
        const uint32_t s = blk % nslot;
        if (blk >= (uint32_t)nslot) mbar_wait(&empty[s], ((blk / nslot) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(ring_u32 + s * SLOT, src, bytes, &full[s]);
        src += bytes;
        ++blk;
      };
      for (int l = 0; l < L; ++l) {
        const int rp = sRq[l] * 64;
        for (int u = 0; u < (rp + 127) / 128; ++u) {
          const uint32_t rows = min(128, rp - u * 128);
          for (int kb = 0; kb < kbx; ++kb) push(rows * 128);
        }
        for (int t = 0; t < ntb; ++t) {
          const uint32_t rows = min(128, a.rpc - t * 128);
          for (int kb = 0; kb < rp / 64; ++kb) {
            if (t == 0 && kb == 0) CTRACE(l, 13);  // producer reaches B(l)'s first block
            push(rows * 128);
            if (t == ntb - 1 && kb == rp / 64 - 1) CTRACE(l, 14);  // B(l)'s last block issued
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1 && a.debug == 1) {
    if (elect_one()) {  // stream-only: consume every ring slot as soon as it lands
      uint32_t blk = 0;
      for (int l = 0; l < L; ++l) {
        const int rp = sRq[l] * 64;
        const int nblk = (rp + 127) / 128 * kbx + ntb * (rp / 64);
        for (int i = 0; i < nblk; ++i, ++blk) {
          const uint32_t s = blk % nslot;
          mbar_wait(&full[s], (blk / nslot) & 1);
          mbar_arrive(&empty[s]);
        }
      }
    }
    __syncwarp();
  } else if (a.debug == 1) {
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32_bmn(128, BN);  // x and T operands are MN-major
      uint32_t blk = 0;
      for (int l = 0; l < L; ++l) {
        const int rp = sRq[l] * 64;
        // phase A(l): D_A[u] = B_in block rows . x
        mbar_wait(xready, l & 1);
        CTRACE(l, 0);
        tc_fence_after();
        for (int u = 0; u < (rp + 127) / 128; ++u)
          for (int kb = 0; kb < kbx; ++kb) {
            const uint32_t s = blk % nslot;
            mbar_wait(&full[s], (blk / nslot) & 1);
            tc_fence_after();
            const uint64_t ad = smem_desc_sw128(smem_u32(ring + s * SLOT));
            const uint64_t bd = smem_desc_sw128(smem_u32(sX + kb * OPB));
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_bf16_ss(tDA + u * BN, ad + 2 * k, bd + 128 * k, idesc, (kb | k) != 0);
            mma_commit(&empty[s]);
            ++blk;
          }
        mma_commit(adone);
        CTRACE(l, 1);
        // phase B(l): D_B[t] = A_out block rows . T   (T written by the owners' st.async)
        mbar_wait_cluster(tready, l & 1);
        CTRACE(l, 2);
        fence_proxy_async_smem();
        CTRACE(l, 8);
        tc_fence_after();
        for (int t = 0; t < ntb; ++t)
          for (int kb = 0; kb < rp / 64; ++kb) {
            const uint32_t s = blk % nslot;
            mbar_wait(&full[s], (blk / nslot) & 1);
            tc_fence_after();
            const uint64_t ad = smem_desc_sw128(smem_u32(ring + s * SLOT));
            if (t == 0 && kb == 0) CTRACE(l, 15);  // B(l)'s first block landed
            const uint64_t bd = smem_desc_sw128(smem_u32(sT + kb * OPB));
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_bf16_ss(tDB + t * BN, ad + 2 * k, bd + 128 * k, idesc, (kb | k) != 0);
            mma_commit(&empty[s]);
            ++blk;
          }
        mma_commit(bdone);
        CTRACE(l, 3);
      }
    }
    __syncwarp();
  } else {
    const int et = threadIdx.x - 64;
    const int lane = lane_id();
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const int c_begin = ((warp - 2) >> 2) * HALF;
    const bool has_cols = c_begin < BN;
    const uint32_t rs_local = smem_u32(sRS);
    const uint32_t t_local = smem_u32(sT);
    pdl_wait();
    // layer-0 input: x[token][crank R + k] -> MN-major operand [k][tokens]
    {
      constexpr int CH = BN / 8;  // 16-byte token chunks per k row
      const int items = a.rpc * CH;
      for (int e = et; e < items; e += CEPI) {
        const int k = e / CH, ch = e % CH;
        const int64_t col = (int64_t)crank * a.rpc + k;
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t0 = ch * 8 + 2 * j;
          const __nv_bfloat16 z = __float2bfloat16_rn(0.f);
          const __nv_bfloat16 lo = t0 < a.tokens ? a.x[(int64_t)t0 * a.ldx + col] : z;
          const __nv_bfloat16 hi = t0 + 1 < a.tokens ? a.x[(int64_t)(t0 + 1) * a.ldx + col] : z;
          w[j] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
        }
        sts128(smem_u32(sX) + (k / 64) * OPB + sw128(k % 64, ch), make_uint4(w[0], w[1], w[2], w[3]));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(xready);
    }
    for (int l = 0; l < L; ++l) {
      const int rp = sRq[l] * 64, rpo = rp / CHAIN_CS;
      if (et == 0) {  // this layer's receive phases (remote bytes may already be landing)
        mbar_arrive_expect_tx(rsfull, (uint32_t)(rp * BN * 4));
        mbar_arrive_expect_tx(tready, (uint32_t)(rp * BN * 2));
      }
      // reduce-scatter: every D_A row to its owner CTA
      mbar_wait(adone, l & 1);
      if (et == 0) CTRACE(l, 4);
      tc_fence_after();
      for (int u = 0; u < (rp + 127) / 128; ++u) {
        const int kap = u * 128 + q * 32 + lane;
        if (has_cols) {
#pragma unroll 1
          for (int c = c_begin; c < c_begin + HALF && c < BN; c += 16) {
            float v[16];
            tmem_ld16(tDA + u * BN + ((q * 32) << 16) + c, v);
            if (kap < rp) {
              const uint32_t o = kap / rpo, rho = kap % rpo;
              const uint32_t dst = mapa_shared(sRS, o) + ((crank * rpo + rho) * BN + c) * 4;
              const uint32_t bar = mapa_shared(rsfull, o);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                st_async16(dst + 16 * j,
                           make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                                      __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3])),
                           bar);
            }
          }
        }
      }
      if (et == 0) CTRACE(l, 11);
      tc_fence_before();
      // owner: sum the 16 partials of my rows (fixed order) and broadcast bf16 T rows
      {
        constexpr int CH = BN / 8;
        if (et < rpo * CH) {
          mbar_wait_cluster(rsfull, l & 1);
          if (et == 0) CTRACE(l, 5);
          const int rho = et / CH, ch = et % CH;
          float s[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) s[i] = 0.f;
#pragma unroll 4
          for (int src = 0; src < CHAIN_CS; ++src) {
            const uint32_t p = rs_local + ((src * rpo + rho) * BN + ch * 8) * 4;
            const float4 a0 = lds128f(p), a1 = lds128f(p + 16);
            s[0] += a0.x; s[1] += a0.y; s[2] += a0.z; s[3] += a0.w;
            s[4] += a1.x; s[5] += a1.y; s[6] += a1.z; s[7] += a1.w;
          }
          const uint4 pk = make_uint4(pack_bf16x2(s[0], s[1]), pack_bf16x2(s[2], s[3]), pack_bf16x2(s[4], s[5]),
                                      pack_bf16x2(s[6], s[7]));
          const int kap = crank * rpo + rho;
          const uint32_t off = (kap / 64) * OPB + sw128(kap % 64, ch);
#pragma unroll 4
          for (int d = 0; d < CHAIN_CS; ++d) st_async16(mapa_shared(sT, d) + off, pk, mapa_shared(tready, d));
          if (et == 0) CTRACE(l, 12);
        }
      }
      // phase B done: y_l -> x operand of layer l+1 (or the output)
      mbar_wait(bdone, l & 1);
      if (et == 0) CTRACE(l, 6);
      tc_fence_after();
      const bool last = l + 1 == L;
      for (int t = 0; t < ntb; ++t) {
        const int k = t * 128 + q * 32 + lane;
        if (has_cols) {
#pragma unroll 1
          for (int c = c_begin; c < c_begin + HALF && c < BN; c += 16) {
            float v[16];
            tmem_ld16(tDB + t * BN + ((q * 32) << 16) + c, v);
            if (k >= a.rpc) continue;
            if (!last) {
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const uint4 p = make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                                           pack_bf16x2(v[8 * j + 4], v[8 * j + 5]),
                                           pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
                sts128(smem_u32(sX) + (k / 64) * OPB + sw128(k % 64, c / 8 + j), p);
              }
            } else {
              __nv_bfloat16* yo = a.y + (int64_t)crank * a.rpc + k;
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (c + e < a.tokens) yo[(int64_t)(c + e) * a.ldy] = __float2bfloat16_rn(v[e]);
            }
          }
        }
      }
      if (et == 0) CTRACE(l, 9);
      if (!last) {
        fence_proxy_async_smem();
        if (et == 0) CTRACE(l, 10);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(xready);
      }
      if (et == 0) CTRACE(l, 7);
    }
    (void)t_local;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while a peer may still address its shared memory
  if (warp == 1) tmem_dealloc<256>(tmem);
}

template <int BN>
int launch_chain_bn(const CChainArgs& a0, cudaStream_t st) {
  CChainArgs a = a0;
  const int kbx = a.rpc / 64;
  size_t fixed = CSmem<BN>::bytes(0, kbx);
  int nslot = (int)((232448 - fixed) / SLOT);
  if (nslot > 8) nslot = 8;
  if (nslot < 2) return (int)cudaErrorInvalidValue;
  a.nslot = nslot;
  const size_t smem = CSmem<BN>::bytes(nslot, kbx);
  cudaError_t e = cudaFuncSetAttribute(chain_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(chain_kernel<BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return (int)e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CHAIN_CS, 1, 1);
  cfg.blockDim = dim3(CT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CHAIN_CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, chain_kernel<BN>, a);
  count_launch();
  return (int)e;
}

// arena repack: one CTA per block, 16-byte chunks placed at their SW128 smem-image position
__global__ void __launch_bounds__(128) repack_kernel(const CChainBlock* __restrict__ blocks, uint8_t* __restrict__ arena) {
  const CChainBlock b = blocks[blockIdx.x];
  for (int i = threadIdx.x; i < b.rows * 8; i += 128) {
    const int r = i >> 3, j = i & 7;
    const uint4 v = *reinterpret_cast<const uint4*>(b.src + (int64_t)(b.row0 + r) * b.ld + b.col0 + j * 8);
    *reinterpret_cast<uint4*>(arena + b.dst + r * 128 + ((j ^ (r & 7)) << 4)) = v;
  }
}

}  // namespace

int launch_chain(const CChainArgs& a, cudaStream_t st) {
  if (a.tokens < 1 || a.tokens > 32 || a.rpc % 64 || a.rpc > 384 || a.n < 1 || a.n > 256)
    return (int)cudaErrorInvalidValue;
  if (a.tokens <= 16) return launch_chain_bn<16>(a, st);
  return launch_chain_bn<32>(a, st);
}

int launch_chain_repack(const CChainBlock* blocks_dev, int64_t nblocks, uint8_t* arena, cudaStream_t st) {
  if (nblocks <= 0) return 0;
  repack_kernel<<<(unsigned)nblocks, 128, 0, st>>>(blocks_dev, arena);
  count_launch();
  return (int)cudaGetLastError();
}

int chain_max_active_clusters(int rpc, int tokens) {
  const int kbx = rpc / 64;
  const size_t fixed = tokens <= 16 ? CSmem<16>::bytes(0, kbx) : CSmem<32>::bytes(0, kbx);
  int nslot = (int)((232448 - fixed) / SLOT);
  if (nslot > 8) nslot = 8;
  const size_t smem = tokens <= 16 ? CSmem<16>::bytes(nslot, kbx) : CSmem<32>::bytes(nslot, kbx);
  auto kern = tokens <= 16 ? chain_kernel<16> : chain_kernel<32>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CHAIN_CS, 1, 1);
  cfg.blockDim = dim3(CT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CHAIN_CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace tnl
