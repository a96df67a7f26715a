// tc_generic.cu — one step of the core-by-core TN chain on the tcgen05 tensor cores.
//
//   C[z][m][n] = sum_k A[z][m][k] * B[z][n][k]        (bf16 operands, fp32 accumulate in TMEM)
//
// The step is the same strided batched contraction the fp32 GENERIC plan runs on CUDA cores
// (generic.cuh: every np.tensordot of tn_decompositions.py:351-361 / tensor_core.py:109,130 once
// the plan has permuted the cores), after the host folded its batch dimensions into the M or N
// side (tnl_api.cu: tcg_from_gstep). The M and N sides are each up to three strided sub-dims, so
// operands are gathered by the threads into SW128 K-major shared-memory tiles (no TMA: the
// strides are arbitrary), one thread issues the MMAs of a 64-k chunk while the next chunk is
// gathered into the other stage, and the epilogue stores C through the same strided view.
// Intermediates of the bf16 chain are bf16 (the fp32 accumulator is rounded once per step).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"
#include "tc_generic.cuh"

namespace tnl {

namespace {

constexpr int GM = 128, GN = 64, GK = 64;
constexpr uint32_t GA_STAGE = GM * GK * 2, GB_STAGE = GN * GK * 2;

// element offset of index `idx` of a side (sub-dims outermost first); the host keeps every side
// below 2^31 elements, so the index arithmetic is 32-bit (int64 division is a long software sequence)
__device__ __forceinline__ int64_t side_offset(const TcgSide& s, int64_t idx64, bool c_view) {
  int64_t off = 0;
  uint32_t idx = (uint32_t)idx64;
#pragma unroll
  for (int d = 2; d >= 0; --d) {
    if (d >= s.nd) continue;
    const uint32_t sz = (uint32_t)s.size[d];
    const uint32_t i = idx % sz;
    idx /= sz;
    off += (int64_t)i * (c_view ? s.sc[d] : s.so[d]);
  }
  return off;
}

__device__ __forceinline__ uint32_t sw_chunk(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// one thread's row of a 64-k chunk, in registers between the gather and the swizzled store:
// 8 x 16 bytes when the row is K-contiguous and aligned, else 64 separate bf16 loads
template <bool VEC>
struct RowChunk;
template <>
struct RowChunk<true> {
  uint4 v[8];
  __device__ __forceinline__ void load(const __nv_bfloat16* base, int64_t, int64_t k0, int64_t K, bool valid) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int64_t k = k0 + c * 8;
      v[c] = (valid && k < K) ? __ldg(reinterpret_cast<const uint4*>(base + k)) : make_uint4(0u, 0u, 0u, 0u);
    }
  }
  __device__ __forceinline__ void store(uint32_t dst_block, int r) const {
#pragma unroll
    for (int c = 0; c < 8; ++c) sts128(dst_block + sw_chunk(r, c), v[c]);
  }
};
template <>
struct RowChunk<false> {
  uint16_t e[64];
  __device__ __forceinline__ void load(const __nv_bfloat16* base, int64_t ks, int64_t k0, int64_t K, bool valid) {
    const unsigned short* p = reinterpret_cast<const unsigned short*>(base) + k0 * ks;
    if (valid && k0 + 64 <= K) {  // full chunk: no per-element bound checks
#pragma unroll
      for (int j = 0; j < 64; ++j) e[j] = __ldg(p + j * ks);
      return;
    }
#pragma unroll
    for (int j = 0; j < 64; ++j) e[j] = (valid && k0 + j < K) ? __ldg(p + j * ks) : (unsigned short)0;
  }
  __device__ __forceinline__ void store(uint32_t dst_block, int r) const {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint4 v;
      v.x = (uint32_t)e[8 * c] | ((uint32_t)e[8 * c + 1] << 16);
      v.y = (uint32_t)e[8 * c + 2] | ((uint32_t)e[8 * c + 3] << 16);
      v.z = (uint32_t)e[8 * c + 4] | ((uint32_t)e[8 * c + 5] << 16);
      v.w = (uint32_t)e[8 * c + 6] | ((uint32_t)e[8 * c + 7] << 16);
      sts128(dst_block + sw_chunk(r, c), v);
    }
  }
};

__global__ void finalize_kernel(const TcgArgs a) {
  // split-K partials (dense fp32 [z][M][N], zero at rest) -> C through the strided view
  pdl_wait();
  const int64_t total = a.z1 * a.z2 * a.M * a.N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e % a.N, m = (e / a.N) % a.M, z = e / (a.N * a.M);
    const int64_t z1 = z / a.z2, z2 = z % a.z2;
    const float v = a.acc32[e];
    a.acc32[e] = 0.f;
    const int64_t off = z1 * a.zc1 + z2 * a.zc2 + side_offset(a.m, m, true) + side_offset(a.n, n, true);
    if (a.c_f32) {
      float* p = static_cast<float*>(a.C) + off;
      *p = a.accumulate ? *p + v : v;
    } else {
      static_cast<__nv_bfloat16*>(a.C)[off] = __float2bfloat16_rn(v);
    }
  }
}

// Persistent, warp-specialised: warps 0-5 gather operand rows (A: 128, B: 64) into a 2-stage
// ring with one chunk of register lookahead, thread 0 issues each chunk's MMAs into one of two TMEM
// accumulators; warps 6-9 run the epilogue of tile t while the loaders gather tile t+1. Steps of the
// chain are often a single 64-k chunk over thousands of tiles, so the per-tile setup (TMEM
// allocation, barrier initialisation, offset arithmetic) is paid once per CTA, not per tile.
constexpr int GT_LOAD = 192, GT_ALL = 320;

__global__ void __launch_bounds__(GT_ALL, 2) tc_generic_kernel(const TcgArgs a, int tiles_m, int tiles_n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;                                             // 2 stages
  uint8_t* sB = sA + 2 * GA_STAGE;                                // 2 stages
  int64_t* cN = reinterpret_cast<int64_t*>(sB + 2 * GB_STAGE);   // [2][GN] C offset of each tile column
  uint64_t* bars = reinterpret_cast<uint64_t*>(cN + 2 * GN);
  uint64_t* sdone = bars;       // [2] ring stage consumed by its MMAs
  uint64_t* tfull = bars + 2;   // [2] accumulator complete
  uint64_t* tempty = bars + 4;  // [2] accumulator read by the 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);

  const int tid = threadIdx.x;
  const uint32_t warp = warp_id();
  const int nk_all = (int)((a.K + GK - 1) / GK);
  const int64_t zz = a.z1 * a.z2;
  const int64_t num_tiles = (int64_t)tiles_m * tiles_n * zz * a.splits;
  auto decode = [&](int64_t t, int64_t& m0, int64_t& n0, int64_t& z, int& split) {
    const int64_t tm = t % tiles_m;  // token-side tiles fastest: consecutive CTAs share B rows in L2
    int64_t r = t / tiles_m;
    const int64_t tn = r % tiles_n;
    r /= tiles_n;
    split = (int)(r % a.splits);
    z = r / a.splits;
    m0 = tm * GM;
    n0 = tn * GN;
  };

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sdone[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<2 * GN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the previous step's output is this step's operand

  if (tid < GT_LOAD) {
    const bool is_a = tid < GM;
    const int r = is_a ? tid : tid - GM;
    const TcgSide& side = is_a ? a.m : a.n;
    const int64_t ks = is_a ? a.ka : a.kb;
    const bool vec = (is_a ? a.a_vec : a.b_vec) != 0;
    const uint32_t my0 = smem_u32(is_a ? sA : sB), my_bytes = is_a ? GA_STAGE : GB_STAGE;
    constexpr uint32_t idesc = idesc_bf16_f32(GM, GN);
    uint32_t g = 0;  // chunks issued by this CTA (ring position)
    int lt = 0;
    for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      int64_t m0, n0, z;
      int split;
      decode(t, m0, n0, z, split);
      const int64_t z1 = z / a.z2, z2 = z % a.z2;
      const int64_t grow = is_a ? m0 + r : n0 + r;
      const bool valid = is_a ? grow < a.M : grow < a.N;
      const __nv_bfloat16* base = is_a ? a.A + z1 * a.za1 + z2 * a.za2 : a.B + z1 * a.zb1 + z2 * a.zb2;
      const __nv_bfloat16* rbase = base + (valid ? side_offset(side, grow, false) : 0);
      const int c_beg = split * a.cps, c_end = min(nk_all, c_beg + a.cps);
      const int acc = lt & 1;
      auto run = [&](auto chunk) {
        chunk.load(rbase, ks, (int64_t)c_beg * GK, a.K, valid);
        for (int c = c_beg; c < c_end; ++c, ++g) {
          const int s = g & 1;
          if (g >= 2) mbar_wait(&sdone[s], ((g - 2) >> 1) & 1);
          chunk.store(my0 + s * my_bytes, r);
          if (c + 1 < c_end) chunk.load(rbase, ks, (int64_t)(c + 1) * GK, a.K, valid);
          fence_proxy_async_smem();
          asm volatile("bar.sync 1, 192;" ::: "memory");
          if (tid == 0) {
            if (c == c_beg && lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint64_t ad = smem_desc_sw128(smem_u32(sA) + s * GA_STAGE);
            const uint64_t bd = smem_desc_sw128(smem_u32(sB) + s * GB_STAGE);
#pragma unroll
            for (int k = 0; k < GK / 16; ++k)
              mma_bf16_ss(tmem + acc * GN, ad + 2 * k, bd + 2 * k, idesc, (c > c_beg || k > 0) ? 1u : 0u);
            mma_commit(&sdone[s]);
            if (c == c_end - 1) mma_commit(&tfull[acc]);
          }
        }
      };
      if (vec)
        run(RowChunk<true>());
      else
        run(RowChunk<false>());
    }
  } else {
    // epilogue: TMEM lane quarter q = warp % 4 -> tile rows q*32 .. q*32+31
    const int et = tid - GT_LOAD;
    const uint32_t q = warp & 3;
    const int lrow = q * 32 + lane_id();
    int lt = 0;
    for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      int64_t m0, n0, z;
      int split;
      decode(t, m0, n0, z, split);
      const int acc = lt & 1;
      const int64_t z1 = z / a.z2, z2 = z % a.z2;
      if (et < GN) {  // this tile's column offsets (the previous user of cN[acc] finished two tiles ago)
        const int64_t col = n0 + et;
        cN[acc * GN + et] = col < a.N ? side_offset(a.n, col, true) : -1;
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      const int64_t row = m0 + lrow;
      const bool rvalid = row < a.M;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * GN + ((q * 32) << 16);
      const int64_t* cn_t = cN + acc * GN;
      if (a.splits > 1) {  // fp32 partial of this K range -> dense scratch (finalize_kernel)
        float* accp = a.acc32 + (z * a.M + row) * a.N + n0;
#pragma unroll 1
        for (int c0 = 0; c0 < GN; c0 += 16) {
          float v[16];
          tmem_ld16(d + c0, v);
          if (!rvalid) continue;
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (n0 + c0 + e < a.N) atomicAdd(accp + c0 + e, v[e]);
        }
      } else {
        const int64_t coff = z1 * a.zc1 + z2 * a.zc2 + (rvalid ? side_offset(a.m, row, true) : 0);
        const bool full_n = n0 + GN <= a.N;
        __nv_bfloat16* c16 = static_cast<__nv_bfloat16*>(a.C) + coff;
#pragma unroll 1
        for (int c0 = 0; c0 < GN; c0 += 16) {
          float v[16];
          tmem_ld16(d + c0, v);
          if (!rvalid) continue;
          if (!a.c_f32 && full_n) {  // bf16 intermediate / output, no column tail
            const int64_t cb = cn_t[c0];
            if (cn_t[c0 + 15] - cb == 15 && ((coff + cb) & 7) == 0 &&
                !(reinterpret_cast<uintptr_t>(a.C) & 15)) {
              // 16 output-contiguous columns (the thread's row runs along y): two 16-byte stores
              uint4 p0, p1;
              p0.x = pack_bf16x2(v[0], v[1]);
              p0.y = pack_bf16x2(v[2], v[3]);
              p0.z = pack_bf16x2(v[4], v[5]);
              p0.w = pack_bf16x2(v[6], v[7]);
              p1.x = pack_bf16x2(v[8], v[9]);
              p1.y = pack_bf16x2(v[10], v[11]);
              p1.z = pack_bf16x2(v[12], v[13]);
              p1.w = pack_bf16x2(v[14], v[15]);
              uint4* dst = reinterpret_cast<uint4*>(c16 + cb);
              dst[0] = p0;
              dst[1] = p1;
              continue;
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) c16[cn_t[c0 + e]] = __float2bfloat16_rn(v[e]);
            continue;
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int64_t cn = cn_t[c0 + e];
            if (cn < 0) continue;
            if (a.c_f32) {
              float* p = static_cast<float*>(a.C) + coff + cn;
              *p = a.accumulate ? *p + v[e] : v[e];
            } else {
              c16[cn] = __float2bfloat16_rn(v[e]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&tempty[acc]);
    }
  }
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<2 * GN>(tmem);
}

}  // namespace

size_t tc_generic_smem() { return 1024 + 2 * (GA_STAGE + GB_STAGE) + 2 * GN * sizeof(int64_t) + 64; }

int launch_tc_generic(const TcgArgs& a, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return 0;
  const int64_t tm = (a.M + GM - 1) / GM, tn = (a.N + GN - 1) / GN, zz = a.z1 * a.z2;
  if (tm > 0x7fffffff || tn > 0x7fffffff || zz < 1 || a.M >= (1ll << 31) || a.N >= (1ll << 31))
    return (int)cudaErrorInvalidValue;
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(tc_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tc_generic_smem());
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  // few output tiles and a long K (decode-sized steps): split K across CTAs, fp32 partials into the
  // zero-at-rest scratch, then one pass through the strided output view
  TcgArgs b = a;
  const int nk = (int)((a.K + GK - 1) / GK);
  const int64_t tiles = tm * tn * zz;
  b.splits = 1;
  b.cps = nk;
  if (a.acc32 && tiles < 74 && nk >= 4) {
    const int want = (int)std::min<int64_t>(nk / 2, std::max<int64_t>(1, 148 / tiles));
    b.cps = (nk + want - 1) / want;
    b.splits = (nk + b.cps - 1) / b.cps;
  }
  const int64_t work = tiles * b.splits;
  const unsigned grid = (unsigned)std::min<int64_t>(work, 2 * 148);  // two persistent CTAs per SM
  cudaError_t e = launch_pdl(tc_generic_kernel, dim3(grid), dim3(GT_ALL), tc_generic_smem(), st, b, (int)tm, (int)tn);
  if (e != cudaSuccess || b.splits == 1) return (int)e;
  const int64_t total = zz * a.M * a.N;
  return (int)launch_pdl(finalize_kernel, dim3((unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8)), dim3(256),
                         0, st, b);
}

}  // namespace tnl
