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
constexpr int GT = 192;  // warps 0-3: A rows (+ epilogue), warps 4-5: B rows
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

// the K loop of one CTA: every thread gathers its row of each chunk (one chunk of lookahead: the
// loads of chunk c+1 are in flight while chunk c is stored, the CTA synchronises and thread 0
// issues the chunk's MMAs into the TMEM accumulator)
template <bool VEC>
__device__ __forceinline__ void k_loop(const __nv_bfloat16* rbase, int64_t ks, int64_t K, bool valid, int c_beg,
                                       int nk, uint32_t my_stage0, uint32_t my_stage_bytes, int r, uint32_t sa0,
                                       uint32_t sb0, uint32_t tmem, uint64_t* mdone) {
  constexpr uint32_t idesc = idesc_bf16_f32(128, 64);
  RowChunk<VEC> f;
  if (nk > 0) f.load(rbase, ks, (int64_t)c_beg * 64, K, valid);
  for (int c = 0; c < nk; ++c) {
    const int s = c & 1;
    if (c >= 2) mbar_wait(&mdone[s], ((c - 2) >> 1) & 1);
    f.store(my_stage0 + s * my_stage_bytes, r);
    if (c + 1 < nk) f.load(rbase, ks, (int64_t)(c_beg + c + 1) * 64, K, valid);
    fence_proxy_async_smem();
    asm volatile("bar.sync 1, 192;" ::: "memory");
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint64_t ad = smem_desc_sw128(sa0 + s * (128 * 64 * 2));
      const uint64_t bd = smem_desc_sw128(sb0 + s * (64 * 64 * 2));
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (c | k) != 0);
      mma_commit(&mdone[s]);
      if (c == nk - 1) mma_commit(&mdone[2]);
    }
  }
}

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

#ifndef TCG_MINB
#define TCG_MINB 3  // co-resident CTAs per SM (96 registers)
#endif
__global__ void __launch_bounds__(GT, TCG_MINB) tc_generic_kernel(const TcgArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;                       // 2 stages
  uint8_t* sB = sA + 2 * GA_STAGE;          // 2 stages
  int64_t* cN = reinterpret_cast<int64_t*>(sB + 2 * GB_STAGE);  // C offset of each tile column
  uint64_t* mdone = reinterpret_cast<uint64_t*>(cN + GN);        // [2] stage consumed, [2] all done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mdone + 4);

  const int tid = threadIdx.x;
  const uint32_t warp = warp_id();
  const int64_t m0 = (int64_t)blockIdx.x * GM, n0 = (int64_t)blockIdx.y * GN;
  const int split = (int)(blockIdx.z % a.splits);
  const int64_t z = blockIdx.z / a.splits, z1 = z / a.z2, z2 = z % a.z2;
  const __nv_bfloat16* A = a.A + z1 * a.za1 + z2 * a.za2;
  const __nv_bfloat16* B = a.B + z1 * a.zb1 + z2 * a.zb2;
  const int64_t cz = z1 * a.zc1 + z2 * a.zc2;

  if (tid == 0) {
    mbar_init(&mdone[0], 1);
    mbar_init(&mdone[1], 1);
    mbar_init(&mdone[2], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<GN>(tmem_slot);
  // this thread's operand row: A rows for warps 0-3, B rows (= tile columns) for warps 4-5
  const bool is_a = tid < GM;
  const int r = is_a ? tid : tid - GM;
  const int64_t grow = is_a ? m0 + r : n0 + r;
  const bool valid = is_a ? grow < a.M : grow < a.N;
  const TcgSide& side = is_a ? a.m : a.n;
  const int64_t roff = valid ? side_offset(side, grow, false) : 0;
  const __nv_bfloat16* rbase = (is_a ? A : B) + roff;
  const int64_t ks = is_a ? a.ka : a.kb;
  const bool vec = (is_a ? a.a_vec : a.b_vec) != 0;
  if (!is_a) cN[r] = valid ? side_offset(a.n, grow, true) : -1;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the previous step's output is this step's operand

  const int nk_all = (int)((a.K + GK - 1) / GK);
  const int c_beg = split * a.cps, c_end = min(nk_all, c_beg + a.cps), nk = c_end - c_beg;
  const uint32_t my0 = smem_u32(is_a ? sA : sB), my_bytes = is_a ? GA_STAGE : GB_STAGE;
  if (vec)
    k_loop<true>(rbase, ks, a.K, valid, c_beg, nk, my0, my_bytes, r, smem_u32(sA), smem_u32(sB), tmem, mdone);
  else
    k_loop<false>(rbase, ks, a.K, valid, c_beg, nk, my0, my_bytes, r, smem_u32(sA), smem_u32(sB), tmem, mdone);
  pdl_launch_dependents();
  if (warp < 4 && nk > 0 && a.splits > 1) {  // fp32 partial of this K range -> dense scratch
    mbar_wait(&mdone[2], 0);
    tc_fence_after();
    const bool rvalid = m0 + tid < a.M;
    float* acc = a.acc32 + (z * a.M + (m0 + tid)) * a.N + n0;
#pragma unroll 1
    for (int c0 = 0; c0 < GN; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((warp * 32) << 16) + c0, v);
      if (!rvalid) continue;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (n0 + c0 + e < a.N) atomicAdd(acc + c0 + e, v[e]);
    }
  } else if (warp < 4 && nk > 0) {
    mbar_wait(&mdone[2], 0);
    tc_fence_after();
    const bool rvalid = m0 + tid < a.M;
    const int64_t coff = cz + (rvalid ? side_offset(a.m, m0 + tid, true) : 0);
    const bool full_n = n0 + GN <= a.N;
    __nv_bfloat16* c16 = static_cast<__nv_bfloat16*>(a.C) + coff;
#pragma unroll 1
    for (int c0 = 0; c0 < GN; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((warp * 32) << 16) + c0, v);
      if (!rvalid) continue;
      if (!a.c_f32 && full_n) {  // bf16 intermediate / output, no column tail
#pragma unroll
        for (int e = 0; e < 16; ++e) c16[cN[c0 + e]] = __float2bfloat16_rn(v[e]);
        continue;
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int64_t cn = cN[c0 + e];
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
  __syncthreads();
  if (warp == 0) tmem_dealloc<GN>(tmem);
}

}  // namespace

size_t tc_generic_smem() { return 1024 + 2 * (GA_STAGE + GB_STAGE) + GN * sizeof(int64_t) + 64; }

int launch_tc_generic(const TcgArgs& a, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return 0;
  const int64_t tm = (a.M + GM - 1) / GM, tn = (a.N + GN - 1) / GN, zz = a.z1 * a.z2;
  if (tm > 0x7fffffff || tn > 65535 || zz > 65535 || zz < 1 || a.M >= (1ll << 31) || a.N >= (1ll << 31))
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
  if (zz * b.splits > 65535) {
    b.splits = 1;
    b.cps = nk;
  }
  cudaError_t e = launch_pdl(tc_generic_kernel, dim3((unsigned)tm, (unsigned)tn, (unsigned)(zz * b.splits)), dim3(GT),
                             tc_generic_smem(), st, b);
  if (e != cudaSuccess || b.splits == 1) return (int)e;
  const int64_t total = zz * a.M * a.N;
  return (int)launch_pdl(finalize_kernel, dim3((unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8)), dim3(256),
                         0, st, b);
}

}  // namespace tnl
