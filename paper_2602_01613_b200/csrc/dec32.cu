// dec32.cu — small-M fp32 forward of the merged-cut plan on CUDA cores (exact FFMA).
//
// The fp32 path is the reference-precision path (rel-err <= 1e-5 vs the float64 oracle), so it
// stays off the tensor cores. For decode-sized batches (cfg1: M = 16) the two-step generic chain
// (memset + split-K tile kernel + tile kernel) is launch-latency bound; these two kernels are the
// fp32 analogue of the bf16 decode phases:
//   phase A  T[kappa][m] += sum_{j in chunk} B_in[kappa][j] x[m][j]    grid (kappa tiles, K chunks),
//            fp32 reductions into the zero-at-rest accumulator at the workspace head
//   phase B  y[m][i] = sum_kappa A_out[i][kappa] T[kappa][m]           grid (row tiles); the A_out
//            tile is staged before the PDL wait, the last CTA re-zeroes T
#include <cuda_runtime.h>

#include "common.cuh"
#include "dec32.cuh"
#include "ptx.cuh"

namespace tnl {

namespace {

constexpr int A_KT = 32;    // kappa rows per phase-A CTA
constexpr int A_KC = 64;    // K chunk per phase-A CTA (64 CTAs at K = 4096)
constexpr int B_RT = 128;   // output rows per phase-B CTA (tile of the row loop)
constexpr int NT = 256;

__global__ void __launch_bounds__(NT) dec32_a_kernel(const float* __restrict__ bin, int64_t ldb, int r_cut, int K,
                                                     const float* __restrict__ x, int64_t ldx, int M, float* t) {
  __shared__ float sB[A_KT][A_KC + 1];
  __shared__ float sX[32][A_KC + 1];
  const int k0 = blockIdx.y * A_KC, kap0 = blockIdx.x * A_KT;
  const int kc = min(A_KC, K - k0);
  const bool v4 = kc == A_KC && ldb % 4 == 0 && ldx % 4 == 0 && !(reinterpret_cast<uintptr_t>(bin) & 15) &&
                  !(reinterpret_cast<uintptr_t>(x) & 15);
  if (v4) {  // 16-byte loads, all in flight before the first smem store
    constexpr int Q = A_KC / 4;
    float4 vb[A_KT * Q / NT], vx[32 * Q / NT];
#pragma unroll
    for (int u = 0; u < A_KT * Q / NT; ++u) {
      const int e = threadIdx.x + u * NT, r = e / Q, c = (e % Q) * 4;
      vb[u] = kap0 + r < r_cut ? __ldg(reinterpret_cast<const float4*>(bin + (int64_t)(kap0 + r) * ldb + k0 + c))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    pdl_wait();  // x may be the previous kernel's output (the weights above are not)
#pragma unroll
    for (int u = 0; u < 32 * Q / NT; ++u) {
      const int e = threadIdx.x + u * NT, r = e / Q, c = (e % Q) * 4;
      vx[u] = r < M ? *reinterpret_cast<const float4*>(x + (int64_t)r * ldx + k0 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < A_KT * Q / NT; ++u) {
      const int e = threadIdx.x + u * NT, r = e / Q, c = (e % Q) * 4;
      sB[r][c] = vb[u].x, sB[r][c + 1] = vb[u].y, sB[r][c + 2] = vb[u].z, sB[r][c + 3] = vb[u].w;
    }
#pragma unroll
    for (int u = 0; u < 32 * Q / NT; ++u) {
      const int e = threadIdx.x + u * NT, r = e / Q, c = (e % Q) * 4;
      sX[r][c] = vx[u].x, sX[r][c + 1] = vx[u].y, sX[r][c + 2] = vx[u].z, sX[r][c + 3] = vx[u].w;
    }
  } else {
    for (int e = threadIdx.x; e < A_KT * A_KC; e += NT) {
      const int r = e / A_KC, c = e % A_KC;
      sB[r][c] = (kap0 + r < r_cut && c < kc) ? bin[(int64_t)(kap0 + r) * ldb + k0 + c] : 0.f;
    }
    pdl_wait();
    for (int e = threadIdx.x; e < 32 * A_KC; e += NT) {
      const int r = e / A_KC, c = e % A_KC;
      sX[r][c] = (r < M && c < kc) ? x[(int64_t)r * ldx + k0 + c] : 0.f;
    }
  }
  __syncthreads();
  pdl_launch_dependents();
  // thread -> (kappa row, token pair): 8 threads share a kappa row (broadcast reads of sB)
  const int r = threadIdx.x / 8, mp = (threadIdx.x % 8) * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int c = 0; c < A_KC; ++c) {
    const float b = sB[r][c];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = fmaf(b, sX[mp + u][c], acc[u]);
  }
  if (kap0 + r < r_cut)
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (mp + u < M) atomicAdd(t + (int64_t)(kap0 + r) * 32 + mp + u, acc[u]);
}

__global__ void __launch_bounds__(NT) dec32_b_kernel(const float* __restrict__ aout, int64_t lda, int rows, int r_cut,
                                                     float* t, int M, float* y, int64_t ldy, unsigned int* counter) {
  extern __shared__ float smem[];
  const int ld = r_cut + 1;
  float* sA = smem;                    // [B_RT][r_cut + 1]
  float* sT = smem + B_RT * ld;        // [r_cut][32]
  const int i0 = blockIdx.x * B_RT;
  if (r_cut % 4 == 0 && lda % 4 == 0 && !(reinterpret_cast<uintptr_t>(aout) & 15)) {
    const int q = r_cut / 4;
    for (int e = threadIdx.x; e < B_RT * q; e += NT) {  // weights: independent of the previous kernel
      const int r = e / q, c = (e % q) * 4;
      const float4 v = i0 + r < rows ? __ldg(reinterpret_cast<const float4*>(aout + (int64_t)(i0 + r) * lda + c))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      sA[r * ld + c] = v.x, sA[r * ld + c + 1] = v.y, sA[r * ld + c + 2] = v.z, sA[r * ld + c + 3] = v.w;
    }
  } else {
    for (int e = threadIdx.x; e < B_RT * r_cut; e += NT) {
      const int r = e / r_cut, c = e % r_cut;
      sA[r * ld + c] = i0 + r < rows ? aout[(int64_t)(i0 + r) * lda + c] : 0.f;
    }
  }
  pdl_wait();
  for (int e = threadIdx.x; e < r_cut * 32; e += NT) sT[e] = __ldcg(t + e);
  __syncthreads();
  pdl_launch_dependents();
  // thread -> (row, 16-token half): lanes walk consecutive rows (coalesced y stores)
  const int r = threadIdx.x % B_RT, m0 = (threadIdx.x / B_RT) * 16;
  if (m0 < M) {
    float acc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] = 0.f;
    for (int c = 0; c < r_cut; ++c) {
      const float a = sA[r * ld + c];
#pragma unroll
      for (int u = 0; u < 16; ++u) acc[u] = fmaf(a, sT[c * 32 + m0 + u], acc[u]);
    }
    if (i0 + r < rows)
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (m0 + u < M) y[(int64_t)(m0 + u) * ldy + i0 + r] = acc[u];
  }
  // the last CTA to finish reading T re-zeroes it (zero at rest for the next call)
  __syncthreads();
  __shared__ unsigned int last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    for (int e = threadIdx.x; e < r_cut * 32; e += NT) t[e] = 0.f;
    if (threadIdx.x == 0) *counter = 0u;
  }
}

}  // namespace

size_t dec32_b_smem(int r_cut) { return sizeof(float) * ((size_t)B_RT * (r_cut + 1) + (size_t)r_cut * 32); }

int launch_dec32(const float* bin, int64_t ldb, const float* aout, int64_t lda, int rows, int r_cut, int K,
                 const float* x, int64_t ldx, int M, float* y, int64_t ldy, float* t, unsigned int* counter,
                 cudaStream_t st) {
  if (M < 1 || M > 32 || r_cut < 1 || r_cut > kDec32MaxCut) return (int)cudaErrorInvalidValue;
  const dim3 ga((r_cut + A_KT - 1) / A_KT, (K + A_KC - 1) / A_KC);
  cudaError_t e = launch_pdl(dec32_a_kernel, ga, dim3(NT), 0, st, bin, ldb, r_cut, K, x, ldx, M, t);
  if (e != cudaSuccess) return (int)e;
  const size_t smem = dec32_b_smem(r_cut);
  static AttrOnce attr;
  int attr_dev = 0;
  if (attr.needed(&attr_dev)) {
    e = cudaFuncSetAttribute(dec32_b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dec32_b_smem(kDec32MaxCut));
    if (e != cudaSuccess) return (int)e;
    attr.done(attr_dev);
  }
  return (int)launch_pdl(dec32_b_kernel, dim3((rows + B_RT - 1) / B_RT), dim3(NT), smem, st, aout, lda, rows, r_cut, t,
                         M, y, ldy, counter);
}

}  // namespace tnl
