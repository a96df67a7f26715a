// rmsnorm.cu — residual add + RMSNorm of the decoder stack driver (cfg4 plumbing, not the TN path).
//
//   x <- x + o (when o != NULL);   h <- x / sqrt(mean(x^2) + eps)      (bf16 storage, fp32 math)
//
// One pass over the residual stream instead of torch's add_ + rms_norm + copy_ (three passes and
// a temporary): at M = 8192, 5120 wide, that is 336 MB of traffic instead of ~590 MB.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace tnl {

namespace {

constexpr int RT = 256, RMAXV = 4;  // threads per row, 8-element vectors per thread (N <= 8192)

__global__ void __launch_bounds__(RT) add_rmsnorm_kernel(__nv_bfloat16* __restrict__ x, int64_t ldx,
                                                         const __nv_bfloat16* __restrict__ o, int64_t ldo,
                                                         __nv_bfloat16* __restrict__ h, int64_t ldh, int n,
                                                         float eps) {
  // PDL: wait for the producer of x / o, then let the consumer of h launch (it prefetches its
  // weights and waits for this grid before reading h)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t row = blockIdx.x;
  uint4* xr = reinterpret_cast<uint4*>(x + row * ldx);
  const uint4* orow = o ? reinterpret_cast<const uint4*>(o + row * ldo) : nullptr;
  uint4* hr = reinterpret_cast<uint4*>(h + row * ldh);
  const int nv = n / 8;
  float v[RMAXV][8];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < RMAXV; ++j) {
    const int c = threadIdx.x + j * RT;
    if (c >= nv) break;
    uint4 xv = xr[c];
    const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv);
    if (orow) {
      const uint4 ov = orow[c];
      const __nv_bfloat162* op = reinterpret_cast<const __nv_bfloat162*>(&ov);
      __nv_bfloat162 s[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 a = __bfloat1622float2(xp[e]), b = __bfloat1622float2(op[e]);
        s[e] = __floats2bfloat162_rn(a.x + b.x, a.y + b.y);
      }
      xv = *reinterpret_cast<uint4*>(s);
      xr[c] = xv;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 a = __bfloat1622float2(xp[e]);
      v[j][2 * e] = a.x;
      v[j][2 * e + 1] = a.y;
      ss = fmaf(a.x, a.x, fmaf(a.y, a.y, ss));
    }
  }
  __shared__ float red[RT / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < RT / 32; ++w) tot += red[w];
  const float inv = rsqrtf(tot / (float)n + eps);
#pragma unroll
  for (int j = 0; j < RMAXV; ++j) {
    const int c = threadIdx.x + j * RT;
    if (c >= nv) break;
    __nv_bfloat162 s[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = __floats2bfloat162_rn(v[j][2 * e] * inv, v[j][2 * e + 1] * inv);
    hr[c] = *reinterpret_cast<uint4*>(s);
  }
}

}  // namespace

int launch_add_rmsnorm(void* x, int64_t ldx, const void* o, int64_t ldo, void* h, int64_t ldh, int64_t m, int64_t n,
                       float eps, cudaStream_t st) {
  if (n % 8 || n > 8 * RT * RMAXV || ldx % 8 || (o && ldo % 8) || ldh % 8) return (int)cudaErrorInvalidValue;
  if (m == 0) return 0;
  return (int)launch_pdl(add_rmsnorm_kernel, dim3((unsigned)m), dim3(RT), 0, st, static_cast<__nv_bfloat16*>(x), ldx,
                         static_cast<const __nv_bfloat16*>(o), ldo, static_cast<__nv_bfloat16*>(h), ldh, (int)n, eps);
}

}  // namespace tnl
