// Layout probe: tcgen05.mma kind::f16 with an F16 accumulator (idesc D format 0). One CTA:
// D (128 x 64) = A (128 x 64 bf16) . B (64 x 64 bf16)^T, then tcgen05.ld 32x32b of TMEM columns
// 0..63 for every lane -> raw 32-bit words. The host checks whether each 32-bit column holds one
// f16 value (upper half zero) or two packed f16 values (columns n, n+1), and times the TMEM read.
#include <cstdio>
#include <cstring>
#include <cmath>
#include <cuda_fp16.h>
#include "../../paper_2602_01613_b200/csrc/ptx.cuh"
using namespace tnl;

__device__ __forceinline__ uint32_t swz(int r, int c) { return (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4); }

template <bool F16>
__global__ void k(const __nv_bfloat16* A, const __nv_bfloat16* B, uint32_t* out, long long* cyc) {
  // (for F16, A and B hold f16 bit patterns)
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  // fill SW128 K-major images
  for (int i = t; i < 128 * 8; i += 128) {
    const int r = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sA + swz(r, c)) = *reinterpret_cast<const uint4*>(A + r * 64 + c * 8);
  }
  for (int i = t; i < 64 * 8; i += 128) {
    const int r = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sB + swz(r, c)) = *reinterpret_cast<const uint4*>(B + r * 64 + c * 8);
  }
  fence_proxy_async_smem();
  if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (t < 32) tmem_alloc<128>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (t == 0) {
    uint32_t idesc = idesc_bf16_f32(128, 64);
    if (F16) idesc &= ~((3u << 4) | (7u << 7) | (7u << 10));  // D F16, A/B F16 (kind::f16 needs f16 in)
    const uint64_t ad = smem_desc_sw128(smem_u32(sA)), bd = smem_desc_sw128(smem_u32(sB));
    for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tmem, ad + 2 * kk, bd + 2 * kk, idesc, kk > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = t / 32;
  long long c0 = clock64();
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((w * 32) << 16) + c, v);
    for (int e = 0; e < 16; ++e) out[(w * 32 + (t & 31)) * 64 + c + e] = __float_as_uint(v[e]);
  }
  long long c1 = clock64();
  if (t == 0) *cyc = c1 - c0;
  tc_fence_before();
  __syncthreads();
  if (t < 32) tmem_dealloc<128>(tmem);
}

int main() {
  __nv_bfloat16 hA[128 * 64], hB[64 * 64];
  float fA[128 * 64], fB[64 * 64];
  for (int i = 0; i < 128 * 64; ++i) { fA[i] = (float)((i * 37 % 17) - 8) / 8.f; hA[i] = __float2bfloat16(fA[i]); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < 64 * 64; ++i) { fB[i] = (float)((i * 53 % 13) - 6) / 8.f; hB[i] = __float2bfloat16(fB[i]); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB; uint32_t* dO; long long* dc;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dO, 128 * 64 * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  static uint32_t o[128 * 64];
  __half gA[128 * 64], gB[64 * 64];
  for (int i = 0; i < 128 * 64; ++i) gA[i] = __float2half(fA[i]);
  for (int i = 0; i < 64 * 64; ++i) gB[i] = __float2half(fB[i]);
  for (int f16 = 0; f16 < 2; ++f16) {
    cudaMemcpy(dA, f16 ? (void*)gA : (void*)hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, f16 ? (void*)gB : (void*)hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaMemset(dO, 0, 128 * 64 * 4);
    if (f16) k<true><<<1, 128>>>(dA, dB, dO, dc); else k<false><<<1, 128>>>(dA, dB, dO, dc);
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, dO, sizeof o, cudaMemcpyDeviceToHost);
    printf("F16=%d err=%s ld-cycles=%lld\n", f16, cudaGetErrorString(e), cyc);
    // reference for row 0..2, cols 0..7
    for (int r = 0; r < 3; ++r) {
      printf(" row %d ref:", r);
      for (int n = 0; n < 6; ++n) { double s = 0; for (int kk = 0; kk < 64; ++kk) s += fA[r * 64 + kk] * fB[n * 64 + kk]; printf(" %.3f", s); }
      printf("\n   raw:");
      for (int c = 0; c < (f16 ? 4 : 6); ++c) {
        uint32_t u = o[r * 64 + c];
        if (f16) { __half lo, hi; uint16_t l = u & 0xffff, h = u >> 16; memcpy(&lo, &l, 2); memcpy(&hi, &h, 2);
          printf(" [%08x %.3f|%.3f]", u, __half2float(lo), __half2float(hi)); }
        else { float f; memcpy(&f, &u, 4); printf(" %.3f", f); }
      }
      printf("\n");
    }
    if (f16) {  // where do columns 32..63 go?
      printf(" row 0 cols 30..35 raw:");
      for (int c = 30; c < 36; ++c) printf(" %08x", o[c]);
      printf("\n");
    }
  }
}
