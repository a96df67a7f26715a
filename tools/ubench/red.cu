// fp32 global reduction patterns of the decode epilogue: G CTAs each add a [KAP][64] fp32
// partial (KAP*256 B) into the same zero-at-rest accumulator.
#include <cstdio>
#include "../../paper_2602_01613_b200/csrc/ptx.cuh"
using namespace tnl;
// mode 0: thread = kappa row (lane quarter layout), 4 x red.v4 per 16 columns (current epilogue)
// mode 1: coalesced red.v4 (consecutive threads -> consecutive 16 B)
// mode 2: coalesced scalar red
// mode 3: plain coalesced st.global.v4 into a per-CTA slot (no atomics; reference for bandwidth)
template <int MODE, int KAP>
__global__ void __launch_bounds__(256) k(float* acc, float* slots, unsigned long long* cyc) {
  __syncthreads();
  long long t0 = clock64();
  const int t = threadIdx.x;
  if (MODE == 0) {
    // 256 threads: warp w (lane quarter w&3, half w>>2), kappa = blk*128 + (w&3)*32 + lane
    const int w = t >> 5, lane = t & 31;
    for (int blk = 0; blk < KAP / 128; ++blk) {
      const int kap = blk * 128 + (w & 3) * 32 + lane;
      for (int c = (w >> 2) * 32; c < (w >> 2) * 32 + 32; c += 16) {
        float* o = acc + kap * 64 + c;
#pragma unroll
        for (int e = 0; e < 16; e += 4) red_add_v4(o + e, 1.f, 1.f, 1.f, 1.f);
      }
    }
  } else if (MODE == 1) {
    for (int i = t; i < KAP * 16; i += 256) red_add_v4(acc + 4 * i, 1.f, 1.f, 1.f, 1.f);
  } else if (MODE == 2) {
    for (int i = t; i < KAP * 64; i += 256) atomicAdd(acc + i, 1.f);
  } else {
    float4* s = reinterpret_cast<float4*>(slots + (size_t)blockIdx.x * KAP * 64);
    for (int i = t; i < KAP * 16; i += 256) s[i] = make_float4(1.f, 1.f, 1.f, 1.f);
  }
  __threadfence();
  __syncthreads();
  long long t1 = clock64();
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE, int KAP>
void run(float* acc, float* slots, unsigned long long* d, int G) {
  for (int it = 0; it < 3; ++it) k<MODE, KAP><<<G, 256>>>(acc, slots, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it) k<MODE, KAP><<<G, 256>>>(acc, slots, d);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[160];
  cudaMemcpy(h, d, 8 * G, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < G; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("mode %d kappa %3d G %3d: %7.0f cyc max per CTA (%.2f us @1.9GHz), %.2f us per launch incl. launch\n", MODE, KAP, G,
         (double)mx, mx / 1900.0, ms * 1000 / 20);
}
int main() {
  float *acc, *slots;
  unsigned long long* d;
  cudaMalloc(&acc, 256 * 64 * 4);
  cudaMalloc(&slots, 160 * 256 * 64 * 4);
  cudaMalloc(&d, 8 * 160);
  for (int G : {40, 80}) {
    run<0, 256>(acc, slots, d, G);
    run<1, 256>(acc, slots, d, G);
    run<2, 256>(acc, slots, d, G);
    run<3, 256>(acc, slots, d, G);
    run<0, 64>(acc, slots, d, G);
    run<1, 64>(acc, slots, d, G);
  }
  return 0;
}
