// tcgen05.mma issue/throughput microbenchmark (sm_100a): one CTA per SM, one thread issues
// R back-to-back MMAs (M=128, N, K=16 bf16, A from TMEM or smem), measures issue time and
// completion time (commit -> mbarrier).
#include <cstdio>
#include "../../paper_2602_01613_b200/csrc/ptx.cuh"
using namespace tnl;
template <int N, bool TS, int R>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t ad = smem_desc_sw128(smem_u32(smem)), bd = smem_desc_sw128(smem_u32(smem + 16384));
    // warm
    for (int r = 0; r < 8; ++r) {
      if (TS) mma_bf16_ts(tmem, tmem + 256 + (r & 3) * 8, bd + 2 * (r & 3), idesc, r > 0);
      else mma_bf16_ss(tmem, ad + 2 * (r & 3), bd + 2 * (r & 3), idesc, r > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t0 = clock64();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (TS) mma_bf16_ts(tmem, tmem + 256 + (r & 3) * 8, bd + 2 * (r & 3), idesc, 1);
      else mma_bf16_ss(tmem, ad + 2 * (r & 3), bd + 2 * (r & 3), idesc, 1);
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
template <int N, bool TS, int R>
void run(unsigned long long* d) {
  cudaFuncSetAttribute(k<N, TS, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<N, TS, R><<<148, 128, 64 * 1024>>>(d);
  k<N, TS, R><<<148, 128, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%3d %s R=%3d: issue %6.1f cyc/mma, complete %6.1f cyc/mma (floor %d) %s\n", N, TS ? "TS" : "SS", R,
         (double)h[0] / R, (double)h[1] / R, 128 * N / 256, e == cudaSuccess ? "" : cudaGetErrorString(e));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  run<64, true, 16>(d);
  run<64, true, 64>(d);
  run<64, true, 256>(d);
  run<64, false, 64>(d);
  run<64, false, 256>(d);
  run<128, true, 64>(d);
  run<128, false, 64>(d);
  run<256, true, 64>(d);
  run<256, false, 64>(d);
  run<32, true, 64>(d);
  return 0;
}
