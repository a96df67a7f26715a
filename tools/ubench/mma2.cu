// cta_group::2 tcgen05.mma issue/throughput (M=256 over a CTA pair, N, K=16 bf16).
#include <cstdio>
#include "../../paper_2602_01613_b200/csrc/ptx.cuh"
using namespace tnl;
template <int N, bool TS, int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x < 32) tmem_alloc_pair<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = idesc_bf16_f32(256, N);
    const uint64_t ad = smem_desc_sw128(smem_u32(smem)), bd = smem_desc_sw128(smem_u32(smem + 16384));
    for (int r = 0; r < 8; ++r) {
      if (TS) mma_bf16_ts_pair(tmem, tmem + 256 + (r & 3) * 8, bd + 2 * (r & 3), idesc, r > 0);
      else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad + 2 * (r & 3)), "l"(bd + 2 * (r & 3)), "r"(idesc), "r"((uint32_t)(r > 0)));
    }
    mma_commit_pair(&bar, 1);
    mbar_wait(&bar, 0);
    long long t0 = clock64();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (TS) mma_bf16_ts_pair(tmem, tmem + 256 + (r & 3) * 8, bd + 2 * (r & 3), idesc, 1);
      else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad + 2 * (r & 3)), "l"(bd + 2 * (r & 3)), "r"(idesc), "r"(1u));
    }
    long long t1 = clock64();
    mma_commit_pair(&bar, 1);
    mbar_wait(&bar, 1);
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) tmem_dealloc_pair<512>(tmem);
}
template <int N, bool TS, int R>
void run(unsigned long long* d) {
  cudaFuncSetAttribute(k<N, TS, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<N, TS, R><<<148, 128, 64 * 1024>>>(d);
  k<N, TS, R><<<148, 128, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("pair M=256 N=%3d %s R=%3d: issue %6.1f cyc/mma, complete %6.1f cyc/mma (per-SM floor %d) %s\n", N,
         TS ? "TS" : "SS", R, (double)h[0] / R, (double)h[1] / R, 128 * N / 256, e == cudaSuccess ? "" : cudaGetErrorString(e));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  run<64, true, 64>(d);
  run<64, false, 64>(d);
  run<128, true, 64>(d);
  run<256, true, 64>(d);
  run<32, true, 64>(d);
  return 0;
}
