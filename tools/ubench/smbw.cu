// Per-SM streaming bandwidth from HBM as a function of the number of active SMs: G CTAs (one
// per SM) each stream a private region with 1-D bulk TMA copies (32 KB chunks, 4-stage ring,
// mbarrier completion). Decides whether a decode design that streams all weights through a
// subset of the SMs (e.g. one 16-CTA cluster per token group) can keep HBM busy.
#include <cstdio>
#include "../../paper_2602_01613_b200/csrc/ptx.cuh"
using namespace tnl;
constexpr int CH = 32768, ST = 4;
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__global__ void __launch_bounds__(32, 1) k(const uint8_t* src, size_t per_cta, int chunks) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[ST];
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  for (int i = 0; i < chunks + ST; ++i) {
    if (i >= ST) mbar_wait(&bar[i % ST], ((i / ST) - 1) & 1);
    if (i < chunks) {
      mbar_arrive_expect_tx(&bar[i % ST], CH);
      bulk_g2s(sm + (i % ST) * CH, base + (size_t)i * CH, CH, &bar[i % ST]);
    }
  }
}
int main() {
  const size_t per_cta = 8u << 20;  // 8 MB per CTA (> L2 / 16 at G >= 16)
  uint8_t* buf;
  cudaMalloc(&buf, per_cta * 148);
  cudaMemset(buf, 1, per_cta * 148);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST);
  int gs[] = {1, 2, 4, 8, 16, 20, 32, 40, 64, 80, 120, 148};
  for (int G : gs) {
    const int chunks = per_cta / CH;
    for (int w = 0; w < 2; ++w) k<<<G, 32, CH * ST>>>(buf, per_cta, chunks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) k<<<G, 32, CH * ST>>>(buf, per_cta, chunks);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = 5.0 * G * per_cta / (ms * 1e6);
    printf("G=%3d  total %7.1f GB/s  per SM %6.1f GB/s\n", G, gbs, gbs / G);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
