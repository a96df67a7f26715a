// SM-driven copy from pinned host memory: load flavours (.cv / .cg / .nc / plain) and request width.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(uint4* dst, const uint4* src, long n16) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
    uint4 v;
    if (MODE == 0) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
    if (MODE == 1) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
    if (MODE == 2) v = __ldg(src + i);
    if (MODE == 3) v = src[i];
    dst[i] = v;
  }
}
int main() {
  const size_t bytes = 655360;
  void* h; cudaHostAlloc(&h, bytes * 4, cudaHostAllocDefault);
  void* d; cudaMalloc(&d, bytes * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t sz : {bytes, bytes * 4}) {
    const long n16 = sz / 16;
    for (int mode = 0; mode < 5; ++mode) {
      for (int grid : {148, 296, 592}) {
        if (mode == 4 && grid != 148) continue;
        auto run = [&]() {
          if (mode == 0) k<0><<<grid, 256>>>((uint4*)d, (const uint4*)h, n16);
          if (mode == 1) k<1><<<grid, 256>>>((uint4*)d, (const uint4*)h, n16);
          if (mode == 2) k<2><<<grid, 256>>>((uint4*)d, (const uint4*)h, n16);
          if (mode == 3) k<3><<<grid, 256>>>((uint4*)d, (const uint4*)h, n16);
          if (mode == 4) cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice);
        };
        for (int w = 0; w < 5; ++w) run();
        cudaEventRecord(a);
        for (int it = 0; it < 50; ++it) run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const char* nm[] = {"ld.cv", "ld.cg", "ldg(nc)", "plain", "memcpy"};
        printf("%7zu B %-8s grid %3d: %6.2f us  %5.1f GB/s\n", sz, nm[mode], grid, ms / 50 * 1e3, sz / (ms / 50 * 1e-3) / 1e9);
      }
    }
  }
  // D2H stores
  for (int grid : {148, 296}) {
    const long n16 = bytes / 16;
    for (int w = 0; w < 5; ++w) k<3><<<grid, 256>>>((uint4*)h, (const uint4*)d, n16);
    cudaEventRecord(a);
    for (int it = 0; it < 50; ++it) k<3><<<grid, 256>>>((uint4*)h, (const uint4*)d, n16);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("D2H stores grid %d: %.2f us %.1f GB/s\n", grid, ms / 50 * 1e3, bytes / (ms / 50 * 1e-3) / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
