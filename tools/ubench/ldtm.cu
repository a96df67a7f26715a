// TMEM read throughput: 4 warps (128 lanes) repeatedly load 64 columns with tcgen05.ld
// 32x32b.x32 (fp32 cells) vs 32x32b.x16.pack::16b (two 16-bit cells per register).
#include <cstdio>
#include "../../paper_2602_01613_b200/csrc/ptx.cuh"
using namespace tnl;

template <bool PACK>
__global__ void k(float* out, long long* cyc) {
  __shared__ uint32_t slot;
  const int t = threadIdx.x, w = t / 32;
  if (t < 32) tmem_alloc<128>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((w * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < 256; ++it) {
    uint32_t r[32];
    if (PACK) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
            "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
            "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(base + (it & 1) * 64));  // 64 columns -> 32 registers
    } else {
      tmem_ld32_nowait(base + (it & 1) * 64, r);       // 32 columns -> 32 registers
    }
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += r[i];
  }
  long long c1 = clock64();
  __syncthreads();
  if (t == 0) *cyc = c1 - c0;
  out[t] = (float)acc;
  tc_fence_before();
  __syncthreads();
  if (t < 32) tmem_dealloc<128>(slot);
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  for (int p = 0; p < 2; ++p) {
    for (int rep = 0; rep < 2; ++rep) { if (p) k<true><<<1, 128>>>(o, c); else k<false><<<1, 128>>>(o, c); }
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    // bytes of TMEM cells touched per iteration: 128 lanes x (32 or 64) cells x 4 B
    const double cells = 128.0 * (p ? 64 : 32);
    printf("%s err=%s: %.1f cycles/iter, %.1f cells(4B)/cycle, %.1f reg-bytes/cycle\n", p ? "pack::16b x32 (64 cols)" : "32x32b.x32 (32 cols)",
           cudaGetErrorString(e), cyc / 256.0, cells / (cyc / 256.0), 128.0 * 32 * 4 / (cyc / 256.0));
  }
}
