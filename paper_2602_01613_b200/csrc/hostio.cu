// hostio.cu — stream-ordered copies executed by the SMs (tnl_copy_async).
//
// Decode steps move little data (M x 5120 bf16 = 640 KB at M = 64) but pay the copy engine's
// fixed cost twice per step, and a memcpy node in a CUDA graph cannot take part in programmatic
// dependent launch. Here the SMs move the bytes themselves: pinned host memory is mapped into the
// unified address space, so 16-byte loads (H2D) or stores (D2H) go straight over the bus with
// every thread of a full-GPU grid keeping one request in flight. The kernel is PDL-launched: it
// releases its successor at once (which prefetches its weights) and waits for its predecessor
// before touching the data.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace tnl {

namespace {

constexpr int CT = 256;

__global__ void __launch_bounds__(CT) copy16_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16,
                                                    uint8_t* __restrict__ dtail, const uint8_t* __restrict__ stail,
                                                    int tail) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t stride = (int64_t)gridDim.x * CT;
  int64_t i = (int64_t)blockIdx.x * CT + threadIdx.x;
  // up to four requests in flight per thread before the first store
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.global.cv.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) {
    uint4 v;
    asm volatile("ld.global.cv.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src + i));
    dst[i] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x < tail) dtail[threadIdx.x] = stail[threadIdx.x];
}

}  // namespace

int launch_copy16(void* dst, const void* src, size_t bytes, int sms, cudaStream_t st) {
  if (bytes == 0) return 0;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) return (int)cudaErrorInvalidValue;
  const int64_t n16 = (int64_t)(bytes / 16);
  const int tail = (int)(bytes % 16);
  int64_t grid = (n16 + CT - 1) / CT;
  if (grid > 2 * sms) grid = 2 * sms;
  if (grid < 1) grid = 1;
  return (int)launch_pdl(copy16_kernel, dim3((unsigned)grid), dim3(CT), 0, st, static_cast<uint4*>(dst),
                         static_cast<const uint4*>(src), n16, static_cast<uint8_t*>(dst) + n16 * 16,
                         static_cast<const uint8_t*>(src) + n16 * 16, tail);
}

}  // namespace tnl
