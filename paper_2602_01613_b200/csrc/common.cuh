// common.cuh — shared host helpers for libtnl.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace tnl {

// One-time per-(kernel, device) setup such as cudaFuncSetAttribute: the attribute is per-device
// state, so a process that drives several GPUs must set it once on each of them.
struct AttrOnce {
  std::atomic<unsigned long long> mask{0};
  bool needed(int* dev) {
    if (cudaGetDevice(dev) != cudaSuccess) *dev = 0;
    return !((mask.load(std::memory_order_acquire) >> (*dev & 63)) & 1ull);
  }
  void done(int dev) { mask.fetch_or(1ull << (dev & 63), std::memory_order_release); }
};

// Per-thread count of libtnl kernel launches (tnl_launch_count).
void count_launch(int64_t n = 1);
int64_t launch_count(bool reset);

// Launch with programmatic dependent launch allowed (the kernel must griddepcontrol.wait before
// touching its predecessor's outputs): a plumbing kernel between two TN kernels then launches
// while its predecessor drains, and releases its own successor early.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  count_launch();
  return e;
}

// rmsnorm.cu: x += o (o may be NULL); h = x / rms(x)   (decoder-stack plumbing)
int launch_add_rmsnorm(void* x, int64_t ldx, const void* o, int64_t ldo, void* h, int64_t ldh, int64_t m, int64_t n,
                       float eps, cudaStream_t st);

// hostio.cu: SM-driven copy (either side may be mapped pinned host memory), 16-byte aligned
int launch_copy16(void* dst, const void* src, size_t bytes, int sms, cudaStream_t st);

// jacobi.cu: batched one-sided Jacobi sweeps (tnl_jacobi_sweeps)
int launch_jacobi_sweeps(double* work, double* rot, int64_t batch, int n, int m, int nv, double tol, int max_sweeps,
                         int32_t* sweeps, cudaStream_t st);
// tucker_chain.cu: fused Tucker-2 prefill chain y = U0 G U1^T x (maps: x box {64,128}; u1 box {64, r1p/2}
// when r1p % 128 == 0 else {64, r1p}; g box {64, r0p}; u0 box {64, 256}; y box {64, 128} SW128).
bool tucker2_chain_ok(int r1p, int r0p);
int launch_tucker2_chain(const CUtensorMap& x, const CUtensorMap& u1, const CUtensorMap& g, const CUtensorMap& u0,
                         const CUtensorMap& y, int M, int rows, int cols, int r1p, int r0p, cudaStream_t st);
int launch_jacobi_parallel(double* work, double* rot, int n, int m, int nv, double tol, int max_sweeps,
                           int32_t* sweeps, unsigned int* sync, int sms, cudaStream_t st);
int launch_svd_finish(const double* work, const double* rot, int64_t batch, int n, int m, double* left, double* values,
                      double* right, double* scratch, cudaStream_t st);

}  // namespace tnl
