// DSMEM store bandwidth: clusters of CS CTAs; every CTA writes BYTES of partials into its
// peers' shared memory (round-robin destinations, st.shared::cluster.v4), then cluster barrier.
#include <cstdio>
#include <cooperative_groups.h>
#include "../../paper_2602_01613_b200/csrc/ptx.cuh"
namespace cg = cooperative_groups;
using namespace tnl;
template <int CS, int BYTES>
__global__ void __launch_bounds__(256) k(unsigned long long* cyc) {
  extern __shared__ __align__(16) uint8_t smem[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  cl.sync();
  long long t0 = clock64();
  // destination d gets slice d of my partial: BYTES / CS bytes into its slot [rank]
  constexpr int SL = BYTES / CS;
  for (int d = 0; d < CS; ++d) {
    const uint32_t dst = (rank + d) % CS;
    float4* remote = reinterpret_cast<float4*>(cl.map_shared_rank(smem, dst)) + (rank * SL) / 16;
    for (int i = threadIdx.x; i < SL / 16; i += 256) remote[i] = make_float4(1.f, 2.f, 3.f, 4.f);
  }
  cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CS, int BYTES>
void run(unsigned long long* d, int G) {
  auto f = k<CS, BYTES>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (CS > 8) cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = BYTES + 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int i = 0; i < 3; ++i) cudaLaunchKernelEx(&cfg, f, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[160];
  cudaMemcpy(h, d, 8 * G, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < G; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("cluster %2d, %6d B per CTA, G %d: %6llu cyc (%.2f us @1.9GHz) %s\n", CS, BYTES, G, mx, mx / 1900.0,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 160);
  run<2, 65536>(d, 40);
  run<4, 65536>(d, 40);
  run<8, 65536>(d, 40);
  run<8, 16384>(d, 40);
  run<16, 65536>(d, 48);
  return 0;
}
