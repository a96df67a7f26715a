// Throughput of the SFU (XU) candidates for the MLP epilogue's SiLU: cycles per warp-instruction
// per SM sub-partition, 16 warps per SM, independent chains.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#define N_IT 4096
template <int OP>
__global__ void k(float* out, unsigned long long* cyc) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  unsigned u0 = threadIdx.x, u1 = u0 + 1, u2 = u0 + 2, u3 = u0 + 3;
  __syncthreads();
  unsigned long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N_IT; ++i) {
    if (OP == 0) {
      asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a0)); asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a1));
      asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a2)); asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a3));
    } else if (OP == 1) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    } else if (OP == 2) {
      asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a3));
    } else if (OP == 3) {
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u0) : "f"(a0), "f"(__uint_as_float(u0)));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u1) : "f"(a1), "f"(__uint_as_float(u1)));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u2) : "f"(a2), "f"(__uint_as_float(u2)));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u3) : "f"(a3), "f"(__uint_as_float(u3)));
    } else if (OP == 4) {
      asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(u0)); asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(u1));
      asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(u2)); asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(u3));
    } else if (OP == 5) {
      asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a0)); asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a1));
      asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a2)); asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a3));
    } else if (OP == 6) {
      asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(u0)); asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(u1));
      asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(u2)); asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(u3));
    }
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + __uint_as_float(u0 ^ u1 ^ u2 ^ u3);
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int OP>
void run(const char* name, float* o, unsigned long long* c) {
  k<OP><<<148, 512>>>(o, c);
  k<OP><<<148, 512>>>(o, c);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  // 16 warps/SM = 4 per SMSP, 4 instr per iteration each
  printf("%-12s %.2f cycles per warp-instr per SMSP\n", name, (double)h / (N_IT * 4.0 * 4.0));
}
int main() {
  float* o;
  unsigned long long* c;
  cudaMalloc(&o, 148 * 512 * 4);
  cudaMalloc(&c, 8);
  run<0>("tanh.f32", o, c);
  run<1>("ex2.f32", o, c);
  run<2>("rcp.f32", o, c);
  run<3>("cvt.bf16x2", o, c);
  run<4>("tanh.f16x2", o, c);
  run<5>("ffma", o, c);
  run<6>("tanh.bf16x2", o, c);
  return 0;
}
