// generic.cu — CUDA-core strided batched contraction (see generic.cuh).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "generic.cuh"

namespace tnl {

namespace {

constexpr int TI = 64, TJ = 64, TP = 16;

template <typename T>
__device__ __forceinline__ float ld_as_float(const T* p);
template <>
__device__ __forceinline__ float ld_as_float<float>(const float* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ float ld_as_float<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// grid.x = output tiles (x batch), grid.y = K-splits: split z reduces p in [z * pspan, (z+1) * pspan)
// and, when gridDim.y > 1, adds its partial with fp32 atomics into a pre-zeroed (or accumulating) C
template <typename TA, typename TB, typename TC>
__global__ void __launch_bounds__(256) generic_step_kernel(GStep s, int64_t tiles_i,
                                                           int64_t tiles_j, int64_t pspan) {
  __shared__ float sA[TP][TI + 4];
  __shared__ float sB[TP][TJ + 4];
  const int64_t tile = blockIdx.x;
  const int64_t tj = tile % tiles_j;
  const int64_t ti = (tile / tiles_j) % tiles_i;
  const int64_t bb = tile / (tiles_j * tiles_i);
  const int64_t b2 = bb % s.b2;
  const int64_t b1 = bb / s.b2;
  const TA* A = static_cast<const TA*>(s.A) + b1 * s.sa1 + b2 * s.sa2;
  const TB* B = static_cast<const TB*>(s.B) + b1 * s.sb1 + b2 * s.sb2;
  TC* C = static_cast<TC*>(s.C) + b1 * s.sc1 + b2 * s.sc2;

  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t i0 = ti * TI, j0 = tj * TJ;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;

  const int64_t pbeg = blockIdx.y * pspan, pend = min(s.P, pbeg + pspan);
  // A tile: TI x TP, B tile: TP x TJ (256 threads, 4 elements each). The next tile is loaded into
  // registers before the current one is consumed, so the global latency of iteration k+1 hides
  // behind the FMAs of iteration k (short chains: cfg1's steps have 2-4 iterations per CTA).
  constexpr int EA = TI * TP / 256, EB = TP * TJ / 256;
  int a_ii[EA], a_pp[EA], b_jj[EB], b_pp[EB];
#pragma unroll
  for (int u = 0; u < EA; ++u) {
    const int e = threadIdx.x + u * 256;
    a_pp[u] = s.sap == 1 ? e % TP : e / TI;  // contiguous along p: consecutive threads walk p
    a_ii[u] = s.sap == 1 ? e / TP : e % TI;
  }
#pragma unroll
  for (int u = 0; u < EB; ++u) {
    const int e = threadIdx.x + u * 256;
    b_jj[u] = s.sbj == 1 ? e % TJ : e / TP;
    b_pp[u] = s.sbj == 1 ? e / TJ : e % TP;
  }
  float ra[EA], rb[EB];
  auto fetch = [&](int64_t p0) {
#pragma unroll
    for (int u = 0; u < EA; ++u) {
      const int64_t gi = i0 + a_ii[u], gp = p0 + a_pp[u];
      ra[u] = (gi < s.I && gp < pend) ? ld_as_float(A + gi * s.sai + gp * s.sap) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < EB; ++u) {
      const int64_t gj = j0 + b_jj[u], gp = p0 + b_pp[u];
      rb[u] = (gj < s.J && gp < pend) ? ld_as_float(B + gp * s.sbp + gj * s.sbj) : 0.f;
    }
  };
  // PDL: the operands may be the previous step's output
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pbeg < pend) fetch(pbeg);
  for (int64_t p0 = pbeg; p0 < pend; p0 += TP) {
#pragma unroll
    for (int u = 0; u < EA; ++u) sA[a_pp[u]][a_ii[u]] = ra[u];
#pragma unroll
    for (int u = 0; u < EB; ++u) sB[b_pp[u]][b_jj[u]] = rb[u];
    __syncthreads();
    if (p0 + TP < pend) fetch(p0 + TP);
#pragma unroll
    for (int pp = 0; pp < TP; ++pp) {
      float a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = sA[pp][ty * 4 + q];
        b[q] = sB[pp][tx * 4 + q];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int64_t gi = i0 + ty * 4 + x;
    if (gi >= s.I) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int64_t gj = j0 + tx * 4 + y;
      if (gj >= s.J) continue;
      TC* dst = C + gi * s.sci + gj * s.scj;
      if constexpr (sizeof(TC) == 4) {
        if (gridDim.y > 1)
          atomicAdd(dst, acc[x][y]);
        else if (s.accumulate)
          *dst += acc[x][y];
        else
          *dst = acc[x][y];
      } else {
        *dst = __float2bfloat16_rn(acc[x][y]);
      }
    }
  }
}

__global__ void zero_strided_kernel(float* C, GStep s) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t n = s.b1 * s.b2 * s.I * s.J;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e % s.J, i = (e / s.J) % s.I, bb = e / (s.J * s.I);
    C[(bb / s.b2) * s.sc1 + (bb % s.b2) * s.sc2 + i * s.sci + j * s.scj] = 0.f;
  }
}

template <typename TA, typename TB>
int launch_c(const GStep& s, int64_t tiles_i, int64_t tiles_j, int64_t blocks, int64_t splits, cudaStream_t st) {
  const int64_t pspan = (s.P + splits - 1) / splits;
  const dim3 grid((unsigned)blocks, (unsigned)splits, 1);
  if (s.c_dt == DT_F32)
    return (int)launch_pdl(generic_step_kernel<TA, TB, float>, grid, dim3(256), 0, st, s, tiles_i, tiles_j, pspan);
  return (int)launch_pdl(generic_step_kernel<TA, TB, __nv_bfloat16>, grid, dim3(256), 0, st, s, tiles_i, tiles_j,
                         pspan);
}

template <typename TA>
int launch_b(const GStep& s, int64_t ti, int64_t tj, int64_t blocks, int64_t splits, cudaStream_t st) {
  if (s.b_dt == DT_F32) return launch_c<TA, float>(s, ti, tj, blocks, splits, st);
  return launch_c<TA, __nv_bfloat16>(s, ti, tj, blocks, splits, st);
}

}  // namespace

static thread_local bool t_deterministic = false;
void set_generic_deterministic(bool on) { t_deterministic = on; }

int launch_generic_step(const GStep& in, cudaStream_t stream) {
  GStep s = in;
  if (s.I <= 0 || s.J <= 0 || s.b1 <= 0 || s.b2 <= 0) return 0;
  // Fold b2 then b1 into I when the operand strides are compatible.
  auto fold = [&](int64_t& bcount, int64_t& sa, int64_t& sb, int64_t& sc) {
    if (bcount > 1 && sb == 0 && sa == s.sai * s.I && sc == s.sci * s.I) {
      s.I *= bcount;
      bcount = 1;
      sa = sb = sc = 0;
    }
  };
  fold(s.b2, s.sa2, s.sb2, s.sc2);
  if (s.b2 == 1) fold(s.b1, s.sa1, s.sb1, s.sc1);
  if (s.P <= 0) return 0;
  const int64_t tiles_i = (s.I + TI - 1) / TI, tiles_j = (s.J + TJ - 1) / TJ;
  const int64_t blocks = tiles_i * tiles_j * s.b1 * s.b2;
  if (blocks > 0x7fffffffLL) return (int)cudaErrorInvalidConfiguration;
  // few output tiles and a long contraction (e.g. cfg1's T = C . t1 step: one 64x64 tile, P = 2048):
  // split P over CTAs and reduce with fp32 atomics (fp32 C only; summation order changes, the
  // exactness contract is fp32 rounding, not bitwise)
  int64_t splits = 1;
  if (!t_deterministic && s.c_dt == DT_F32 && blocks < 148 && s.P >= 4 * TP * 2)
    splits = std::max<int64_t>(1, std::min<int64_t>((2 * 148 + blocks - 1) / blocks, s.P / (4 * TP)));
  if (splits > 1 && !s.accumulate) {
    const int64_t n = s.b1 * s.b2 * s.I * s.J;
    if (cudaError_t e = launch_pdl(zero_strided_kernel, dim3((unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8)),
                                   dim3(256), 0, stream, static_cast<float*>(s.C), s))
      return (int)e;
  }
  if (s.a_dt == DT_F32) return launch_b<float>(s, tiles_i, tiles_j, blocks, splits, stream);
  return launch_b<__nv_bfloat16>(s, tiles_i, tiles_j, blocks, splits, stream);
}

}  // namespace tnl
