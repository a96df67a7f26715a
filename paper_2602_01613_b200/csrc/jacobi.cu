// jacobi.cu — batched cyclic one-sided Jacobi sweeps, fp64.
//
// Same contract as the reference's only native component, `_jacobi_cy.jacobi_sweeps`
// (pkg/src/minima/_jacobi_cy.pyx:11-53, numpy twin _jacobi_py.py:16-49): the n rows of `work`
// (length m) are orthogonalised in place by plane rotations, visiting every pair (p, q), p < q,
// in lexicographic order each sweep and skipping pairs with app == 0 or aqq == 0 or
// |apq| <= tol * sqrt(app * aqq); `rot` (n x nv, identity on entry in _jacobi_svd) accumulates
// the rotations; a sweep with no rotation ends the loop; the sweep count is returned.
//
// B200 mapping: one warp per problem (a batch of independent matrices, e.g. every unfolding of
// a TT-SVD or the per-layer problems of a compression run), lane l owns elements i ≡ l (mod 32)
// of every row, so a rotation needs only the three dot products' butterfly reduction and no
// cross-lane data movement or barriers. Rows stay in global memory (L1/L2 resident for the
// sizes the decompositions produce). Products and sums are rounded separately (no FMA
// contraction), as the reference's scalar C; only the order of the dot-product summation
// differs (lane-strided partials + butterfly), which is exactly the latitude the reference
// grants its own numpy twin ("bit-for-bit up to summation order inside dot products").
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace tnl {

namespace {

constexpr int JW = 4;  // problems (warps) per CTA

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(32 * JW) jacobi_sweeps_kernel(double* __restrict__ work, double* __restrict__ rot,
                                                                int64_t batch, int n, int m, int nv, double tol,
                                                                int max_sweeps, int32_t* __restrict__ sweeps_out) {
  const int64_t b = (int64_t)blockIdx.x * JW + (threadIdx.x >> 5);
  if (b >= batch) return;
  const int lane = threadIdx.x & 31;
  double* W = work + b * (int64_t)n * m;
  double* R = rot + b * (int64_t)n * nv;
  int sweeps = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p) {
      double* wp_row = W + (int64_t)p * m;
      double* rp_row = R + (int64_t)p * nv;
      for (int q = p + 1; q < n; ++q) {
        double* wq_row = W + (int64_t)q * m;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double wp = wp_row[i], wq = wq_row[i];
          app = __dadd_rn(app, __dmul_rn(wp, wp));
          aqq = __dadd_rn(aqq, __dmul_rn(wq, wq));
          apq = __dadd_rn(apq, __dmul_rn(wp, wq));
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        if (app == 0.0 || aqq == 0.0) continue;
        if (fabs(apq) <= __dmul_rn(tol, sqrt(__dmul_rn(app, aqq)))) continue;
        const double zeta = __ddiv_rn(__dsub_rn(aqq, app), __dmul_rn(2.0, apq));
        const double t = __ddiv_rn(copysign(1.0, zeta), __dadd_rn(fabs(zeta), sqrt(__dadd_rn(1.0, __dmul_rn(zeta, zeta)))));
        const double c = __ddiv_rn(1.0, sqrt(__dadd_rn(1.0, __dmul_rn(t, t))));
        const double s = __dmul_rn(c, t);
        for (int i = lane; i < m; i += 32) {
          const double wp = wp_row[i], wq = wq_row[i];
          wp_row[i] = __dsub_rn(__dmul_rn(c, wp), __dmul_rn(s, wq));
          wq_row[i] = __dadd_rn(__dmul_rn(s, wp), __dmul_rn(c, wq));
        }
        double* rq_row = R + (int64_t)q * nv;
        for (int i = lane; i < nv; i += 32) {
          const double vp = rp_row[i], vq = rq_row[i];
          rp_row[i] = __dsub_rn(__dmul_rn(c, vp), __dmul_rn(s, vq));
          rq_row[i] = __dadd_rn(__dmul_rn(s, vp), __dmul_rn(c, vq));
        }
        rotated = true;
      }
    }
    ++sweeps;
    if (!rotated) break;
  }
  if (lane == 0 && sweeps_out) sweeps_out[b] = sweeps;
}

// Register-resident variant (m <= 32*EW, nv <= 32*ER): lane l keeps its elements of row p of
// work/rot in registers for the whole q loop (written back when p advances) and prefetches row
// q+1 while rotating against row q, so each pair visit costs one streamed row instead of two
// dependent L2 round trips. Same arithmetic, same order as jacobi_sweeps_kernel.
template <int EW, int ER>
__global__ void __launch_bounds__(32 * JW) jacobi_sweeps_reg_kernel(double* __restrict__ work, double* __restrict__ rot,
                                                                    int64_t batch, int n, int m, int nv, double tol,
                                                                    int max_sweeps, int32_t* __restrict__ sweeps_out) {
  const int64_t b = (int64_t)blockIdx.x * JW + (threadIdx.x >> 5);
  if (b >= batch) return;
  const int lane = threadIdx.x & 31;
  double* W = work + b * (int64_t)n * m;
  double* R = rot + b * (int64_t)n * nv;
  auto ldw = [&](int row, double* v) {
#pragma unroll
    for (int e = 0; e < EW; ++e) {
      const int i = lane + 32 * e;
      v[e] = i < m ? W[(int64_t)row * m + i] : 0.0;
    }
  };
  auto ldr = [&](int row, double* v) {
#pragma unroll
    for (int e = 0; e < ER; ++e) {
      const int i = lane + 32 * e;
      v[e] = i < nv ? R[(int64_t)row * nv + i] : 0.0;
    }
  };
  auto stw = [&](int row, const double* v) {
#pragma unroll
    for (int e = 0; e < EW; ++e) {
      const int i = lane + 32 * e;
      if (i < m) W[(int64_t)row * m + i] = v[e];
    }
  };
  auto str = [&](int row, const double* v) {
#pragma unroll
    for (int e = 0; e < ER; ++e) {
      const int i = lane + 32 * e;
      if (i < nv) R[(int64_t)row * nv + i] = v[e];
    }
  };
  int sweeps = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p) {
      double wp[EW], rp[ER], wq[EW], rq[ER], wn[EW], rn[ER];
      ldw(p, wp);
      ldr(p, rp);
      ldw(p + 1, wq);
      ldr(p + 1, rq);
      for (int q = p + 1; q < n; ++q) {
        if (q + 1 < n) {  // prefetch the next partner row
          ldw(q + 1, wn);
          ldr(q + 1, rn);
        }
        double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
        for (int e = 0; e < EW; ++e) {
          app = __dadd_rn(app, __dmul_rn(wp[e], wp[e]));
          aqq = __dadd_rn(aqq, __dmul_rn(wq[e], wq[e]));
          apq = __dadd_rn(apq, __dmul_rn(wp[e], wq[e]));
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        if (!(app == 0.0 || aqq == 0.0) && !(fabs(apq) <= __dmul_rn(tol, sqrt(__dmul_rn(app, aqq))))) {
          const double zeta = __ddiv_rn(__dsub_rn(aqq, app), __dmul_rn(2.0, apq));
          const double t =
              __ddiv_rn(copysign(1.0, zeta), __dadd_rn(fabs(zeta), sqrt(__dadd_rn(1.0, __dmul_rn(zeta, zeta)))));
          const double c = __ddiv_rn(1.0, sqrt(__dadd_rn(1.0, __dmul_rn(t, t))));
          const double s = __dmul_rn(c, t);
#pragma unroll
          for (int e = 0; e < EW; ++e) {
            const double a = wp[e], bq = wq[e];
            wp[e] = __dsub_rn(__dmul_rn(c, a), __dmul_rn(s, bq));
            wq[e] = __dadd_rn(__dmul_rn(s, a), __dmul_rn(c, bq));
          }
#pragma unroll
          for (int e = 0; e < ER; ++e) {
            const double a = rp[e], bq = rq[e];
            rp[e] = __dsub_rn(__dmul_rn(c, a), __dmul_rn(s, bq));
            rq[e] = __dadd_rn(__dmul_rn(s, a), __dmul_rn(c, bq));
          }
          stw(q, wq);
          str(q, rq);
          rotated = true;
        }
        if (q + 1 < n) {
#pragma unroll
          for (int e = 0; e < EW; ++e) wq[e] = wn[e];
#pragma unroll
          for (int e = 0; e < ER; ++e) rq[e] = rn[e];
        }
      }
      stw(p, wp);
      str(p, rp);
    }
    ++sweeps;
    if (!rotated) break;
  }
  if (lane == 0 && sweeps_out) sweeps_out[b] = sweeps;
}

}  // namespace

int launch_jacobi_sweeps(double* work, double* rot, int64_t batch, int n, int m, int nv, double tol, int max_sweeps,
                         int32_t* sweeps, cudaStream_t st) {
  if (batch <= 0) return 0;
  const int64_t grid = (batch + JW - 1) / JW;
  const int ew = (m + 31) / 32, er = (nv + 31) / 32;
  auto pick = [](int e) { return e <= 1 ? 1 : e <= 2 ? 2 : e <= 4 ? 4 : e <= 8 ? 8 : 0; };
  const int pw = pick(ew), pr = pick(er > 0 ? er : 1);
#define JAC_REG(EW_, ER_)                                                                                   \
  if (pw == EW_ && pr == ER_) {                                                                             \
    jacobi_sweeps_reg_kernel<EW_, ER_><<<(unsigned)grid, 32 * JW, 0, st>>>(work, rot, batch, n, m, nv, tol, \
                                                                          max_sweeps, sweeps);              \
    count_launch();                                                                                         \
    return (int)cudaGetLastError();                                                                         \
  }
  JAC_REG(1, 1) JAC_REG(2, 1) JAC_REG(2, 2) JAC_REG(4, 1) JAC_REG(4, 2) JAC_REG(4, 4) JAC_REG(8, 2) JAC_REG(8, 4)
  JAC_REG(8, 8)
#undef JAC_REG
  jacobi_sweeps_kernel<<<(unsigned)grid, 32 * JW, 0, st>>>(work, rot, batch, n, m, nv, tol, max_sweeps, sweeps);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace tnl
