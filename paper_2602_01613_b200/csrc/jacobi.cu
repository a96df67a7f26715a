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

#include <algorithm>
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


// ---------------------------------------------------------------------------------------------
// Parallel-ordering sweeps for one LARGE problem (opt-in; the single
// unfoldings of a Qwen-shaped decomposition take hours in the reference's cyclic order).
//
// Brent-Luk round-robin ("circle") ordering: a sweep is n' - 1 steps (n' = n rounded up to even),
// each step rotates n'/2 DISJOINT pairs, so all pairs of a step run concurrently — one warp per
// pair, pairs spread over a persistent cooperative grid, one grid barrier per step. Every pair is
// visited once per sweep, with the reference's skip rules and rotation formulas (the (p, q) roles
// follow p < q, as in the cyclic order); the pair ORDER differs from the reference's cyclic
// order, so results agree up to rounding (spectrum parity <= 1e-10, singular vectors up to the
// sign convention applied afterwards) and the sweep count may differ. A sweep with no rotation
// ends the loop, as in the reference.
// ---------------------------------------------------------------------------------------------

namespace {

__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = *(volatile unsigned int*)gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*(volatile unsigned int*)gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// partner layout of the circle method: position 0 fixed, positions 1..n'-1 rotate by one per step
__device__ __forceinline__ int rr_member(int pos, int step, int np) {
  return pos == 0 ? 0 : 1 + ((pos - 1 + step) % (np - 1));
}

// one CTA (4 warps) per pair of a step: the three dot products and the rotation are spread over
// 128 threads (40 elements each at m = 5120) instead of one warp, so the per-pair latency chain is
// 4x shorter; CTAs loop over the step's pairs, one grid barrier per step.
constexpr int JP_THREADS = 128;

__global__ void __launch_bounds__(JP_THREADS) jacobi_parallel_kernel(double* __restrict__ W, double* __restrict__ R, int n,
                                                                     int m, int nv, double tol, int max_sweeps,
                                                                     int32_t* sweeps_out, unsigned int* sync) {
  __shared__ double red[3][JP_THREADS / 32];
  unsigned int* bar_count = sync;
  unsigned int* bar_gen = sync + 1;
  unsigned int* rot_sweep = sync + 2;  // 1 + index of the last sweep that rotated (monotonic)
  const int np = n + (n & 1);
  const int pairs = np / 2;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int sweeps = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int step = 0; step < np - 1; ++step) {
      for (int k = blockIdx.x; k < pairs; k += gridDim.x) {
        int p = rr_member(k, step, np), q = rr_member(np - 1 - k, step, np);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q >= n) continue;  // the dummy column of an odd n (uniform over the CTA)
        double* wp_row = W + (int64_t)p * m;
        double* wq_row = W + (int64_t)q * m;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int i = threadIdx.x; i < m; i += JP_THREADS) {
          const double wp = wp_row[i], wq = wq_row[i];
          app = __dadd_rn(app, __dmul_rn(wp, wp));
          aqq = __dadd_rn(aqq, __dmul_rn(wq, wq));
          apq = __dadd_rn(apq, __dmul_rn(wp, wq));
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        if (lane == 0) {
          red[0][wid] = app;
          red[1][wid] = aqq;
          red[2][wid] = apq;
        }
        __syncthreads();
        app = aqq = apq = 0.0;
#pragma unroll
        for (int w = 0; w < JP_THREADS / 32; ++w) {
          app = __dadd_rn(app, red[0][w]);
          aqq = __dadd_rn(aqq, red[1][w]);
          apq = __dadd_rn(apq, red[2][w]);
        }
        __syncthreads();  // red[] is rewritten by the next pair
        if (app == 0.0 || aqq == 0.0) continue;
        if (fabs(apq) <= __dmul_rn(tol, sqrt(__dmul_rn(app, aqq)))) continue;
        const double zeta = __ddiv_rn(__dsub_rn(aqq, app), __dmul_rn(2.0, apq));
        const double t = __ddiv_rn(copysign(1.0, zeta), __dadd_rn(fabs(zeta), sqrt(__dadd_rn(1.0, __dmul_rn(zeta, zeta)))));
        const double c = __ddiv_rn(1.0, sqrt(__dadd_rn(1.0, __dmul_rn(t, t))));
        const double s = __dmul_rn(c, t);
        for (int i = threadIdx.x; i < m; i += JP_THREADS) {
          const double wp = wp_row[i], wq = wq_row[i];
          wp_row[i] = __dsub_rn(__dmul_rn(c, wp), __dmul_rn(s, wq));
          wq_row[i] = __dadd_rn(__dmul_rn(s, wp), __dmul_rn(c, wq));
        }
        double* rp_row = R + (int64_t)p * nv;
        double* rq_row = R + (int64_t)q * nv;
        for (int i = threadIdx.x; i < nv; i += JP_THREADS) {
          const double vp = rp_row[i], vq = rq_row[i];
          rp_row[i] = __dsub_rn(__dmul_rn(c, vp), __dmul_rn(s, vq));
          rq_row[i] = __dadd_rn(__dmul_rn(s, vp), __dmul_rn(c, vq));
        }
        if (threadIdx.x == 0) atomicMax(rot_sweep, (unsigned int)sweep + 1u);
      }
      grid_barrier(bar_count, bar_gen, gridDim.x);
    }
    ++sweeps;
    if (*(volatile unsigned int*)rot_sweep < (unsigned int)sweep + 1u) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && sweeps_out) *sweeps_out = sweeps;
}

// ---------------------------------------------------------------------------------------------
// SVD post-processing of _jacobi_svd (tensor_core.py:214-235) on the device, one CTA per problem:
// column norms of the swept work rows, stable descending order, normalised left vectors,
// right = rot[order]^T, greedy canonical completion of the left basis for exactly-zero values
// (_complete_basis, tensor_core.py:185-200: residual I - B B^T, largest column norm, lowest index on
// ties, orthogonalise, normalise), and the sign convention (largest-|.| entry of each left vector
// positive, right flipped with it). Outputs per problem: left (m x n), values (n), right (n x n),
// row-major. Summation order inside the norms / dot products differs from numpy's.
// ---------------------------------------------------------------------------------------------

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = __dadd_rn(s, red[i]);
  return s;
}

// argmax of v over [0, n) (first index on ties); returns the index (all threads)
__device__ int block_argmax(double v, int idx, double* redv, int* redi) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    redv[w] = v;
    redi[w] = idx;
  }
  __syncthreads();
  double bv = redv[0];
  int bi = redi[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
    if (redv[i] > bv || (redv[i] == bv && redi[i] < bi)) {
      bv = redv[i];
      bi = redi[i];
    }
  return bi;
}

__global__ void __launch_bounds__(256) svd_finish_kernel(const double* __restrict__ work, const double* __restrict__ rot,
                                                         int n, int m, double* __restrict__ left, double* __restrict__ values,
                                                         double* __restrict__ right, double* __restrict__ scratch) {
  __shared__ double redv[8];
  __shared__ int redi[8];
  const int64_t b = blockIdx.x;
  const double* Wb = work + b * (int64_t)n * m;
  const double* Rb = rot + b * (int64_t)n * n;
  double* Lb = left + b * (int64_t)m * n;
  double* Vb = values + b * (int64_t)n;
  double* RTb = right + b * (int64_t)n * n;
  double* norms = scratch + b * (int64_t)(2 * n + 2 * m);  // [n] norms, [n] order (as double), [m] v, [m] c-norms^2
  double* orderd = norms + n;
  double* vbuf = orderd + n;
  // 1. row norms of work
  for (int j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) acc = __dadd_rn(acc, __dmul_rn(Wb[(int64_t)j * m + i], Wb[(int64_t)j * m + i]));
    acc = block_sum(acc, redv);
    if (threadIdx.x == 0) norms[j] = sqrt(acc);
  }
  __syncthreads();
  // 2. stable descending order: rank_j = #{i : norm_i > norm_j} + #{i < j : norm_i == norm_j}
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double nj = norms[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) rank += (norms[i] > nj) || (norms[i] == nj && i < j);
    orderd[rank] = (double)j;
  }
  __syncthreads();
  // 3. values, left = work[order] / values (positive values), right = rot[order]^T
  int positive = 0;
  for (int k = 0; k < n; ++k) positive += norms[(int)orderd[k]] > 0.0;
  for (int k = 0; k < n; ++k) {
    const int j = (int)orderd[k];
    const double v = norms[j];
    if (threadIdx.x == 0) Vb[k] = v;
    for (int i = threadIdx.x; i < m; i += blockDim.x)
      Lb[(int64_t)i * n + k] = k < positive ? __ddiv_rn(Wb[(int64_t)j * m + i], v) : 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) RTb[(int64_t)i * n + k] = Rb[(int64_t)j * n + i];
  }
  __syncthreads();
  // 4. _complete_basis for the exactly-zero tail
  for (int j = positive; j < n; ++j) {
    // column norms of resid = I - B B^T, B = left[:, :j]
    double best = -1.0;
    int besti = 0;
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      double s2 = 0.0;
      for (int r = 0; r < m; ++r) {
        double bb = 0.0;
        for (int k = 0; k < j; ++k) bb = __dadd_rn(bb, __dmul_rn(Lb[(int64_t)r * n + k], Lb[(int64_t)c * n + k]));
        const double e = __dsub_rn(r == c ? 1.0 : 0.0, bb);
        s2 = __dadd_rn(s2, __dmul_rn(e, e));
      }
      const double nc = sqrt(s2);
      if (nc > best) {
        best = nc;
        besti = c;
      }
    }
    const int pick = block_argmax(best, besti, redv, redi);
    // v = resid[:, pick]; v -= B (B^T v); u_j = v / |v|
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      double bb = 0.0;
      for (int k = 0; k < j; ++k) bb = __dadd_rn(bb, __dmul_rn(Lb[(int64_t)r * n + k], Lb[(int64_t)pick * n + k]));
      vbuf[r] = __dsub_rn(r == pick ? 1.0 : 0.0, bb);
    }
    __syncthreads();
    for (int k = 0; k < j; ++k) {  // coefficients B^T v, then v -= B coef
      double acc = 0.0;
      for (int r = threadIdx.x; r < m; r += blockDim.x) acc = __dadd_rn(acc, __dmul_rn(Lb[(int64_t)r * n + k], vbuf[r]));
      acc = block_sum(acc, redv);
      if (threadIdx.x == 0) orderd[k] = acc;  // order no longer needed: reuse as coefficient buffer
      __syncthreads();
    }
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      double acc = 0.0;
      for (int k = 0; k < j; ++k) acc = __dadd_rn(acc, __dmul_rn(Lb[(int64_t)r * n + k], orderd[k]));
      vbuf[r] = __dsub_rn(vbuf[r], acc);
    }
    __syncthreads();
    double nn = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) nn = __dadd_rn(nn, __dmul_rn(vbuf[r], vbuf[r]));
    nn = sqrt(block_sum(nn, redv));
    for (int r = threadIdx.x; r < m; r += blockDim.x) Lb[(int64_t)r * n + j] = __ddiv_rn(vbuf[r], nn);
    __syncthreads();
  }
  // 5. sign convention
  for (int j = 0; j < n; ++j) {
    double best = -1.0;
    int besti = 0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      const double a = fabs(Lb[(int64_t)r * n + j]);
      if (a > best) {
        best = a;
        besti = r;
      }
    }
    const int piv = block_argmax(best, besti, redv, redi);
    const bool flip = Lb[(int64_t)piv * n + j] < 0.0;
    __syncthreads();
    if (flip) {
      for (int r = threadIdx.x; r < m; r += blockDim.x) Lb[(int64_t)r * n + j] = -Lb[(int64_t)r * n + j];
      for (int r = threadIdx.x; r < n; r += blockDim.x) RTb[(int64_t)r * n + j] = -RTb[(int64_t)r * n + j];
    }
    __syncthreads();
  }
}

}  // namespace

int launch_jacobi_parallel(double* work, double* rot, int n, int m, int nv, double tol, int max_sweeps,
                           int32_t* sweeps, unsigned int* sync, int sms, cudaStream_t st) {
  // one CTA per pair of a step (up to all pairs at once), co-resident for the grid barrier
  const int pairs = (n + 1) / 2;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_parallel_kernel, JP_THREADS, 0);
  const int blocks = std::max(1, std::min(pairs, std::max(1, per_sm) * sms));
  if (cudaMemsetAsync(sync, 0, 4 * sizeof(unsigned int), st) != cudaSuccess) return (int)cudaGetLastError();
  void* args[] = {&work, &rot, &n, &m, &nv, &tol, &max_sweeps, &sweeps, &sync};
  cudaError_t e =
      cudaLaunchCooperativeKernel((const void*)jacobi_parallel_kernel, dim3(blocks), dim3(JP_THREADS), args, 0, st);
  count_launch();
  return (int)e;
}

int launch_svd_finish(const double* work, const double* rot, int64_t batch, int n, int m, double* left, double* values,
                      double* right, double* scratch, cudaStream_t st) {
  if (batch <= 0) return 0;
  svd_finish_kernel<<<(unsigned)batch, 256, 0, st>>>(work, rot, n, m, left, values, right, scratch);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace tnl
