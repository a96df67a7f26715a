// tnl_api.cu — C-ABI (include/tnl.h) + host planner for the TN-linear layer.
//
// Reference anchors (arxiv/paper_2602_01613, /root/reference/pkg/src/minima):
//   validate            tn_decompositions.py:97-126   -> validate_desc
//   matrix_shape/ranks  tn_decompositions.py:82-95    -> Plan::rows/cols, cut_rank
//   reconstruct         tn_decompositions.py:346-361  -> tnl_reconstruct (chain on identity)
//   layer_to_matrix @ x tn_decompositions.py:364 + sensitivity.py:156 -> tnl_forward
//   param_count         tn_decompositions.py:368-374  -> tnl_plan_query
//   errors              errors.py:8-21                -> tnl_status + tnl_last_error
//
// Plans. Every layer factorises through its cut bond (row modes first,
// tn_decompositions.py:59-63): y = A_out (B_in x). The planner keeps
//   * GENERIC: the core-by-core chain as CUDA-core strided steps (exact fp32);
//   * CUT    : B_in (r_cut x cols) and A_out (rows x r_cut) pre-contracted once
//              at plan time, forward = two tcgen05 GEMM steps;
//   * CHAIN  : Tucker-2 as three tcgen05 GEMM steps (U_in, G, U_out);
//   * DENSE  : one tcgen05 GEMM step.
// bf16 plans use the tensor-core steps; fp32 plans use GENERIC.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tnl.h"
#include "../../include/tnl_stack.h"
#include "chain.cuh"
#include "common.cuh"
#include "decode.cuh"
#include "generic.cuh"
#include "tc_generic.cuh"
#include "dec32.cuh"
#include "mlp.cuh"
#include "tc_gemm.cuh"

namespace tnl {

static thread_local int64_t g_launches = 0;
void count_launch(int64_t n) { g_launches += n; }
int64_t launch_count(bool reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

static thread_local std::string g_err;

static tnl_status fail(tnl_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (cudaError_t)(expr);                                               \
    if (_e != cudaSuccess)                                                              \
      return fail(TNL_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

// Plan-build stage timer (TNL_BUILD_PROFILE=1: one line per plan on stderr; measurement aid).
struct BuildTimer {
  bool on = getenv("TNL_BUILD_PROFILE") && atoi(getenv("TNL_BUILD_PROFILE")) != 0;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  char buf[512];
  int len = 0;
  void mark(const char* what) {
    if (!on) return;
    cudaDeviceSynchronize();
    auto n = std::chrono::steady_clock::now();
    len += snprintf(buf + len, sizeof buf - len, " %s=%.2fms", what,
                    std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// Device allocations of plans, MLP blocks and their build temporaries come from the device's
// stream-ordered memory pool with an unlimited release threshold: building the 448 projections of
// the cfg4 stack allocates and frees ~900 panel temporaries, which cudaMalloc / cudaFree turned into
// driver calls with implicit device synchronisation (seconds in total); from the pool they are
// sub-allocations of memory the process already holds.
static cudaError_t dev_alloc(void** p, size_t bytes) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    configured = dev;
  }
  cudaError_t e = cudaMallocAsync(p, bytes, 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  return e;
}
static void dev_free(void* p) {
  if (p) cudaFreeAsync(p, 0);
}
template <typename T>
static cudaError_t dev_alloc(T** p, size_t bytes) {
  return dev_alloc(reinterpret_cast<void**>(p), bytes);
}

static inline int64_t prod(const int64_t* a, int lo, int hi) {
  int64_t p = 1;
  for (int i = lo; i < hi; ++i) p *= a[i];
  return p;
}
static inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// small device kernels
// ---------------------------------------------------------------------------
__global__ void f32_to_bf16_2d(const float* __restrict__ src, int64_t lds, __nv_bfloat16* dst,
                               int64_t ldd, int64_t rows, int64_t cols) {
  int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    dst[r * ldd + c] = __float2bfloat16_rn(src[r * lds + c]);
  }
}
// contiguous fp32 -> bf16, 8 elements per thread (n % 8 == 0, 16-byte aligned buffers)
__global__ void f32_to_bf16_v8(const float4* __restrict__ src, uint4* __restrict__ dst, int64_t n8) {
  // PDL: wait for the producer of src (split-K reductions), release the consumer of dst early
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n8; e += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = src[2 * e], b = src[2 * e + 1];
    __nv_bfloat162 o[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                           __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
    dst[e] = *reinterpret_cast<uint4*>(o);
  }
}
__global__ void identity_f32(float* dst, int64_t rows, int64_t cols, int64_t offset) {
  // dst[r][c] = (c == r + offset)
  int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    dst[e] = (c == r + offset) ? 1.f : 0.f;
  }
}
// out[a][b][c][d] (contiguous) = X[a*sxa + c*sxc] * Y[b*syb + d*syd] — the Kronecker-structured
// panel of a two-mode Tucker side with no core in between (plan-time panel builder)
__global__ void kron2_f32(float* out, const float* X, int64_t sxa, int64_t sxc, const float* Y, int64_t syb,
                          int64_t syd, int64_t Da, int64_t Db, int64_t Dc, int64_t Dd) {
  const int64_t n = Da * Db * Dc * Dd;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t dd = e % Dd, cc = (e / Dd) % Dc, bb = (e / (Dd * Dc)) % Db, aa = e / (Dd * Dc * Db);
    out[e] = X[aa * sxa + cc * sxc] * Y[bb * syb + dd * syd];
  }
}
__global__ void copy_2d_any(const void* src, int s_dt, int64_t s_r, int64_t s_c, void* dst, int d_dt,
                            int64_t d_r, int64_t d_c, int64_t rows, int64_t cols) {
  int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    float v = s_dt == DT_F32 ? static_cast<const float*>(src)[r * s_r + c * s_c]
                             : __bfloat162float(static_cast<const __nv_bfloat16*>(src)[r * s_r + c * s_c]);
    if (d_dt == DT_F32)
      static_cast<float*>(dst)[r * d_r + c * d_c] = v;
    else
      static_cast<__nv_bfloat16*>(dst)[r * d_r + c * d_c] = __float2bfloat16_rn(v);
  }
}
static int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 16); }
// dense [rows][cols] fp32 -> bf16 (both contiguous)
// [rows][cols] fp32 -> bf16 with row r scaled by rsqrt(ss[r] / n + eps) (folded RMSNorm of the
// layer input: the cut activations are linear in x, so normalising them == normalising x)
__global__ void f32_to_bf16_rowscale(const float4* __restrict__ src, uint4* __restrict__ dst, int64_t n8, int64_t cols8,
                                     const float* __restrict__ ss, float inv_n, float eps) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n8; e += (int64_t)gridDim.x * blockDim.x) {
    const float sc = rsqrtf(ss[e / cols8] * inv_n + eps);
    const float4 a = src[2 * e], b = src[2 * e + 1];
    __nv_bfloat162 o[4] = {__floats2bfloat162_rn(a.x * sc, a.y * sc), __floats2bfloat162_rn(a.z * sc, a.w * sc),
                           __floats2bfloat162_rn(b.x * sc, b.y * sc), __floats2bfloat162_rn(b.z * sc, b.w * sc)};
    dst[e] = *reinterpret_cast<uint4*>(o);
  }
}
static void to_bf16_scaled(const float* src, __nv_bfloat16* dst, int64_t rows, int64_t cols, const tnl_fwd_opts* o,
                           cudaStream_t st) {
  const int64_t n8 = rows * cols / 8;
  launch_pdl(f32_to_bf16_rowscale, dim3(grid_for(n8)), dim3(256), 0, st, reinterpret_cast<const float4*>(src),
             reinterpret_cast<uint4*>(dst), n8, cols / 8, o->ss_in, 1.f / (float)o->rms_n, o->rms_eps);
}
static void to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, cudaStream_t st) {
  if (n % 8 == 0 && !(reinterpret_cast<uintptr_t>(src) & 15) && !(reinterpret_cast<uintptr_t>(dst) & 15))
    launch_pdl(f32_to_bf16_v8, dim3(grid_for(n / 8)), dim3(256), 0, st, reinterpret_cast<const float4*>(src),
               reinterpret_cast<uint4*>(dst), n / 8);
  else {
    f32_to_bf16_2d<<<grid_for(n), 256, 0, st>>>(src, n, dst, n, 1, n);
    count_launch();
  }
}
// ss[row] = sum_j x[row][j]^2 (one CTA per row; the folded RMSNorm's statistics)
// one warp per row, 8 rows per CTA: every lane keeps its row's 16-byte loads in flight at once
// (a CTA per row left ~2 loads per thread and the SMs mostly waiting on block launches)
__global__ void __launch_bounds__(256) row_sumsq_bf16(const __nv_bfloat16* __restrict__ x, int64_t ldx, int64_t n,
                                                      int64_t m, float* __restrict__ ss) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= m) return;
  const int lane = threadIdx.x & 31;
  const uint4* r = reinterpret_cast<const uint4*>(x + row * ldx);
  const int64_t nv = n / 8;
  float s = 0.f;
  constexpr int U = 8;
  for (int64_t c0 = 0; c0 < nv; c0 += 32 * U) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + u * 32 + lane;
      w[u] = c < nv ? r[c] : make_uint4(0u, 0u, 0u, 0u);  // default caching: the next GEMM re-reads x from L2
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = __bfloat1622float2(h[t]);
        s = fmaf(f.x, f.x, fmaf(f.y, f.y, s));
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) ss[row] = s;
}
// unfused MLP fallback: g <- silu(g) * u (bf16, 8 elements per thread)
__global__ void silu_mul_bf16(__nv_bfloat16* g, const __nv_bfloat16* u, int64_t n8) {
  // PDL (launch_pdl): wait for gate/up, release the down projection's weight prefetch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n8; e += (int64_t)gridDim.x * blockDim.x) {
    uint4 gv = reinterpret_cast<uint4*>(g)[e];
    const uint4 uv = reinterpret_cast<const uint4*>(u)[e];
    __nv_bfloat162* gh = reinterpret_cast<__nv_bfloat162*>(&gv);
    const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&uv);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 a = __bfloat1622float2(gh[i]), b = __bfloat1622float2(uh[i]);
      a.x = a.x / (1.f + __expf(-a.x)) * b.x;
      a.y = a.y / (1.f + __expf(-a.y)) * b.y;
      gh[i] = __floats2bfloat162_rn(a.x, a.y);
    }
    reinterpret_cast<uint4*>(g)[e] = gv;
  }
}

// ---------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------
enum Segment { SEG_FULL = 0, SEG_INPUT = 1, SEG_OUTPUT = 2 };

struct Operand {
  const void* p;
  int32_t dt;
  int64_t s_m, s_c;  // element strides: token, feature
};

struct TmapKey {
  const void* p;
  int64_t k, rows, ld;
  int box;
  int kind;  // 0: bf16 SW128 (box 64 x box); else: 1 + f32*2 + sw*4 with box_in in `extra`
  int extra;
  bool operator==(const TmapKey& o) const {
    return p == o.p && k == o.k && rows == o.rows && ld == o.ld && box == o.box && kind == o.kind &&
           extra == o.extra;
  }
};

}  // namespace tnl

struct tnl_plan {
  int32_t family = 0, d = 0, rm = 0, compute_dtype = TNL_F32, flags = 0;
  int64_t ms[TNL_MAX_MODES] = {0};
  int64_t rk[TNL_MAX_MODES + 1] = {0};
  int64_t rows = 0, cols = 0, row_begin = 0, row_end = 0;
  int64_t r_cut = 0, r_pad = 0, param_count = 0;
  int64_t chain_flops = 0, cut_flops = 0;
  bool tucker_cut_in = true;  // Tucker: cut = prod R_in (else prod R_out)
  int device = 0;
  // device arena
  void* arena = nullptr;
  size_t arena_bytes = 0;
  // generic fp32 cores (device, permuted layouts; see build_steps)
  std::vector<float*> gcore;  // TT/TR: per core; Tucker: [0]=core, [1+k]=factor k; dense: [0]
  // bf16 tensor-core panels
  __nv_bfloat16* bin = nullptr;   // (r_pad x cols)
  __nv_bfloat16* aout = nullptr;  // (rows_local x r_pad)
  __nv_bfloat16* u1t = nullptr;   // Tucker-2 chain: (R1p x cols)
  __nv_bfloat16* gmat = nullptr;  //                 (R0p x R1p)
  __nv_bfloat16* u0 = nullptr;    //                 (rows_local x R0p)
  int64_t r0p = 0, r1p = 0;
  __nv_bfloat16* wdense = nullptr;  // dense (rows_local x cols)
  unsigned long long* trace = nullptr;  // optional decode timeline buffer (debug)
  // tcgen05 core-by-core input chain (two-mode TT/TR input side)
  bool chain_ok = false;
  bool tucker_chain = false;  // Tucker-2 three-step chain plan
  __nv_bfloat16* chain_d = nullptr;  // Dp [(alpha, c_pad)][n_b]
  __nv_bfloat16* chain_c = nullptr;  // Cp [(j_a, b_pad)][c_pad]
  int32_t ch_na = 0, ch_nb = 0, ch_r0 = 0, ch_c = 0, ch_cpad = 0, ch_b = 0, ch_bpad = 0;
  // bf16 core-by-core chain on the tensor cores (tc_generic.cu), TNL_PLAN_CHAIN: the GENERIC step
  // list with bf16 cores / intermediates. tcg_out: two-mode input chain kernel, then the output
  // cores one by one; tcg_full: every core one by one (TT/TR of any shape, Tucker d >= 3).
  std::vector<__nv_bfloat16*> gcore16;
  bool tcg_out = false, tcg_full = false;

  float* gen_w_out = nullptr;       // generic dense rows slice (fp32) for sharded generic plans
  // fp32 merged cut (CUDA-core FFMA): B_in (r_cut x cols), A_out rows (rows_local x r_cut)
  float* bin32 = nullptr;
  float* aout32 = nullptr;
  int32_t plan_large = TNL_PLAN_GENERIC, plan_small = TNL_PLAN_GENERIC;
  int32_t decode_max_m = 0;
  int64_t max_state = 0;  // generic chain: max intermediate elements per token
  // host staging for tnl_forward_host
  int64_t max_m = 0;
  void* stage_x = nullptr;
  void* stage_y = nullptr;
  void* stage_ws = nullptr;
  size_t stage_ws_bytes = 0;
  // tensor-map cache
  std::mutex tm_mu;
  std::vector<std::pair<tnl::TmapKey, CUtensorMap>> tm_cache;
};

namespace tnl {

// Returns 0 and fills *m (by value: cache entries may move on insertion).
static int get_tmap(tnl_plan* P, CUtensorMap* m, const void* p, int64_t k, int64_t rows,
                    int64_t ld, int box) {
  TmapKey key{p, k, rows, ld, box, 0, 0};
  std::lock_guard<std::mutex> g(P->tm_mu);
  for (auto& e : P->tm_cache)
    if (e.first == key) {
      *m = e.second;
      return 0;
    }
  int err = make_tmap_bf16(m, p, k, rows, ld, box);
  if (err) return err;
  if (P->tm_cache.size() >= 64) P->tm_cache.erase(P->tm_cache.begin());
  P->tm_cache.emplace_back(key, *m);
  return 0;
}

// Cached general map (make_tmap_2d parameters).
static int get_tmap2(tnl_plan* P, CUtensorMap* m, const void* p, bool f32, int64_t inner,
                     int64_t outer, int64_t ld, int box_in, int box_out, int sw) {
  TmapKey key{p, inner, outer, ld, box_out, 1 + (f32 ? 1 : 0) + 2 * sw, box_in};
  std::lock_guard<std::mutex> g(P->tm_mu);
  for (auto& e : P->tm_cache)
    if (e.first == key) {
      *m = e.second;
      return 0;
    }
  int err = make_tmap_2d(m, p, f32, inner, outer, ld, box_in, box_out, sw);
  if (err) return err;
  if (P->tm_cache.size() >= 64) P->tm_cache.erase(P->tm_cache.begin());
  P->tm_cache.emplace_back(key, *m);
  return 0;
}

// ---------------------------------------------------------------------------
// Validation: tn_decompositions.py:97-126 (same checks, same messages)
// ---------------------------------------------------------------------------
static tnl_status validate_desc(const tnl_layer_desc* L) {
  if (!L) return fail(TNL_ERR_ARG, "null layer descriptor");
  const int d = L->ndim;
  if (d < 2 || d > TNL_MAX_MODES)
    return fail(TNL_ERR_SHAPE, "mode shape length must be in [2, %d], got %d", TNL_MAX_MODES, d);
  for (int k = 0; k < d; ++k)
    if (L->mode_shape[k] < 1)
      return fail(TNL_ERR_SHAPE, "all mode sizes must be >= 1, got %lld",
                  (long long)L->mode_shape[k]);
  if (!(1 <= L->row_mode_count && L->row_mode_count < d))
    return fail(TNL_ERR_SHAPE, "row_mode_count %d invalid for %d modes", L->row_mode_count, d);
  if (L->src_dtype != TNL_F64 && L->src_dtype != TNL_F32 && L->src_dtype != TNL_BF16)
    return fail(TNL_ERR_ARG, "unknown source dtype %d", L->src_dtype);
  switch (L->family) {
    case TNL_FAMILY_DENSE:
      if (!L->arrays[0]) return fail(TNL_ERR_SHAPE, "dense layer must hold its matricized payload");
      break;
    case TNL_FAMILY_TUCKER:
      if (!L->arrays[0]) return fail(TNL_ERR_SHAPE, "tucker layer needs a core and one factor per mode");
      for (int k = 0; k < d; ++k) {
        if (!L->arrays[1 + k])
          return fail(TNL_ERR_SHAPE, "tucker layer needs a core and one factor per mode");
        if (L->ranks[k] < 1) return fail(TNL_ERR_RANK, "ranks must be >= 1");
      }
      break;
    case TNL_FAMILY_TT:
    case TNL_FAMILY_TR:
      for (int k = 0; k < d; ++k) {
        if (!L->arrays[k]) return fail(TNL_ERR_SHAPE, "%s layer needs %d cores",
                                       L->family == TNL_FAMILY_TT ? "tt" : "tr", d);
        if (L->ranks[k] < 1 || L->ranks[k + 1] < 1) return fail(TNL_ERR_RANK, "ranks must be >= 1");
      }
      if (L->family == TNL_FAMILY_TT && (L->ranks[0] != 1 || L->ranks[d] != 1))
        return fail(TNL_ERR_SHAPE, "tt boundary ranks must be 1");
      if (L->family == TNL_FAMILY_TR && L->ranks[d] != L->ranks[0])
        return fail(TNL_ERR_SHAPE, "tr closing bond mismatch");
      break;
    default:
      return fail(TNL_ERR_SHAPE, "unknown family %d", L->family);
  }
  return TNL_OK;
}

// host conversion of one source array to float (with optional bf16 rounding)
static float bf16_round(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
static void load_host(const tnl_layer_desc* L, int idx, int64_t n, bool round, std::vector<float>& out) {
  out.resize(n);
  const void* src = L->arrays[idx];
  for (int64_t e = 0; e < n; ++e) {
    float v;
    if (L->src_dtype == TNL_F64)
      v = (float)static_cast<const double*>(src)[e];
    else if (L->src_dtype == TNL_F32)
      v = static_cast<const float*>(src)[e];
    else {
      uint16_t b = static_cast<const uint16_t*>(src)[e];
      uint32_t u = (uint32_t)b << 16;
      memcpy(&v, &u, 4);
    }
    out[e] = round ? bf16_round(v) : v;
  }
}

// ---------------------------------------------------------------------------
// Generic chain step construction (torch orientation, token-major states)
// ---------------------------------------------------------------------------
struct ChainIO {
  Operand in;   // x (FULL/INPUT) or cut state (OUTPUT)
  Operand out;  // y (FULL/OUTPUT) or cut state (INPUT)
  float* ws[2];
};

static GStep mk(int64_t b1, int64_t b2, int64_t I, int64_t P, int64_t J) {
  GStep s;
  memset(&s, 0, sizeof s);
  s.b1 = b1;
  s.b2 = b2;
  s.I = I;
  s.P = P;
  s.J = J;
  s.a_dt = s.b_dt = s.c_dt = DT_F32;
  return s;
}

// States (per token), TT/TR with closure size r0 (1 for TT):
//   input after core k : [alpha][pre(k)][b_k]        pre(k) = prod ms[rm..k-1]
//   cut                : [alpha][b_rm]   (kappa = alpha*b_rm + b)
//   output after core k: [alpha][a_k][post(k)]       post(k) = prod ms[k..rm-1]
//   y                  : [i_0][post(1)]
// Device core layouts (gcore): last core permuted to [alpha][j][c]; core 0
// permuted to [i0][(alpha, a)]; the others natural (b, n, c).
static void steps_ttr(const tnl_plan* P, int seg, int64_t M, const ChainIO& io,
                      std::vector<GStep>& out) {
  const int d = P->d, rm = P->rm;
  const int64_t* ms = P->ms;
  const int64_t* r = P->rk;  // bonds: core k is (r[k], ms[k], r[k+1])
  const int64_t r0 = r[0];
  int wsi = 0;
  // current state operand description
  const void* cur = nullptr;
  int cur_dt = DT_F32;
  auto next_ws = [&]() { float* p = io.ws[wsi]; wsi ^= 1; return p; };
  if (seg == SEG_FULL || seg == SEG_INPUT) {
    // k = d-1: state[m][alpha][pre][c] = sum_j x[m][pre][j] D[c][j][alpha]
    {
      const int k = d - 1;
      const int64_t pre = prod(ms, rm, k), n = ms[k], c = r[k];
      GStep s = mk(M, r0, pre, n, c);
      s.A = io.in.p;
      s.a_dt = io.in.dt;
      s.sa1 = io.in.s_m;
      s.sa2 = 0;
      s.sai = n * io.in.s_c;
      s.sap = io.in.s_c;
      s.B = P->gcore[k];
      s.sb1 = 0;
      s.sb2 = n * c;
      s.sbp = c;
      s.sbj = 1;
      const bool last = (k == rm) && seg == SEG_INPUT;
      if (last) {  // cut state [alpha][c] -> out operand kappa = alpha*c + b
        s.C = const_cast<void*>(io.out.p);
        s.c_dt = io.out.dt;
        s.sc1 = io.out.s_m;
        s.sc2 = c * io.out.s_c;
        s.sci = 0;
        s.scj = io.out.s_c;
      } else {
        float* w = next_ws();
        s.C = w;
        s.sc1 = r0 * pre * c;
        s.sc2 = pre * c;
        s.sci = c;
        s.scj = 1;
        cur = w;
      }
      out.push_back(s);
    }
    for (int k = d - 2; k >= rm; --k) {
      const int64_t pre = prod(ms, rm, k), n = ms[k], c = r[k + 1], b = r[k];
      GStep s = mk(M, r0, pre, n * c, b);
      s.A = cur;
      s.a_dt = DT_F32;
      s.sa1 = r0 * pre * n * c;
      s.sa2 = pre * n * c;
      s.sai = n * c;
      s.sap = 1;
      s.B = P->gcore[k];
      s.sbp = 1;
      s.sbj = n * c;
      const bool last = (k == rm) && seg == SEG_INPUT;
      if (last) {
        s.C = const_cast<void*>(io.out.p);
        s.c_dt = io.out.dt;
        s.sc1 = io.out.s_m;
        s.sc2 = b * io.out.s_c;
        s.sci = 0;
        s.scj = io.out.s_c;
      } else {
        float* w = next_ws();
        s.C = w;
        s.sc1 = r0 * pre * b;
        s.sc2 = pre * b;
        s.sci = b;
        s.scj = 1;
        cur = w;
      }
      out.push_back(s);
    }
    if (seg == SEG_INPUT) return;
  }
  // output side; state [m][alpha][a][post], cut has a = r[rm], post = 1
  int64_t a = r[rm], post = 1;
  int64_t s_m, s_alpha, s_a, s_post;
  if (seg == SEG_OUTPUT) {
    cur = io.in.p;
    cur_dt = io.in.dt;
    s_m = io.in.s_m;
    s_alpha = a * io.in.s_c;
    s_a = io.in.s_c;
    s_post = 0;
  } else {
    cur_dt = DT_F32;
    s_m = r0 * a;
    s_alpha = a;
    s_a = 1;
    s_post = 0;
  }
  for (int k = rm - 1; k >= 1; --k) {
    const int64_t n = ms[k], ap = r[k];  // core (ap, n, a)
    GStep s = mk(M, r0, ap * n, a, post);
    s.A = P->gcore[k];
    s.sai = a;
    s.sap = 1;
    s.B = cur;
    s.b_dt = cur_dt;
    s.sb1 = s_m;
    s.sb2 = s_alpha;
    s.sbp = s_a;
    s.sbj = post > 1 ? s_post : 1;
    float* w = next_ws();
    s.C = w;
    s.sc1 = r0 * ap * n * post;
    s.sc2 = ap * n * post;
    s.sci = post;
    s.scj = 1;
    out.push_back(s);
    cur = w;
    cur_dt = DT_F32;
    post *= n;
    a = ap;
    s_m = r0 * a * post;
    s_alpha = a * post;
    s_a = post;
    s_post = 1;
  }
  // core 0: y[m][i0][post] = sum_{(alpha,a)} G0p[i0][(alpha,a)] U[m][alpha][a][post]
  {
    const int64_t n0 = ms[0];
    GStep s = mk(M, 1, n0, r0 * a, post);
    s.A = P->gcore[0];
    s.sai = r0 * a;
    s.sap = 1;
    s.B = cur;
    s.b_dt = cur_dt;
    s.sb1 = s_m;
    s.sbp = s_a;  // (alpha, a) composite: alpha stride == a * s_a
    s.sbj = post > 1 ? s_post : 1;
    s.C = const_cast<void*>(io.out.p);
    s.c_dt = io.out.dt;
    s.sc1 = io.out.s_m;
    s.sci = post * io.out.s_c;
    s.scj = io.out.s_c;
    out.push_back(s);
  }
}

// Tucker: factors U_k (n_k x R_k), core G (R_0..R_{d-1}) as (Rout x Rin).
static void steps_tucker(const tnl_plan* P, int seg, int64_t M, const ChainIO& io,
                         std::vector<GStep>& out) {
  const int d = P->d, rm = P->rm;
  const int64_t* ms = P->ms;
  const int64_t* R = P->rk;
  const int64_t Rin = prod(R, rm, d), Rout = prod(R, 0, rm);
  int wsi = 0;
  auto next_ws = [&]() { float* p = io.ws[wsi]; wsi ^= 1; return p; };
  const bool cut_in = P->tucker_cut_in;
  // state description: [m][dims...] contiguous per token, with feature stride sf
  const void* cur = nullptr;
  int cur_dt = DT_F32;
  int64_t cur_sm = 0, cur_sf = 1;
  const bool do_in = (seg == SEG_FULL || seg == SEG_INPUT);
  const bool do_core = seg == SEG_FULL || (seg == SEG_INPUT && !cut_in) || (seg == SEG_OUTPUT && cut_in);
  const bool do_out = (seg == SEG_FULL || seg == SEG_OUTPUT);
  // which step is the final one of this segment
  int total = (do_in ? d - rm : 0) + (do_core ? 1 : 0) + (do_out ? rm : 0);
  int idx = 0;
  if (seg == SEG_OUTPUT || !do_in) {
    cur = io.in.p;
    cur_dt = io.in.dt;
    cur_sm = io.in.s_m;
    cur_sf = io.in.s_c;
  } else {
    cur = io.in.p;
    cur_dt = io.in.dt;
    cur_sm = io.in.s_m;
    cur_sf = io.in.s_c;
  }
  auto dst = [&](GStep& s, int64_t per_token) {
    ++idx;
    if (idx == total) {
      s.C = const_cast<void*>(io.out.p);
      s.c_dt = io.out.dt;
      return std::make_pair(io.out.s_m, io.out.s_c);
    }
    float* w = next_ws();
    s.C = w;
    s.c_dt = DT_F32;
    return std::make_pair(per_token, (int64_t)1);
  };
  if (do_in) {
    // state[m][pre_n][n_k][post_R] -> [m][pre_n][R_k][post_R], k = d-1 .. rm
    for (int k = d - 1; k >= rm; --k) {
      const int64_t pre = prod(ms, rm, k), n = ms[k], Rk = R[k], post = prod(R, k + 1, d);
      GStep s = mk(M, pre, Rk, n, post);
      s.A = P->gcore[1 + k];
      s.sai = 1;
      s.sap = Rk;  // A[i=R][p=j] = U[j][R]
      s.B = cur;
      s.b_dt = cur_dt;
      s.sb1 = cur_sm;
      s.sb2 = n * post * cur_sf;
      s.sbp = post * cur_sf;
      s.sbj = cur_sf;
      auto o = dst(s, pre * Rk * post);
      s.sc1 = o.first;
      s.sc2 = Rk * post * o.second;
      s.sci = post * o.second;
      s.scj = o.second;
      out.push_back(s);
      cur = s.C;
      cur_dt = s.c_dt;
      cur_sm = o.first;
      cur_sf = o.second;
    }
  }
  if (do_core) {
    GStep s = mk(1, 1, M, Rin, Rout);
    s.A = cur;
    s.a_dt = cur_dt;
    s.sai = cur_sm;
    s.sap = cur_sf;
    s.B = P->gcore[0];
    s.sbp = 1;
    s.sbj = Rin;
    auto o = dst(s, Rout);
    s.sci = o.first;
    s.scj = o.second;
    out.push_back(s);
    cur = s.C;
    cur_dt = s.c_dt;
    cur_sm = o.first;
    cur_sf = o.second;
  }
  if (do_out) {
    for (int k = 0; k < rm; ++k) {
      const int64_t pre = prod(ms, 0, k), n = ms[k], Rk = R[k], post = prod(R, k + 1, rm);
      GStep s = mk(M, pre, n, Rk, post);
      s.A = P->gcore[1 + k];
      s.sai = Rk;
      s.sap = 1;
      s.B = cur;
      s.b_dt = cur_dt;
      s.sb1 = cur_sm;
      s.sb2 = Rk * post * cur_sf;
      s.sbp = post * cur_sf;
      s.sbj = cur_sf;
      auto o = dst(s, pre * n * post);
      s.sc1 = o.first;
      s.sc2 = n * post * o.second;
      s.sci = post * o.second;
      s.scj = o.second;
      out.push_back(s);
      cur = s.C;
      cur_dt = s.c_dt;
      cur_sm = o.first;
      cur_sf = o.second;
    }
  }
}

static void steps_dense(const tnl_plan* P, int64_t M, const ChainIO& io, std::vector<GStep>& out) {
  GStep s = mk(1, 1, M, P->cols, P->rows);
  s.A = io.in.p;
  s.a_dt = io.in.dt;
  s.sai = io.in.s_m;
  s.sap = io.in.s_c;
  s.B = P->gcore[0];
  s.sbp = 1;
  s.sbj = P->cols;
  s.C = const_cast<void*>(io.out.p);
  s.c_dt = io.out.dt;
  s.sci = io.out.s_m;
  s.scj = io.out.s_c;
  out.push_back(s);
}

static void build_steps(const tnl_plan* P, int seg, int64_t M, const ChainIO& io,
                        std::vector<GStep>& out) {
  if (P->family == TNL_FAMILY_TT || P->family == TNL_FAMILY_TR)
    steps_ttr(P, seg, M, io, out);
  else if (P->family == TNL_FAMILY_TUCKER)
    steps_tucker(P, seg, M, io, out);
  else
    steps_dense(P, M, io, out);
}

static int64_t max_state_per_token(const tnl_plan* P) {
  const int d = P->d, rm = P->rm;
  const int64_t* ms = P->ms;
  const int64_t* r = P->rk;
  int64_t mx = 1;
  if (P->family == TNL_FAMILY_TT || P->family == TNL_FAMILY_TR) {
    const int64_t r0 = r[0];
    for (int k = d - 1; k >= rm; --k) mx = std::max(mx, r0 * prod(ms, rm, k) * r[k]);
    int64_t post = 1;
    for (int k = rm - 1; k >= 1; --k) {
      post *= ms[k];
      mx = std::max(mx, r0 * r[k] * post);
    }
  } else if (P->family == TNL_FAMILY_TUCKER) {
    for (int k = d - 1; k >= rm; --k) mx = std::max(mx, prod(ms, rm, k) * prod(r, k, d));
    mx = std::max(mx, prod(r, 0, rm));
    for (int k = 0; k < rm; ++k) mx = std::max(mx, prod(ms, 0, k + 1) * prod(r, k + 1, rm));
  }
  return mx;
}

// One GENERIC step as a tensor-core step (tc_generic.cu): batch dims that only one operand depends on
// are folded into that operand's free side (a core shared by every token becomes the B operand of
// an MMA whose N side runs over the tokens), the larger side becomes the MMA's M = 128 side.
static bool tcg_from_gstep(const GStep& g, TcgArgs* t) {
  if (g.a_dt != DT_BF16 || g.b_dt != DT_BF16) return false;
  struct D {
    int64_t size, so, sc;
  };
  std::vector<D> Is = {{g.I, g.sai, g.sci}}, Js = {{g.J, g.sbj, g.scj}}, Zs;
  std::vector<std::pair<int64_t, int64_t>> zab;  // (sa, sb) of the true batch dims
  auto batch = [&](int64_t b, int64_t sa, int64_t sb, int64_t sc) {
    if (b <= 1) return;
    if (sa == 0 && sb != 0)
      Js.insert(Js.begin(), {b, sb, sc});
    else if (sb == 0 && sa != 0)
      Is.insert(Is.begin(), {b, sa, sc});
    else {
      Zs.push_back({b, 0, sc});
      zab.push_back({sa, sb});
    }
  };
  batch(g.b2, g.sa2, g.sb2, g.sc2);
  batch(g.b1, g.sa1, g.sb1, g.sc1);
  auto squeeze = [](std::vector<D>& v) {
    std::vector<D> o;
    for (auto& e : v)
      if (e.size > 1) o.push_back(e);
    if (o.empty()) o.push_back({1, 0, 0});
    v = o;
  };
  squeeze(Is);
  squeeze(Js);
  if (Is.size() > 3 || Js.size() > 3 || Zs.size() > 2) return false;
  auto total = [](const std::vector<D>& v) {
    int64_t n = 1;
    for (auto& e : v) n *= e.size;
    return n;
  };
  const bool swap = total(Js) > total(Is);
  const std::vector<D>& Ms = swap ? Js : Is;
  const std::vector<D>& Ns = swap ? Is : Js;
  memset(t, 0, sizeof *t);
  t->A = static_cast<const __nv_bfloat16*>(swap ? g.B : g.A);
  t->B = static_cast<const __nv_bfloat16*>(swap ? g.A : g.B);
  t->ka = swap ? g.sbp : g.sap;
  t->kb = swap ? g.sap : g.sbp;
  t->C = g.C;
  t->c_f32 = g.c_dt == DT_F32;
  t->accumulate = g.accumulate;
  t->K = g.P;
  auto fill = [](const std::vector<D>& v, TcgSide& sd) {
    sd.nd = (int32_t)v.size();
    for (size_t i = 0; i < v.size(); ++i) {
      sd.size[i] = v[i].size;
      sd.so[i] = v[i].so;
      sd.sc[i] = v[i].sc;
    }
  };
  fill(Ms, t->m);
  fill(Ns, t->n);
  t->M = total(Ms);
  t->N = total(Ns);
  t->z1 = Zs.size() == 2 ? Zs[0].size : 1;
  t->z2 = Zs.empty() ? 1 : Zs.back().size;
  if (Zs.size() == 2) {
    t->za1 = swap ? zab[0].second : zab[0].first;
    t->zb1 = swap ? zab[0].first : zab[0].second;
    t->zc1 = Zs[0].sc;
  }
  if (!Zs.empty()) {
    t->za2 = swap ? zab.back().second : zab.back().first;
    t->zb2 = swap ? zab.back().first : zab.back().second;
    t->zc2 = Zs.back().sc;
  }
  auto vec_ok = [&](const __nv_bfloat16* p, int64_t ks, const TcgSide& sd, int64_t z1s, int64_t z2s) {
    if (ks != 1 || t->K % 8 || (reinterpret_cast<uintptr_t>(p) & 15) || z1s % 8 || z2s % 8) return 0;
    for (int i = 0; i < sd.nd; ++i)
      if (sd.size[i] > 1 && sd.so[i] % 8) return 0;
    return 1;
  };
  t->a_vec = vec_ok(t->A, t->ka, t->m, t->za1, t->za2);
  t->b_vec = vec_ok(t->B, t->kb, t->n, t->zb1, t->zb2);
  return true;
}

static int run_steps(const std::vector<GStep>& steps, cudaStream_t st) {
  for (const auto& s : steps) {
    int e = launch_generic_step(s, st);
    if (e) return e;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Flop accounting (SPEC.md:465-473 currency; SURVEY App. A canonical order)
// ---------------------------------------------------------------------------
static int64_t chain_flops(const tnl_plan* P) {
  const int d = P->d, rm = P->rm;
  const int64_t* ms = P->ms;
  const int64_t* r = P->rk;
  int64_t f = 0;
  if (P->family == TNL_FAMILY_DENSE) return 2 * P->rows * P->cols;
  if (P->family == TNL_FAMILY_TUCKER) {
    std::vector<int64_t> cur(ms + rm, ms + d);
    for (int k = d - 1; k >= rm; --k) {
      int64_t p = 1;
      for (auto v : cur) p *= v;
      f += 2 * p * r[k];
      cur[k - rm] = r[k];
    }
    f += 2 * prod(r, 0, rm) * prod(r, rm, d);
    std::vector<int64_t> c2(r, r + rm);
    for (int k = 0; k < rm; ++k) {
      int64_t p = 1;
      for (auto v : c2) p *= v;
      f += 2 * p * ms[k];
      c2[k] = ms[k];
    }
    return f;
  }
  const int64_t r0 = r[0];
  for (int k = rm; k < d; ++k) {
    int64_t mult = (k != d - 1 && r0 > 1) ? r0 : 1;
    f += 2 * prod(ms, rm, k) * ms[k] * r[k + 1] * r[k] * mult;
  }
  for (int k = 0; k < rm; ++k) {
    int64_t mult = (k != 0 && r0 > 1) ? r0 : 1;
    f += 2 * prod(ms, k + 1, rm) * r[k + 1] * ms[k] * r[k] * mult;
  }
  return f;
}

// ---------------------------------------------------------------------------
// Device-side panel construction (fp32 generic steps on identity inputs)
// ---------------------------------------------------------------------------
static tnl_status alloc_arena(tnl_plan* P, size_t bytes) {
  CUDA_TRY(dev_alloc(&P->arena, bytes));
  P->arena_bytes = bytes;
  CUDA_TRY(cudaMemset(P->arena, 0, bytes));
  return TNL_OK;
}

// Direct two-mode panel construction (see build_panel_f32); TNL_ERR_UNSUPPORTED when the side is
// not two modes (or the row range is not aligned to the second output mode).
static tnl_status build_panel_2mode(tnl_plan* P, int seg, float* out, cudaStream_t st) {
  const int d = P->d, rm = P->rm;
  const int64_t* ms = P->ms;
  const int64_t* r = P->rk;
  const int64_t K = P->r_cut;
  const bool ttr = P->family == TNL_FAMILY_TT || P->family == TNL_FAMILY_TR;
  const bool tucker = P->family == TNL_FAMILY_TUCKER;
  if (!(ttr || tucker)) return TNL_ERR_UNSUPPORTED;
  if (seg == SEG_INPUT && d - rm == 2) {
    const int64_t na = ms[rm], nb = ms[d - 1];
    if (ttr) {
      // B_in[alpha*B + b][ja*nb + jb] = sum_c C[b][ja][c] D[c][jb][alpha]; C natural (B, na, c),
      // D permuted [alpha][jb][c]
      const int64_t B = r[rm], c = r[d - 1], r0 = r[d];
      GStep g = mk(r0, 1, B * na, c, nb);
      g.A = P->gcore[rm];
      g.sai = c;
      g.sap = 1;
      g.B = P->gcore[d - 1];
      g.sb1 = nb * c;
      g.sbp = 1;
      g.sbj = c;
      g.C = out;
      g.sc1 = B * P->cols;
      g.sci = nb;
      g.scj = 1;
      if (launch_generic_step(g, st)) return fail(TNL_ERR_CUDA, "panel (two-mode input) launch failed");
    } else if (P->tucker_cut_in) {
      // B_in[(ra, rb)][(ja, jb)] = Ua[ja][ra] * Ub[jb][rb]
      const int64_t Ra = r[rm], Rb = r[d - 1];
      const int64_t n = Ra * Rb * na * nb;
      kron2_f32<<<grid_for(n), 256, 0, st>>>(out, P->gcore[1 + rm], 1, Ra, P->gcore[1 + d - 1], 1, Rb, Ra, Rb, na, nb);
    } else {
      // B_in[kappa][(ja, jb)] = sum_{ra, rb} G[kappa][ra][rb] Ua[ja][ra] Ub[jb][rb]  (kappa = out ranks)
      const int64_t Ra = r[rm], Rb = r[d - 1];
      float* w = nullptr;
      CUDA_TRY(dev_alloc(&w, sizeof(float) * K * Ra * nb));
      GStep g1 = mk(1, 1, K * Ra, Rb, nb);  // W[(kappa, ra)][jb] = sum_rb G[(kappa, ra)][rb] Ub[jb][rb]
      g1.A = P->gcore[0];
      g1.sai = Rb;
      g1.sap = 1;
      g1.B = P->gcore[1 + d - 1];
      g1.sbp = 1;
      g1.sbj = Rb;
      g1.C = w;
      g1.sci = nb;
      g1.scj = 1;
      GStep g2 = mk(K, 1, na, Ra, nb);  // B_in[kappa][ja][jb] = sum_ra Ua[ja][ra] W[kappa][ra][jb]
      g2.A = P->gcore[1 + rm];
      g2.sai = Ra;
      g2.sap = 1;
      g2.B = w;
      g2.sb1 = Ra * nb;
      g2.sbp = nb;
      g2.sbj = 1;
      g2.C = out;
      g2.sc1 = P->cols;
      g2.sci = nb;
      g2.scj = 1;
      const bool bad = launch_generic_step(g1, st) || launch_generic_step(g2, st);
      cudaStreamSynchronize(st);
      dev_free(w);
      if (bad) return fail(TNL_ERR_CUDA, "panel (two-mode Tucker input) launch failed");
    }
  } else if (seg == SEG_OUTPUT && rm == 2 && P->row_begin % ms[1] == 0 && P->row_end % ms[1] == 0) {
    const int64_t n1 = ms[1];
    const int64_t i0b = P->row_begin / n1, n0l = (P->row_end - P->row_begin) / n1;
    if (ttr) {
      // A_out[(i0, i1)][alpha*B + b] = sum_a A0[i0][(alpha, a)] B1[a][i1][b]; A0 permuted [i0][(alpha, a)]
      const int64_t r0 = r[0], a = r[1], B = r[2];
      GStep g = mk(r0, n1, n0l, a, B);
      g.A = P->gcore[0] + i0b * r0 * a;
      g.sa1 = a;
      g.sai = r0 * a;
      g.sap = 1;
      g.B = P->gcore[1];
      g.sb2 = B;
      g.sbp = n1 * B;
      g.sbj = 1;
      g.C = out;
      g.sc1 = B;
      g.sc2 = K;
      g.sci = n1 * K;
      g.scj = 1;
      if (launch_generic_step(g, st)) return fail(TNL_ERR_CUDA, "panel (two-mode output) launch failed");
    } else if (!P->tucker_cut_in) {
      // A_out[(i0, i1)][(r0, r1)] = U0[i0][r0] * U1[i1][r1]
      const int64_t R0 = r[0], R1 = r[1];
      const int64_t n = n0l * n1 * R0 * R1;
      kron2_f32<<<grid_for(n), 256, 0, st>>>(out, P->gcore[1] + i0b * R0, R0, 1, P->gcore[2], R1, 1, n0l, n1, R0, R1);
    } else {
      // A_out[i0][i1][kappa] = sum_r0 U0[i0][r0] sum_r1 U1[i1][r1] G[r0][r1][kappa]
      const int64_t R0 = r[0], R1 = r[1];
      float* w = nullptr;
      CUDA_TRY(dev_alloc(&w, sizeof(float) * R0 * n1 * K));
      GStep g1 = mk(R0, 1, n1, R1, K);  // W[r0][i1][kappa]
      g1.A = P->gcore[2];
      g1.sai = R1;
      g1.sap = 1;
      g1.B = P->gcore[0];
      g1.sb1 = R1 * K;
      g1.sbp = K;
      g1.sbj = 1;
      g1.C = w;
      g1.sc1 = n1 * K;
      g1.sci = K;
      g1.scj = 1;
      GStep g2 = mk(1, 1, n0l, R0, n1 * K);  // A_out[i0][(i1, kappa)]
      g2.A = P->gcore[1] + i0b * R0;
      g2.sai = R0;
      g2.sap = 1;
      g2.B = w;
      g2.sbp = n1 * K;
      g2.sbj = 1;
      g2.C = out;
      g2.sci = n1 * K;
      g2.scj = 1;
      const bool bad = launch_generic_step(g1, st) || launch_generic_step(g2, st);
      cudaStreamSynchronize(st);
      dev_free(w);
      if (bad) return fail(TNL_ERR_CUDA, "panel (two-mode Tucker output) launch failed");
    }
  } else {
    return TNL_ERR_UNSUPPORTED;
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  return TNL_OK;
}

// Computes the fp32 (rows_out x K) matrix  OUT[i][kappa] for SEG_OUTPUT
// (A_out restricted to [row_begin,row_end)) or OUT[kappa][j] for SEG_INPUT (B_in),
// by running the segment's chain on identity inputs in chunks.
static tnl_status build_panel_f32(tnl_plan* P, int seg, float* out, cudaStream_t st) {
  const int64_t K = P->r_cut;
  // Single-mode sides: the panel is one core, permuted (TT/TR, Tucker factor) or one
  // GEMM (Tucker U0 . G); no identity chain needed.
  const int d = P->d, rm = P->rm;
  const int64_t nr = P->row_end - P->row_begin;
  const bool ttr = P->family == TNL_FAMILY_TT || P->family == TNL_FAMILY_TR;
  if (seg == SEG_INPUT && d - rm == 1 && (ttr || P->tucker_cut_in)) {
    const int64_t n = P->ms[d - 1];
    if (ttr) {  // B_in[(alpha,b)][j] = D[b][j][alpha]; gcore[d-1] is [alpha][j][b]
      const int64_t b = P->rk[d - 1], r0 = P->rk[d];
      for (int64_t al = 0; al < r0; ++al)
        copy_2d_any<<<grid_for(b * n), 256, 0, st>>>(P->gcore[d - 1] + al * n * b, DT_F32, 1, b,
                                                     out + al * b * n, DT_F32, n, 1, b, n);
    } else {  // B_in = U_{d-1}^T
      const int64_t R = P->rk[d - 1];
      copy_2d_any<<<grid_for(R * n), 256, 0, st>>>(P->gcore[1 + d - 1], DT_F32, 1, R, out, DT_F32, n, 1, R, n);
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaGetLastError());
    return TNL_OK;
  }
  if (seg == SEG_OUTPUT && rm == 1) {
    if (ttr) {  // A_out[i][(alpha,b)] = G0[alpha][i][b]; gcore[0] is [i][(alpha,b)] already
      copy_2d_any<<<grid_for(nr * K), 256, 0, st>>>(P->gcore[0] + P->row_begin * K, DT_F32, K, 1, out, DT_F32, K,
                                                    1, nr, K);
    } else if (P->tucker_cut_in) {  // A_out = U0[rows] . G  (rows x R_in)
      const int64_t R0 = P->rk[0], Rin = K;
      GStep g = mk(1, 1, nr, R0, Rin);
      g.A = P->gcore[1] + P->row_begin * R0;
      g.sai = R0;
      g.sap = 1;
      g.B = P->gcore[0];
      g.sbp = Rin;
      g.sbj = 1;
      g.C = out;
      g.sci = Rin;
      g.scj = 1;
      if (launch_generic_step(g, st)) return fail(TNL_ERR_CUDA, "panel GEMM launch failed");
    } else {  // cut on R_out: A_out = U0[rows]
      copy_2d_any<<<grid_for(nr * K), 256, 0, st>>>(P->gcore[1] + P->row_begin * K, DT_F32, K, 1, out, DT_F32, K,
                                                    1, nr, K);
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaGetLastError());
    return TNL_OK;
  }
  // Two-mode sides (every BASELINE shape with d = 4, rm = 2): the panel is one contraction of the
  // side's two cores (TT/TR: one batched step per closure index; Tucker: a Kronecker product of
  // the two factors, or two factor steps applied to the core), built directly instead of by
  // running the chain on identity columns (cfg4 down projections: 25600 identity columns).
  {
    tnl_status ds = build_panel_2mode(P, seg, out, st);
    if (ds != TNL_ERR_UNSUPPORTED) return ds;
  }
  const int64_t n_in = (seg == SEG_INPUT) ? P->cols : K;       // identity size
  const int64_t chunk = std::min<int64_t>(n_in, 512);
  float *eye = nullptr, *ws0 = nullptr, *ws1 = nullptr, *tmp = nullptr;
  const int64_t ms_tok = std::max<int64_t>(max_state_per_token(P), 1);
  const int64_t out_feats = (seg == SEG_INPUT) ? K : P->rows;
  CUDA_TRY(dev_alloc(&eye, sizeof(float) * chunk * n_in));
  CUDA_TRY(dev_alloc(&ws0, sizeof(float) * chunk * ms_tok));
  CUDA_TRY(dev_alloc(&ws1, sizeof(float) * chunk * ms_tok));
  CUDA_TRY(dev_alloc(&tmp, sizeof(float) * chunk * out_feats));
  tnl_status st_ret = TNL_OK;
  for (int64_t c0 = 0; c0 < n_in && st_ret == TNL_OK; c0 += chunk) {
    const int64_t m = std::min(chunk, n_in - c0);
    identity_f32<<<grid_for(m * n_in), 256, 0, st>>>(eye, m, n_in, c0);
    ChainIO io;
    io.in = Operand{eye, DT_F32, n_in, 1};
    io.out = Operand{tmp, DT_F32, out_feats, 1};
    io.ws[0] = ws0;
    io.ws[1] = ws1;
    std::vector<GStep> steps;
    build_steps(P, seg, m, io, steps);
    if (run_steps(steps, st)) st_ret = fail(TNL_ERR_CUDA, "panel build launch failed");
    // tmp[mm][f]: SEG_INPUT -> B_in[f][c0+mm]; SEG_OUTPUT -> A_out[f-row_begin][c0+mm]
    if (seg == SEG_INPUT) {
      copy_2d_any<<<grid_for(m * K), 256, 0, st>>>(tmp, DT_F32, K, 1, out + c0, DT_F32, 1, P->cols,
                                                   m, K);
    } else {
      const int64_t nr = P->row_end - P->row_begin;
      copy_2d_any<<<grid_for(m * nr), 256, 0, st>>>(tmp + P->row_begin, DT_F32, P->rows, 1,
                                                    out + c0, DT_F32, 1, K, m, nr);
    }
  }
  cudaStreamSynchronize(st);
  dev_free(eye);
  dev_free(ws0);
  dev_free(ws1);
  dev_free(tmp);
  if (st_ret == TNL_OK) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TNL_ERR_CUDA, "panel build: %s", cudaGetErrorString(e));
  }
  return st_ret;
}

// ---------------------------------------------------------------------------
// tnl_plan_create
// ---------------------------------------------------------------------------
static tnl_status create_impl(const tnl_layer_desc* L, int32_t compute_dtype, int64_t max_m,
                              int32_t flags, int64_t row_begin, int64_t row_end, tnl_plan** out) {
  if (!out) return fail(TNL_ERR_ARG, "null output pointer");
  *out = nullptr;
  tnl_status vs = validate_desc(L);
  if (vs != TNL_OK) return vs;
  if (compute_dtype != TNL_F32 && compute_dtype != TNL_BF16)
    return fail(TNL_ERR_ARG, "compute dtype must be TNL_F32 or TNL_BF16");
  std::unique_ptr<tnl_plan> P(new tnl_plan());
  struct DetGuard {  // deterministic panel construction (generic.cuh)
    DetGuard() { set_generic_deterministic(true); }
    ~DetGuard() { set_generic_deterministic(false); }
  } det_guard;
  BuildTimer bt;
  P->family = L->family;
  P->d = L->ndim;
  P->rm = L->row_mode_count;
  P->compute_dtype = compute_dtype;
  P->flags = flags;
  for (int k = 0; k < P->d; ++k) P->ms[k] = L->mode_shape[k];
  for (int k = 0; k <= P->d; ++k) P->rk[k] = L->ranks[k];
  const int d = P->d, rm = P->rm;
  P->rows = prod(P->ms, 0, rm);
  P->cols = prod(P->ms, rm, d);
  if (row_begin == 0 && row_end == 0) row_end = P->rows;
  if (!(0 <= row_begin && row_begin < row_end && row_end <= P->rows))
    return fail(TNL_ERR_SHAPE, "row range [%lld, %lld) outside %lld rows", (long long)row_begin,
                (long long)row_end, (long long)P->rows);
  P->row_begin = row_begin;
  P->row_end = row_end;
  CUDA_TRY(cudaGetDevice(&P->device));
  const bool bf16 = compute_dtype == TNL_BF16;
  const int64_t* ms = P->ms;
  const int64_t* r = P->rk;

  // ---- load cores to host fp32, permute into generic layouts ----
  std::vector<std::vector<float>> host;  // generic layouts
  int64_t pc = 0;
  if (P->family == TNL_FAMILY_DENSE) {
    std::vector<float> w;
    load_host(L, 0, P->rows * P->cols, bf16, w);
    pc = P->rows * P->cols;
    host.push_back(std::move(w));
    P->r_cut = std::min(P->rows, P->cols);
  } else if (P->family == TNL_FAMILY_TUCKER) {
    std::vector<float> g;
    load_host(L, 0, prod(r, 0, d), bf16, g);
    pc += (int64_t)g.size();
    host.push_back(std::move(g));
    for (int k = 0; k < d; ++k) {
      std::vector<float> u;
      load_host(L, 1 + k, ms[k] * r[k], bf16, u);
      pc += (int64_t)u.size();
      host.push_back(std::move(u));
    }
    const int64_t Rin = prod(r, rm, d), Rout = prod(r, 0, rm);
    P->tucker_cut_in = Rin <= Rout;
    P->r_cut = std::min(Rin, Rout);
  } else {
    const int64_t r0 = r[0];
    for (int k = 0; k < d; ++k) {
      std::vector<float> c;
      const int64_t a = r[k], n = ms[k], b = r[k + 1];
      load_host(L, k, a * n * b, bf16, c);
      pc += (int64_t)c.size();
      if (k == d - 1) {  // [alpha][j][c] = D[c][j][alpha]
        std::vector<float> p(c.size());
        for (int64_t cc = 0; cc < a; ++cc)
          for (int64_t j = 0; j < n; ++j)
            for (int64_t al = 0; al < b; ++al) p[(al * n + j) * a + cc] = c[(cc * n + j) * b + al];
        c.swap(p);
      } else if (k == 0) {  // [i0][(alpha, a)] = G0[alpha][i0][a]
        std::vector<float> p(c.size());
        for (int64_t al = 0; al < a; ++al)
          for (int64_t i = 0; i < n; ++i)
            for (int64_t aa = 0; aa < b; ++aa) p[i * (a * b) + al * b + aa] = c[(al * n + i) * b + aa];
        c.swap(p);
      }
      host.push_back(std::move(c));
    }
    // d == 1 never (d >= 2). If d-1 == 0 impossible.
    P->r_cut = r0 * r[rm];
  }
  P->param_count = pc;
  bt.mark("host_load");
  P->chain_flops = chain_flops(P.get());
  P->cut_flops = 2 * P->r_cut * (P->rows + P->cols);
  P->max_state = max_state_per_token(P.get());
  P->r_pad = round_up(P->r_cut, 16);

  // ---- choose plans ----
  const bool tc_ok = bf16 && (P->cols % 8 == 0) && !(flags & TNL_PLAN_GENERIC);
  const int64_t rows_local = P->row_end - P->row_begin;
  const bool tucker2 = P->family == TNL_FAMILY_TUCKER && d == 2;
  int32_t large = TNL_PLAN_GENERIC;
  if (tc_ok) {
    if (P->family == TNL_FAMILY_DENSE)
      large = TNL_PLAN_CUT;  // single GEMM (W plays A_out, identity cut)
    else if ((flags & TNL_PLAN_CHAIN) && tucker2)
      large = TNL_PLAN_CHAIN;
    else
      large = TNL_PLAN_CUT;
  }
  // core-by-core tcgen05 chain for a two-mode TT/TR input side (cores C = core rm, D = core d-1)
  if (tc_ok && (P->family == TNL_FAMILY_TT || P->family == TNL_FAMILY_TR) && d - rm == 2) {
    const int64_t c = r[d - 1], b = r[rm], r0 = r[d], na = ms[rm], nb = ms[d - 1];
    const int64_t cpad = c <= 16 ? 16 : (c <= 32 ? 32 : (c <= 64 ? 64 : 0));
    const int64_t bpad = round_up(b, 16);
    if (cpad && nb % 16 == 0 && r0 * cpad <= 256 && r0 * bpad <= 256) {
      P->chain_ok = true;
      P->ch_na = (int32_t)na;
      P->ch_nb = (int32_t)nb;
      P->ch_r0 = (int32_t)r0;
      P->ch_c = (int32_t)c;
      P->ch_cpad = (int32_t)cpad;
      P->ch_b = (int32_t)b;
      P->ch_bpad = (int32_t)bpad;
      if (flags & TNL_PLAN_CHAIN) large = TNL_PLAN_CHAIN;
    }
  }
  // fp32: the merged cut on CUDA cores (two FFMA steps through an r_cut-wide fp32 T) whenever it
  // needs fewer flops than the core-by-core chain; TNL_PLAN_GENERIC / _CHAIN keep the chain
  const bool cut32 = !bf16 && P->family != TNL_FAMILY_DENSE && !(flags & (TNL_PLAN_GENERIC | TNL_PLAN_CHAIN)) &&
                     P->cut_flops <= P->chain_flops;
  if (cut32) large = TNL_PLAN_CUT;
  // bf16 core-by-core chain for every other TT/TR/Tucker shape (unsharded plans)
  if (tc_ok && (flags & TNL_PLAN_CHAIN) && P->family != TNL_FAMILY_DENSE && !tucker2 && P->row_begin == 0 &&
      P->row_end == P->rows) {
    if (P->chain_ok) {
      P->tcg_out = rm >= 2;  // rm == 1: the output "panel" is the single output core itself
    } else {
      P->tcg_full = true;
      large = TNL_PLAN_CHAIN;
    }
  }
  P->plan_large = large;
  P->plan_small = large;
  P->decode_max_m = (tc_ok && P->family != TNL_FAMILY_DENSE && round_up(P->r_cut, 16) <= 256 &&
                     !(flags & TNL_PLAN_NO_DECODE)) ? 64 : 0;
  if (P->decode_max_m) P->plan_small = TNL_PLAN_CUT;

  // ---- device arena: generic cores + panels ----
  size_t bytes = 0;
  std::vector<size_t> off;
  for (auto& h : host) {
    off.push_back(bytes);
    bytes += round_up((int64_t)h.size() * 4, 256);
  }
  size_t off_bin = 0, off_aout = 0, off_u1 = 0, off_g = 0, off_u0 = 0, off_w = 0;
  const bool dense = P->family == TNL_FAMILY_DENSE;
  const bool want_cut = tc_ok && !dense;
  if (want_cut) {
    off_bin = bytes;
    bytes += round_up(P->r_pad * P->cols * 2, 256);
    off_aout = bytes;
    bytes += round_up(rows_local * P->r_pad * 2, 256);
  }
  if (large == TNL_PLAN_CUT && dense) {
    off_w = bytes;
    bytes += round_up(rows_local * P->cols * 2, 256);
  }
  size_t off_b32 = 0, off_a32 = 0;
  if (cut32) {
    off_b32 = bytes;
    bytes += round_up(P->r_cut * P->cols * 4, 256);
    off_a32 = bytes;
    bytes += round_up(rows_local * P->r_cut * 4, 256);
  }
  std::vector<size_t> off16;
  if (P->tcg_out || P->tcg_full)
    for (auto& h : host) {
      off16.push_back(bytes);
      bytes += round_up((int64_t)h.size() * 2, 256);
    }
  size_t off_chd = 0, off_chc = 0;
  if (P->chain_ok) {
    off_chd = bytes;
    bytes += round_up((int64_t)P->ch_r0 * P->ch_cpad * P->ch_nb * 2, 256);
    off_chc = bytes;
    bytes += round_up((int64_t)P->ch_na * P->ch_bpad * P->ch_cpad * 2, 256);
  }
  P->tucker_chain = large == TNL_PLAN_CHAIN && tucker2;
  if (P->tucker_chain) {
    P->r1p = round_up(r[1], 16);
    P->r0p = round_up(r[0], 16);
    off_u1 = bytes;
    bytes += round_up(P->r1p * P->cols * 2, 256);
    off_g = bytes;
    bytes += round_up(P->r0p * P->r1p * 2, 256);
    off_u0 = bytes;
    bytes += round_up(rows_local * P->r0p * 2, 256);
  }
  tnl_status as = alloc_arena(P.get(), bytes);
  if (as != TNL_OK) return as;
  bt.mark("arena");
  char* base = static_cast<char*>(P->arena);
  for (size_t i = 0; i < host.size(); ++i) {
    float* dptr = reinterpret_cast<float*>(base + off[i]);
    CUDA_TRY(cudaMemcpy(dptr, host[i].data(), host[i].size() * 4, cudaMemcpyHostToDevice));
    P->gcore.push_back(dptr);
  }
  bt.mark("upload");
  cudaStream_t st = 0;
  for (size_t i = 0; i < off16.size(); ++i) {
    __nv_bfloat16* d16 = reinterpret_cast<__nv_bfloat16*>(base + off16[i]);
    to_bf16(P->gcore[i], d16, (int64_t)host[i].size(), st);
    P->gcore16.push_back(d16);
  }
  if (large == TNL_PLAN_CUT && dense) {
    P->wdense = reinterpret_cast<__nv_bfloat16*>(base + off_w);
    copy_2d_any<<<grid_for(rows_local * P->cols), 256, 0, st>>>(
        P->gcore[0] + P->row_begin * P->cols, DT_F32, P->cols, 1, P->wdense, DT_BF16, P->cols, 1,
        rows_local, P->cols);
  }
  if (want_cut) {
    P->bin = reinterpret_cast<__nv_bfloat16*>(base + off_bin);
    P->aout = reinterpret_cast<__nv_bfloat16*>(base + off_aout);
    float *fb = nullptr, *fa = nullptr;
    CUDA_TRY(dev_alloc(&fb, sizeof(float) * P->r_cut * P->cols));
    CUDA_TRY(dev_alloc(&fa, sizeof(float) * rows_local * P->r_cut));
    tnl_status s1 = build_panel_f32(P.get(), SEG_INPUT, fb, st);
    tnl_status s2 = s1 == TNL_OK ? build_panel_f32(P.get(), SEG_OUTPUT, fa, st) : s1;
    if (s2 == TNL_OK) {
      copy_2d_any<<<grid_for(P->r_cut * P->cols), 256, 0, st>>>(fb, DT_F32, P->cols, 1, P->bin,
                                                                DT_BF16, P->cols, 1, P->r_cut,
                                                                P->cols);
      copy_2d_any<<<grid_for(rows_local * P->r_cut), 256, 0, st>>>(
          fa, DT_F32, P->r_cut, 1, P->aout, DT_BF16, P->r_pad, 1, rows_local, P->r_cut);
    }
    cudaStreamSynchronize(st);
    dev_free(fb);
    dev_free(fa);
    if (s2 != TNL_OK) return s2;
    bt.mark("panels");
  }
  if (cut32) {
    P->bin32 = reinterpret_cast<float*>(base + off_b32);
    P->aout32 = reinterpret_cast<float*>(base + off_a32);
    tnl_status s1 = build_panel_f32(P.get(), SEG_INPUT, P->bin32, st);
    if (s1 == TNL_OK) s1 = build_panel_f32(P.get(), SEG_OUTPUT, P->aout32, st);
    CUDA_TRY(cudaStreamSynchronize(st));
    if (s1 != TNL_OK) return s1;
  }
  if (P->chain_ok) {
    const int64_t na = P->ch_na, nb = P->ch_nb, r0 = P->ch_r0, c = P->ch_c, cp = P->ch_cpad,
                  b = P->ch_b, bp = P->ch_bpad;
    std::vector<__nv_bfloat16> hd(r0 * cp * nb, __float2bfloat16(0.f)), hc(na * bp * cp, __float2bfloat16(0.f));
    const std::vector<float>& D = host[d - 1];  // permuted [alpha][j][c]
    const std::vector<float>& C = host[rm];     // natural (b, n_a, c)
    for (int64_t al = 0; al < r0; ++al)
      for (int64_t j = 0; j < nb; ++j)
        for (int64_t cc = 0; cc < c; ++cc)
          hd[(al * cp + cc) * nb + j] = __float2bfloat16(D[(al * nb + j) * c + cc]);
    for (int64_t ja = 0; ja < na; ++ja)
      for (int64_t bb = 0; bb < b; ++bb)
        for (int64_t cc = 0; cc < c; ++cc)
          hc[(ja * bp + bb) * cp + cc] = __float2bfloat16(C[(bb * na + ja) * c + cc]);
    P->chain_d = reinterpret_cast<__nv_bfloat16*>(base + off_chd);
    P->chain_c = reinterpret_cast<__nv_bfloat16*>(base + off_chc);
    CUDA_TRY(cudaMemcpy(P->chain_d, hd.data(), hd.size() * 2, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(P->chain_c, hc.data(), hc.size() * 2, cudaMemcpyHostToDevice));
  }
  if (large == TNL_PLAN_CHAIN && tucker2) {
    // Tucker-2: U1^T (R1p x cols), G (R0p x R1p), U0 rows (rows_local x R0p)
    P->u1t = reinterpret_cast<__nv_bfloat16*>(base + off_u1);
    P->gmat = reinterpret_cast<__nv_bfloat16*>(base + off_g);
    P->u0 = reinterpret_cast<__nv_bfloat16*>(base + off_u0);
    copy_2d_any<<<grid_for(r[1] * P->cols), 256, 0, st>>>(P->gcore[2], DT_F32, 1, r[1], P->u1t,
                                                          DT_BF16, P->cols, 1, r[1], P->cols);
    copy_2d_any<<<grid_for(r[0] * r[1]), 256, 0, st>>>(P->gcore[0], DT_F32, r[1], 1, P->gmat,
                                                       DT_BF16, P->r1p, 1, r[0], r[1]);
    copy_2d_any<<<grid_for(rows_local * r[0]), 256, 0, st>>>(
        P->gcore[1] + P->row_begin * r[0], DT_F32, r[0], 1, P->u0, DT_BF16, P->r0p, 1, rows_local,
        r[0]);
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());

  bt.mark("chain_ops");
  // ---- host staging for tnl_forward_host ----
  P->max_m = max_m;
  if (max_m > 0) {
    const size_t es = bf16 ? 2 : 4;
    CUDA_TRY(dev_alloc(&P->stage_x, es * max_m * P->cols));
    CUDA_TRY(dev_alloc(&P->stage_y, es * max_m * rows_local));
  }
  if (bt.on)
    fprintf(stderr, "[tnl build] family=%d d=%d rm=%d rows=%lld cols=%lld r_cut=%lld%s\n", P->family, P->d, P->rm,
            (long long)P->rows, (long long)P->cols, (long long)P->r_cut, bt.buf);
  *out = P.release();
  return TNL_OK;
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
static constexpr int64_t kSwapMaxM = 64;  // tokens: swap-AB (weights on the M side) below this

constexpr size_t kDecHeadBytes = sizeof(float) * 64 * 512;  // decode accumulator (r_pad <= 256; 512 for a stacked gate/up cut)
// one decode slot = accumulator + counter + the GEMV variant's T scratch (M <= 8, r_pad <= 256).
// Every workspace layout reserves kDecSlots slots at fixed offsets, so a decode call may run on
// slot 1 (a forked stream) concurrently with one on slot 0 (MLP gate || up) and no layout ever
// places scratch inside a zero-at-rest accumulator.
constexpr size_t kDecSlotBytes = kDecHeadBytes + 256 + sizeof(float) * 8 * 256;
constexpr int kDecSlots = 3;  // slots 0..2 double as the three rotating accumulators of a fused stack

static size_t ws_layout(const tnl_plan* P, int64_t M, size_t* o_f32, size_t* o_b0, size_t* o_b1,
                        size_t* o_s = nullptr) {
  size_t bytes = 0;
  auto take = [&](size_t n) {
    size_t o = bytes;
    bytes += round_up((int64_t)n, 256);
    return o;
  };
  const int64_t rows_local = P->row_end - P->row_begin;
  if (P->plan_large == TNL_PLAN_GENERIC) {
    *o_b0 = take(sizeof(float) * M * P->max_state);
    *o_b1 = take(sizeof(float) * M * P->max_state);
    // sharded generic plans compute full rows into a temp y
    *o_f32 = (rows_local != P->rows) ? take(sizeof(float) * M * P->rows) : 0;
    return bytes;
  }
  // decode accumulator + counter (zero at rest: the caller zero-fills the workspace once). The
  // head has the same size for every decode-capable plan (the 64 x 256 fp32 maximum) so plans
  // sharing one workspace (stacks, MLP blocks) never place scratch inside another plan's
  // zero-at-rest accumulator.
  // (reserved even by plans without a decode path, whose prefill scratch would otherwise land
  // in the head of a decode-capable plan sharing the workspace)
  take(kDecSlots * kDecSlotBytes);
  int64_t kmax = P->r_pad;
  if (P->tucker_chain) kmax = std::max(P->r0p, P->r1p);
  *o_f32 = take(sizeof(float) * M * kmax);
  *o_b0 = take(2 * M * kmax);
  *o_b1 = take(2 * M * kmax);
  if (P->tcg_out || P->tcg_full) {  // the bf16 chain's two intermediate states + split-K scratch
    const size_t s0 = take(2 * M * P->max_state);
    take(2 * M * P->max_state);
    // split-K scratch (zero at rest): a step splits K only below 74 output tiles of 128 x 64
    take(4 * std::min<int64_t>(M * std::max<int64_t>(P->max_state, std::max(P->rows, P->r_pad)), 74 * 128 * 64));
    if (o_s) *o_s = s0;
  }
  return bytes;
}

static int pick_bn(int64_t n) {
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  return 256;
}

// one tensor-core GEMM step, either orientation.
//   normal : out[m][n] = sum_k X[m][k] W[n][k]   (X: tokens, M-side)
//   swapped: same result, W on the M side (tokens on N) -> split-K fp32 atomics
//            when out_f32 != nullptr, else direct bf16 store.
static tnl_status tc_step(tnl_plan* P, const void* X, int64_t ldx, const void* W, int64_t ldw,
                          int64_t M, int64_t N, int64_t K, void* out, int64_t ldo, bool out_f32,
                          bool swapped, int splits, cudaStream_t st) {
  int err = 0;
  CUtensorMap ta, tb;
  TcGemmArgs a;
  a.K = (int32_t)K;
  const int total_kb = (int)((K + 63) / 64);
  if (!swapped) {
    const int bn = pick_bn(N);
    if ((err = get_tmap(P, &ta, X, K, M, ldx, 128)))
      return fail(TNL_ERR_CUDA, "tensor map (activations) failed: %d", err);
    if ((err = get_tmap(P, &tb, W, K, N, ldw, bn)))
      return fail(TNL_ERR_CUDA, "tensor map (weights) failed: %d", err);
    a.M = (int32_t)M;
    a.N = (int32_t)N;
    a.kb_per_split = (total_kb + splits - 1) / splits;
    splits = (total_kb + a.kb_per_split - 1) / a.kb_per_split;
    a.out = out;
    a.ldo_i = ldo;
    a.ldo_j = 1;
    a.out_mode = out_f32 ? (splits > 1 ? TC_OUT_F32_ATOMIC : TC_OUT_F32) : TC_OUT_BF16;
    err = launch_tc_gemm(ta, tb, a, bn, splits, true, st);
  } else {
    const int bn = pick_bn(M);
    if ((err = get_tmap(P, &ta, W, K, N, ldw, 128)))
      return fail(TNL_ERR_CUDA, "tensor map (weights) failed: %d", err);
    if ((err = get_tmap(P, &tb, X, K, M, ldx, bn)))
      return fail(TNL_ERR_CUDA, "tensor map (activations) failed: %d", err);
    a.M = (int32_t)N;
    a.N = (int32_t)M;
    a.kb_per_split = (total_kb + splits - 1) / splits;
    splits = (total_kb + a.kb_per_split - 1) / a.kb_per_split;
    a.out = out;
    a.ldo_i = 1;
    a.ldo_j = ldo;
    a.out_mode = out_f32 ? (splits > 1 ? TC_OUT_F32_ATOMIC : TC_OUT_F32) : TC_OUT_BF16;
    err = launch_tc_gemm(ta, tb, a, bn, splits, true, st);
  }
  if (err) return fail(TNL_ERR_CUDA, "tc_gemm launch failed: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

// split count so that m_tiles * n_tiles * splits ~ one wave of 148 SMs
static int choose_splits(int64_t tiles, int64_t K) {
  const int64_t total_kb = (K + 63) / 64;
  int64_t s = std::max<int64_t>(1, 148 / std::max<int64_t>(tiles, 1));
  return (int)std::min<int64_t>(s, total_kb);
}

// TT/TR input chain kernel: T[m][kappa] at out (strides s_m, s_k), bf16 or fp32 reductions.
static tnl_status chain_in(tnl_plan* P, const void* x, int64_t ldx, int64_t M, void* out, int64_t s_m,
                           int64_t s_k, bool f32_atomic, int splits, cudaStream_t st) {
  CUtensorMap tx, td, tcm;
  int err;
  const int n1 = P->ch_r0 * P->ch_cpad;
  if ((err = get_tmap2(P, &tx, x, false, P->cols, M, ldx, 16, 128, 32)) ||
      (err = get_tmap2(P, &td, P->chain_d, false, P->ch_nb, n1, P->ch_nb, 16, n1, 32)) ||
      (err = get_tmap2(P, &tcm, P->chain_c, false, P->ch_cpad, (int64_t)P->ch_na * P->ch_bpad, P->ch_cpad,
                       P->ch_cpad, P->ch_bpad, 2 * P->ch_cpad)))
    return fail(TNL_ERR_CUDA, "tensor map (chain) failed: %d", err);
  ChainArgs a;
  memset(&a, 0, sizeof a);
  a.M = (int32_t)M;
  a.n_a = P->ch_na;
  a.n_b = P->ch_nb;
  a.r0 = P->ch_r0;
  a.c = P->ch_c;
  a.c_pad = P->ch_cpad;
  a.b = P->ch_b;
  a.b_pad = P->ch_bpad;
  a.ja_per_split = (P->ch_na + splits - 1) / splits;
  splits = (P->ch_na + a.ja_per_split - 1) / a.ja_per_split;
  a.out = out;
  a.s_m = s_m;
  a.s_k = s_k;
  a.out_f32_atomic = f32_atomic ? 1 : 0;
  if ((err = launch_chain_in2(tx, td, tcm, a, splits, st)))
    return fail(TNL_ERR_CUDA, "chain kernel launch: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

static constexpr int64_t kDecMaxM = 64;  // decode path (plan-owned accumulator capacity)


// Small-M path of the merged-cut plan: phase A (B_in, split-K, fp32 reductions into the
// plan-owned accumulator) + phase B (A_out, reads the fp32 accumulator, re-zeroes it).
static tnl_status forward_decode(tnl_plan* P, const void* x, int64_t M, int64_t ldx, void* y,
                                 int64_t ldy, void* ws, cudaStream_t st) {
  // decode accumulator (64 x r_pad fp32, zero at rest) and counter live at the workspace head
  float* tacc = static_cast<float*>(ws);
  unsigned int* counter = reinterpret_cast<unsigned int*>(static_cast<char*>(ws) + kDecHeadBytes);
  const int64_t rows_local = P->row_end - P->row_begin;
  int err = 0;
  const bool use_chain = P->plan_large == TNL_PLAN_CHAIN && P->chain_ok;
  if (M <= 8 && !use_chain && (P->flags & TNL_PLAN_GEMV)) {
    // CUDA-core GEMV variant; T goes to the (non-accumulating) scratch after the accumulator
    float* t = reinterpret_cast<float*>(static_cast<char*>(ws) + kDecHeadBytes + 256);
    err = launch_gemv_a(P->bin, P->cols, (int)P->r_pad, (int)P->cols, static_cast<const __nv_bfloat16*>(x), ldx,
                        (int)M, t, P->r_pad, st);
    if (err) return fail(TNL_ERR_CUDA, "gemv_a launch: %s", cudaGetErrorString((cudaError_t)err));
    err = launch_gemv_b(P->aout, P->r_pad, (int)rows_local, (int)P->r_pad, t, P->r_pad, (int)M,
                        static_cast<__nv_bfloat16*>(y), ldy, st);
    if (err) return fail(TNL_ERR_CUDA, "gemv_b launch: %s", cudaGetErrorString((cudaError_t)err));
    return TNL_OK;
  }
  CUtensorMap tw, tx, tw2, tt, ty;
  const int bn = pick_bn(M);
  const int64_t ldk = kDecMaxM;  // kappa-major accumulator row pitch (tokens)
  if ((err = get_tmap(P, &tw, P->bin, P->cols, P->r_pad, P->cols, 128)) ||
      (err = get_tmap(P, &tx, x, P->cols, M, ldx, bn)) ||
      (err = get_tmap(P, &tw2, P->aout, P->r_pad, rows_local, P->r_pad, 128)))
    return fail(TNL_ERR_CUDA, "tensor map (decode) failed: %d", err);
  if ((err = get_tmap2(P, &tt, tacc, true, ldk, P->r_pad, ldk, bn, 64, 0)) ||
      (err = get_tmap2(P, &ty, y, false, rows_local, M, ldy, 128, bn, 0)))
    return fail(TNL_ERR_CUDA, "tensor map (decode accumulator / y) failed: %d", err);
  DecArgs a;
  memset(&a, 0, sizeof a);
  a.M_rows = (int32_t)P->r_pad;
  a.tokens = (int32_t)M;
  a.K = (int32_t)P->cols;
  const int total_kb = (int)((P->cols + 63) / 64);
  // K blocks per split: fewer partials -> less reduction traffic to drain before phase B
  static const int kb_env = [] {
    const char* e = getenv("TNL_DEC_KB");
    return e ? atoi(e) : 0;
  }();
  a.kb_per_split = kb_env > 0 ? kb_env : 4;
  int splits = (total_kb + a.kb_per_split - 1) / a.kb_per_split;
  a.out = tacc;
  a.ldo_i = ldk;
  a.ldo_j = 1;
  a.out_f32_atomic = 1;
  a.trace = P->trace;
  if (use_chain) {
    // core-by-core input chain, j_a split across CTAs, fp32 reductions into the accumulator
    tnl_status cs = chain_in(P, x, ldx, M, tacc, 1, ldk, true, std::min(16, P->ch_na), st);
    if (cs) return cs;
  } else if ((err = launch_dec_a(tw, tx, a, splits, st))) {
    return fail(TNL_ERR_CUDA, "decode phase A launch: %s", cudaGetErrorString((cudaError_t)err));
  }
  DecArgs b;
  memset(&b, 0, sizeof b);
  b.M_rows = (int32_t)rows_local;
  b.tokens = (int32_t)M;
  b.K = (int32_t)P->r_pad;
  b.kb_per_split = (int32_t)((P->r_pad + 63) / 64);
  b.act_f32 = tacc;
  b.act_ld = ldk;
  b.out = y;
  b.ldo_i = 1;
  b.ldo_j = ldy;
  b.out_f32_atomic = 0;
  b.counter = counter;
  b.zero_elems = P->r_pad * ldk;
  b.trace = P->trace ? P->trace + 16 * 1024 : nullptr;
  if ((err = launch_dec_b(tw2, tt, ty, b, st)))
    return fail(TNL_ERR_CUDA, "decode phase B launch: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

// Large-M GEMM step on the persistent kernel: out (M x N) = X (M x K) . W (N x K)^T.
// out_f32: fp32 split-K reductions into `out` (zeroed here); else bf16 via TMA store.
static tnl_status tc_step_p(tnl_plan* P, const void* X, int64_t ldx, const void* W, int64_t ldw,
                            int64_t M, int64_t N, int64_t K, void* out, int64_t ldo, bool out_f32,
                            int splits, cudaStream_t st, int bn_force = 0, const tnl_fwd_opts* in_o = nullptr,
                            const tnl_fwd_opts* out_o = nullptr) {
  const int bn = bn_force ? bn_force : (N <= 64 ? 64 : (N <= 128 ? 128 : 256));
  CUtensorMap ta, tb, tc;
  int err;
  if ((err = get_tmap(P, &ta, X, K, M, ldx, 128)) || (err = get_tmap(P, &tb, W, K, N, ldw, bn)))
    return fail(TNL_ERR_CUDA, "tensor map (persistent step) failed: %d", err);
  TcGemmArgs a;
  memset(&a, 0, sizeof a);
  a.M = (int32_t)M;
  a.N = (int32_t)N;
  a.K = (int32_t)K;
  const int total_kb = (int)((K + 63) / 64);
  a.kb_per_split = (total_kb + splits - 1) / splits;
  splits = (total_kb + a.kb_per_split - 1) / a.kb_per_split;
  a.out = out;
  a.ldo_i = ldo;
  a.ldo_j = 1;
  if (out_f32) {
    a.out_mode = TC_OUT_F32_ATOMIC;
    if (cudaMemsetAsync(out, 0, sizeof(float) * M * ldo, st) != cudaSuccess)
      return fail(TNL_ERR_CUDA, "memset failed");
    tc = ta;  // unused
  } else {
    a.out_mode = TC_OUT_BF16;
    if ((err = get_tmap2(P, &tc, out, false, N, M, ldo, 64, 128, 128)))
      return fail(TNL_ERR_CUDA, "tensor map (output) failed: %d", err);
    if (in_o && (in_o->ss_in || in_o->rms_fused)) {  // folded RMSNorm of X: scale the output rows
      a.ss_in = in_o->ss_in;
      a.ss_fused = (in_o->rms_fused && splits == 1) ? 1 : 0;  // statistics from the streamed A tiles
      a.rms_n = in_o->rms_n;
      a.rms_eps = in_o->rms_eps;
    }
    if (out_o && out_o->accumulate) a.reduce_add = 1;  // out += D (TMA reduce-add)
  }
  // CTA pairs (M=256 MMAs, each CTA streams half of the weight tile) once there are two token
  // tiles and a wide enough weight tile; TNL_PAIR_GEMM=0 disables
  static const bool pair_env = !(getenv("TNL_PAIR_GEMM") && atoi(getenv("TNL_PAIR_GEMM")) == 0);
  // 128-wide weight tiles (the N-split halves of the rank-256 first steps) too: half the weight
  // bytes per CTA, a 7-deep ring (q 66.7 -> 64.0 us, o 70.4 -> 66.2 us; TNL_PAIR128=0 disables)
  static const bool pair128_env = !(getenv("TNL_PAIR128") && atoi(getenv("TNL_PAIR128")) == 0);
  if (pair_env && M >= 256 && (bn == 256 || (pair128_env && bn == 128 && !out_f32))) {
    CUtensorMap tbh;
    if ((err = get_tmap(P, &tbh, W, K, N, ldw, bn / 2)))
      return fail(TNL_ERR_CUDA, "tensor map (pair step) failed: %d", err);
    err = launch_tc_gemm_pair(ta, tbh, tc, a, bn, splits, st);
  } else {
    err = launch_tc_gemm_persistent(ta, tb, tc, a, bn, splits, 148, true, st);
  }
  if (err) return fail(TNL_ERR_CUDA, "persistent gemm launch: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

static bool no_splitk2() {  // A/B switch (TNL_SPLITK2=0: fp32 split-K + conversion instead)
  static const bool v = getenv("TNL_SPLITK2") && atoi(getenv("TNL_SPLITK2")) == 0;
  return v;
}

// TNL_PLAN_CHAIN in bf16 for the shapes without a fused chain kernel: the GENERIC core-by-core step
// list (cores in their permuted layouts, ring closure carried as a batch index) with bf16 cores and
// bf16 intermediates, every step on the tensor cores (tc_generic.cu). tcg_out plans run the input
// side in the two-mode chain kernel (intermediates on chip) and only the output cores as steps.
static tnl_status forward_tcg(tnl_plan* P, const void* x, int64_t M, int64_t ldx, void* y, int64_t ldy, void* ws,
                              size_t ws_bytes, cudaStream_t st) {
  size_t o_f32, o_b0, o_b1, o_s = 0;
  const size_t need = ws_layout(P, M, &o_f32, &o_b0, &o_b1, &o_s);
  if (ws_bytes < need) return fail(TNL_ERR_ARG, "workspace %zu < required %zu bytes", ws_bytes, need);
  char* w = static_cast<char*>(ws);
  ChainIO io;
  io.ws[0] = reinterpret_cast<float*>(w + o_s);  // bf16 states (the step builder only passes them on)
  io.ws[1] = reinterpret_cast<float*>(w + o_s + round_up(2 * M * P->max_state, 256));
  float* acc32 = reinterpret_cast<float*>(w + o_s + 2 * round_up(2 * M * P->max_state, 256));
  io.out = {y, DT_BF16, ldy, 1};
  int seg = SEG_FULL;
  if (P->tcg_out) {
    __nv_bfloat16* t0 = reinterpret_cast<__nv_bfloat16*>(w + o_b0);
    float* tf = reinterpret_cast<float*>(w + o_f32);
    const int64_t tiles_m = (M + 127) / 128;
    const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(P->ch_na / 4, 148 / tiles_m));
    tnl_status cs;
    if (splits > 1) {
      if (cudaMemsetAsync(tf, 0, sizeof(float) * M * P->r_pad, st) != cudaSuccess)
        return fail(TNL_ERR_CUDA, "memset failed");
      cs = chain_in(P, x, ldx, M, tf, P->r_pad, 1, true, splits, st);
      if (cs) return cs;
      to_bf16(tf, t0, M * P->r_pad, st);
    } else {
      cs = chain_in(P, x, ldx, M, t0, P->r_pad, 1, false, 1, st);
      if (cs) return cs;
    }
    io.in = {t0, DT_BF16, P->r_pad, 1};
    seg = SEG_OUTPUT;
  } else {
    io.in = {x, DT_BF16, ldx, 1};
  }
  std::vector<GStep> steps;
  build_steps(P, seg, M, io, steps);
  auto is_state = [&](const void* p) { return p == io.ws[0] || p == io.ws[1]; };
  for (GStep g : steps) {
    auto to16 = [&](const void*& p, int32_t& dt) {
      if (is_state(p)) dt = DT_BF16;
      for (size_t k = 0; k < P->gcore.size(); ++k)
        if (p == P->gcore[k]) {
          p = P->gcore16[k];
          dt = DT_BF16;
        }
    };
    to16(g.A, g.a_dt);
    to16(g.B, g.b_dt);
    if (is_state(g.C)) g.c_dt = DT_BF16;
    TcgArgs t;
    if (!tcg_from_gstep(g, &t)) return fail(TNL_ERR_UNSUPPORTED, "bf16 chain: step not expressible on the tensor cores");
    t.acc32 = acc32;
    const int err = launch_tc_generic(t, st);
    if (err) return fail(TNL_ERR_CUDA, "bf16 chain step launch: %s", cudaGetErrorString((cudaError_t)err));
  }
  return TNL_OK;
}

static tnl_status forward_tc(tnl_plan* P, const void* x, int64_t M, int64_t ldx, void* y, int64_t ldy,
                             void* ws, size_t ws_bytes, cudaStream_t st, const tnl_fwd_opts* o = nullptr) {
  const bool fold = o && (o->accumulate || o->ss_in);
  size_t o_f32, o_b0, o_b1;
  size_t need = ws_layout(P, M, &o_f32, &o_b0, &o_b1);
  if (ws_bytes < need) return fail(TNL_ERR_ARG, "workspace %zu < required %zu bytes", ws_bytes, need);
  char* w = static_cast<char*>(ws);
  float* tf = reinterpret_cast<float*>(w + o_f32);
  __nv_bfloat16* t0 = reinterpret_cast<__nv_bfloat16*>(w + o_b0);
  __nv_bfloat16* t1 = reinterpret_cast<__nv_bfloat16*>(w + o_b1);
  const int64_t rows_local = P->row_end - P->row_begin;
  const bool swap = M <= kSwapMaxM;
  if (fold && (M <= kSwapMaxM || P->family == TNL_FAMILY_DENSE || P->plan_large == TNL_PLAN_CHAIN ||
               (reinterpret_cast<uintptr_t>(y) & 15) || ldy % 8 || (P->r_pad % 8)))
    return fail(TNL_ERR_UNSUPPORTED, "folded residual / RMSNorm: prefill (M > %lld) cut plans only", (long long)kSwapMaxM);
  if (P->tcg_out || P->tcg_full) return forward_tcg(P, x, M, ldx, y, ldy, ws, ws_bytes, st);
  if (M <= kDecMaxM && P->decode_max_m && !(reinterpret_cast<uintptr_t>(y) & 15) && ldy % 8 == 0)
    return forward_decode(P, x, M, ldx, y, ldy, ws, st);
  tnl_status s;
  if (P->family == TNL_FAMILY_DENSE) {
    if (!swap && !(reinterpret_cast<uintptr_t>(y) & 15) && ldy % 8 == 0)
      return tc_step_p(P, x, ldx, P->wdense, P->cols, M, rows_local, P->cols, y, ldy, false, 1, st);
    return tc_step(P, x, ldx, P->wdense, P->cols, M, rows_local, P->cols, y, ldy, false, swap, 1, st);
  }
  // first step: T = X . Win^T  (Win = B_in or U1^T), K = cols
  if (P->plan_large == TNL_PLAN_CHAIN && P->chain_ok && !swap &&
      !(reinterpret_cast<uintptr_t>(y) & 15) && ldy % 8 == 0) {
    // TT/TR core-by-core input chain -> T (bf16, or fp32 reductions when j_a is split), then
    // the output panel GEMM. K of step 2 = r_cut (TMA zero-fills the padded columns).
    const int64_t tiles_m = (M + 127) / 128;
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>(P->ch_na / 4, 148 / tiles_m));
    if (splits > 1) {
      if (cudaMemsetAsync(tf, 0, sizeof(float) * M * P->r_pad, st) != cudaSuccess)
        return fail(TNL_ERR_CUDA, "memset failed");
      s = chain_in(P, x, ldx, M, tf, P->r_pad, 1, true, splits, st);
      if (s) return s;
      to_bf16(tf, t0, M * P->r_pad, st);
    } else {
      s = chain_in(P, x, ldx, M, t0, P->r_pad, 1, false, 1, st);
      if (s) return s;
    }
    return tc_step_p(P, t0, P->r_pad, P->aout, P->r_pad, M, rows_local, P->r_cut, y, ldy, false, 1, st);
  }
  // Tucker-2 chain plan, prefill: the fused on-chip chain (tucker_chain.cu) — U1, G and U0 in one
  // kernel, T1/T2 in TMEM/smem, a 2-CTA cluster per token tile
  static const bool no_fused_tucker = getenv("TNL_TUCKER_FUSED") && atoi(getenv("TNL_TUCKER_FUSED")) == 0;  // A/B
  if (P->tucker_chain && !swap && !fold && !no_fused_tucker && tucker2_chain_ok((int)P->r1p, (int)P->r0p) &&
      !(reinterpret_cast<uintptr_t>(y) & 15) && ldy % 8 == 0) {
    const int64_t r1h = P->r1p % 128 == 0 ? P->r1p / 2 : P->r1p;
    CUtensorMap tx, tu1, tg, tu0, ty;
    int err;
    if ((err = get_tmap(P, &tx, x, P->cols, M, ldx, 128)) || (err = get_tmap(P, &tu1, P->u1t, P->cols, P->r1p, P->cols, (int)r1h)) ||
        (err = get_tmap(P, &tg, P->gmat, P->r1p, P->r0p, P->r1p, (int)P->r0p)) ||
        (err = get_tmap(P, &tu0, P->u0, P->r0p, rows_local, P->r0p, 256)) ||
        (err = get_tmap2(P, &ty, y, false, rows_local, M, ldy, 64, 128, 128)))
      return fail(TNL_ERR_CUDA, "tensor map (fused Tucker-2 chain) failed: %d", err);
    if ((err = launch_tucker2_chain(tx, tu1, tg, tu0, ty, (int)M, (int)rows_local, (int)P->cols, (int)P->r1p,
                                    (int)P->r0p, st)))
      return fail(TNL_ERR_CUDA, "fused Tucker-2 chain launch: %s", cudaGetErrorString((cudaError_t)err));
    return TNL_OK;
  }
  const __nv_bfloat16* win = P->tucker_chain ? P->u1t : P->bin;
  const int64_t k1 = P->tucker_chain ? P->r1p : P->r_pad;
  const __nv_bfloat16* wout = P->tucker_chain ? P->u0 : P->aout;
  const bool y_tma_ok = !(reinterpret_cast<uintptr_t>(y) & 15) && ldy % 8 == 0;
  if (!swap && y_tma_ok) {
    // prefill: persistent steps. Step 1 has few output tiles (N = r_pad): split K so
    // the grid covers the SMs, reducing in fp32, then round T to bf16 once.
    const int64_t tiles1 = ((M + 127) / 128) * ((k1 + 255) / 256);
    const int64_t kb1 = (P->cols + 63) / 64;
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>(148 / std::max<int64_t>(tiles1, 1), kb1 / 8));
    static const bool no_nsplit = getenv("TNL_STEP1_NSPLIT") && atoi(getenv("TNL_STEP1_NSPLIT")) == 0;  // A/B
    if (!no_nsplit && splits > 1 && k1 >= 128 && k1 % 128 == 0 && ((M + 127) / 128) * 2 >= 96 && P->cols <= 12288) {
      // split the cut dimension instead of K: two half-width tiles per token tile, full K each ->
      // no fp32 partials, no memset, no conversion pass (Tucker-2 R256 at M=8192: q 73.5 -> 66.2 us,
      // o 73.8 -> 70.1 us). A long K (down, 25600) keeps the CTA-pair split-K: 84.6 vs 103 us.
      s = tc_step_p(P, x, ldx, win, P->cols, M, k1, P->cols, t0, k1, false, 1, st, (int)(k1 / 2), o, nullptr);
      if (s) return s;
    } else if (splits == 2 && k1 <= 64 && !(o && o->ss_in) && !no_splitk2()) {
      // two K halves over a CTA pair, partial exchanged through DSMEM: bf16 T straight out
      CUtensorMap ta, tb;
      int err;
      if ((err = get_tmap(P, &ta, x, P->cols, M, ldx, 128)) || (err = get_tmap(P, &tb, win, P->cols, k1, P->cols, 64)))
        return fail(TNL_ERR_CUDA, "tensor map (split-K pair step) failed: %d", err);
      if ((err = launch_tc_gemm_splitk2(ta, tb, t0, k1, (int)M, (int)k1, (int)P->cols, st)))
        return fail(TNL_ERR_CUDA, "split-K pair launch: %s", cudaGetErrorString((cudaError_t)err));
    } else if (splits > 1) {
      s = tc_step_p(P, x, ldx, win, P->cols, M, k1, P->cols, tf, k1, true, splits, st);
      if (s) return s;
      if (o && o->ss_in)
        to_bf16_scaled(tf, t0, M, k1, o, st);
      else
        to_bf16(tf, t0, M * k1, st);
    } else {
      s = tc_step_p(P, x, ldx, win, P->cols, M, k1, P->cols, t0, k1, false, 1, st, 0, o, nullptr);
      if (s) return s;
    }
    const __nv_bfloat16* tcur = t0;
    int64_t kc = k1;
    if (P->tucker_chain) {  // T2 = T1 . G^T
      s = tc_step_p(P, t0, k1, P->gmat, P->r1p, M, P->r0p, P->r1p, t1, P->r0p, false, 1, st);
      if (s) return s;
      tcur = t1;
      kc = P->r0p;
    }
    return tc_step_p(P, tcur, kc, wout, kc, M, rows_local, kc, y, ldy, false, 1, st, 0, nullptr, o);
  }
  if (fold) return fail(TNL_ERR_UNSUPPORTED, "folded residual / RMSNorm: needs the persistent prefill path");
  // first step: T = X . Win^T  (Win = B_in or U1^T), K = cols
  if (swap) {
    const int64_t tiles = (k1 + 127) / 128;
    const int splits = choose_splits(tiles, P->cols);
    if (splits > 1) {
      if (cudaMemsetAsync(tf, 0, sizeof(float) * M * k1, st) != cudaSuccess)
        return fail(TNL_ERR_CUDA, "memset failed");
      s = tc_step(P, x, ldx, win, P->cols, M, k1, P->cols, tf, k1, true, true, splits, st);
      if (s) return s;
      to_bf16(tf, t0, M * k1, st);
    } else {
      s = tc_step(P, x, ldx, win, P->cols, M, k1, P->cols, t0, k1, false, true, 1, st);
      if (s) return s;
    }
  } else {
    s = tc_step(P, x, ldx, win, P->cols, M, k1, P->cols, t0, k1, false, false, 1, st);
    if (s) return s;
  }
  const __nv_bfloat16* tcur = t0;
  int64_t kc = k1;
  if (P->tucker_chain) {  // T2 = T1 . G^T   (R0p x R1p)
    s = tc_step(P, t0, k1, P->gmat, P->r1p, M, P->r0p, P->r1p, t1, P->r0p, false, swap, 1, st);
    if (s) return s;
    tcur = t1;
    kc = P->r0p;
  }
  return tc_step(P, tcur, kc, wout, kc, M, rows_local, kc, y, ldy, false, swap, 1, st);
}

static tnl_status forward_generic(tnl_plan* P, const void* x, int64_t M, int64_t ldx, void* y,
                                  int64_t ldy, void* ws, size_t ws_bytes, cudaStream_t st) {
  size_t o_f32, o_b0, o_b1;
  size_t need = ws_layout(P, M, &o_f32, &o_b0, &o_b1);
  if (ws_bytes < need) return fail(TNL_ERR_ARG, "workspace %zu < required %zu bytes", ws_bytes, need);
  char* w = static_cast<char*>(ws);
  const int dt = P->compute_dtype == TNL_BF16 ? DT_BF16 : DT_F32;
  if (P->bin32 && M <= 32 && P->r_cut <= kDec32MaxCut && !(P->flags & TNL_PLAN_NO_DECODE)) {
    // small M: the two fp32 decode phases (dec32.cu), accumulator + counter at the workspace head
    float* tacc = reinterpret_cast<float*>(w);
    unsigned int* counter = reinterpret_cast<unsigned int*>(w + kDecHeadBytes);
    const int err = launch_dec32(P->bin32, P->cols, P->aout32, P->r_cut, (int)(P->row_end - P->row_begin),
                                 (int)P->r_cut, (int)P->cols, static_cast<const float*>(x), ldx, (int)M,
                                 static_cast<float*>(y), ldy, tacc, counter, st);
    if (err) return fail(TNL_ERR_CUDA, "fp32 decode launch: %s", cudaGetErrorString((cudaError_t)err));
    return TNL_OK;
  }
  if (P->bin32) {
    // fp32 merged cut: T[kappa][m] = sum_j B_in[kappa][j] x[m][j] (split-K FFMA, fp32 atomics),
    // then y[m][i] = sum_kappa A_out[i][kappa] T[kappa][m]
    float* t = reinterpret_cast<float*>(w + o_f32);
    const int64_t rl = P->row_end - P->row_begin;
    GStep a = mk(1, 1, P->r_cut, P->cols, M);
    a.A = P->bin32;
    a.sai = P->cols;
    a.sap = 1;
    a.B = x;
    a.b_dt = dt;
    a.sbp = 1;
    a.sbj = ldx;
    a.C = t;
    a.sci = M;
    a.scj = 1;
    GStep b = mk(1, 1, rl, P->r_cut, M);
    b.A = P->aout32;
    b.sai = P->r_cut;
    b.sap = 1;
    b.B = t;
    b.sbp = M;
    b.sbj = 1;
    b.C = y;
    b.c_dt = dt;
    b.sci = 1;
    b.scj = ldy;
    if (launch_generic_step(a, st) || launch_generic_step(b, st))
      return fail(TNL_ERR_CUDA, "fp32 cut step launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return TNL_OK;
  }
  const int64_t rows_local = P->row_end - P->row_begin;
  ChainIO io;
  io.in = Operand{x, dt, ldx, 1};
  const bool sharded = rows_local != P->rows;
  float* ytmp = reinterpret_cast<float*>(w + o_f32);
  io.out = sharded ? Operand{ytmp, DT_F32, P->rows, 1} : Operand{y, dt, ldy, 1};
  io.ws[0] = reinterpret_cast<float*>(w + o_b0);
  io.ws[1] = reinterpret_cast<float*>(w + o_b1);
  std::vector<GStep> steps;
  build_steps(P, SEG_FULL, M, io, steps);
  if (run_steps(steps, st)) return fail(TNL_ERR_CUDA, "generic step launch failed: %s",
                                        cudaGetErrorString(cudaGetLastError()));
  if (sharded) {
    copy_2d_any<<<grid_for(M * rows_local), 256, 0, st>>>(ytmp + P->row_begin, DT_F32, P->rows, 1,
                                                          y, dt, ldy, 1, M, rows_local);
    count_launch();
  }
  return TNL_OK;
}


// ---------------------------------------------------------------------------
// Decode stacks: one fused kernel per layer boundary (decode_fused.cu)
// ---------------------------------------------------------------------------
static bool stack_fusable(const tnl_plan* const* plans, int32_t n, int64_t m) {
  if (n < 2 || m < 1 || m > kDecMaxM) return false;
  for (int i = 0; i < n; ++i) {
    const tnl_plan* P = plans[i];
    if (!P || !P->decode_max_m || P->plan_large != TNL_PLAN_CUT || P->compute_dtype != TNL_BF16 ||
        P->row_begin != 0 || P->row_end != P->rows)
      return false;
    if (i + 1 < n && (P->rows != plans[i + 1]->cols || P->rows % 128)) return false;
  }
  return true;
}

static size_t stack_ws_bytes(const tnl_plan* const* plans, int32_t n, int64_t m) {
  if (stack_fusable(plans, n, m)) return kDecSlots * kDecSlotBytes;
  size_t mx = 0;
  int64_t width = 0;
  for (int i = 0; i < n; ++i) {
    size_t a, b, c;
    mx = std::max(mx, ws_layout(plans[i], std::max<int64_t>(m, 1), &a, &b, &c));
    width = std::max(width, plans[i]->row_end - plans[i]->row_begin);
  }
  return mx + 2 * round_up(2 * m * width, 256);
}

}  // namespace tnl (stack helpers)
namespace tnl {

// ---------------------------------------------------------------------------
// Fused TN MLP block: y = down(silu(gate(x)) * up(x))  (mlp.cu)
// ---------------------------------------------------------------------------
}  // namespace tnl

struct tnl_mlp {
  tnl_plan* g = nullptr;
  tnl_plan* u = nullptr;
  tnl_plan* d = nullptr;
  bool fused = false;
  bool dual = false;  // gate/up output GEMMs + SiLU*mul in one kernel (ranks the fused path cannot hold)
  int64_t hidden = 0, inter = 0, rg = 0, ru = 0, rd = 0;
  __nv_bfloat16* bgu = nullptr;  // [B_g (rg rows) ; B_u (ru rows)] x hidden
  // decode gated boundary (rg + ru <= 256): A_gu = [A_g | A_u] (inter x (rg + ru)); one phase A
  // of the stacked [B_g; B_u], then ONE kernel does gate/up phase B, SiLU*mul and down's phase A
  bool gated = false;
  __nv_bfloat16* agu = nullptr;
  // decode: up runs on a forked stream (workspace slot 1) concurrently with gate (slot 0)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::mutex fork_mu;  // the fork/join section reuses the events: one caller at a time
};

namespace tnl {

// T_gu = x . [B_g; B_u]^T (M x (rg + ru) bf16): the concatenated cut activation of gate and up
static tnl_status mlp_tgu(tnl_mlp* B, const void* x, int64_t m, int64_t ldx, float* tgu32, __nv_bfloat16* tgu,
                          cudaStream_t st, const tnl_fwd_opts* in_o = nullptr) {
  const int64_t rgu = B->rg + B->ru;
  const int64_t tiles1 = ((m + 127) / 128) * ((rgu + 255) / 256);
  const int64_t kb = (B->hidden + 63) / 64;
  const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(148 / std::max<int64_t>(tiles1, 1), kb / 8));
  tnl_status s;
  const bool one_pass = rgu <= 128 && ((m + 127) / 128) * ((rgu + 63) / 64) >= 96;
  if (in_o && in_o->rms_fused && !one_pass && splits > 1)
    return fail(TNL_ERR_UNSUPPORTED, "rms_fused: the gate/up input step splits K at M = %lld", (long long)m);
  if (one_pass) {
    // enough 64-wide output tiles to fill the SMs: no split-K, bf16 straight from the epilogue
    return tc_step_p(B->g, x, ldx, B->bgu, B->hidden, m, rgu, B->hidden, tgu, rgu, false, 1, st, 64, in_o);
  }
  if (splits > 1) {
    if ((s = tc_step_p(B->g, x, ldx, B->bgu, B->hidden, m, rgu, B->hidden, tgu32, rgu, true, splits, st))) return s;
    if (in_o && in_o->ss_in)
      to_bf16_scaled(tgu32, tgu, m, rgu, in_o, st);
    else
      to_bf16(tgu32, tgu, m * rgu, st);
    return TNL_OK;
  }
  return tc_step_p(B->g, x, ldx, B->bgu, B->hidden, m, rgu, B->hidden, tgu, rgu, false, 1, st, 0, in_o);
}

static void mlp_ws_layout(const tnl_mlp* B, int64_t M, size_t off[4], size_t* total) {
  size_t bytes = 0;
  auto take = [&](size_t n) {
    size_t o = bytes;
    bytes += round_up((int64_t)n, 256);
    return o;
  };
  // every layout keeps the decode head (zero-at-rest accumulators of the three layers' decode
  // calls, and of any other plan sharing the workspace) untouched
  if (B->fused && M > kSwapMaxM) {
    take(kDecSlots * kDecSlotBytes);
    off[0] = take(sizeof(float) * M * (B->rg + B->ru));  // T_gu fp32 (split-K)
    off[1] = take(2 * M * (B->rg + B->ru));              // T_gu bf16
    off[2] = take(sizeof(float) * M * B->rd);            // T_d fp32 (slice reductions)
    off[3] = take(2 * M * B->rd);                        // T_d bf16
  } else if (B->dual && M > kSwapMaxM) {
    size_t a, b, c;
    off[0] = take(ws_layout(B->d, M, &a, &b, &c));       // down's layer workspace
    off[1] = take(sizeof(float) * M * (B->rg + B->ru));  // T_gu fp32 (split-K)
    off[2] = take(2 * M * (B->rg + B->ru));              // T_gu bf16
    off[3] = take(2 * M * B->inter);                     // h
  } else {
    size_t a, b, c, mx = 0;
    for (const tnl_plan* P : {B->g, B->u, B->d}) mx = std::max(mx, ws_layout(P, M, &a, &b, &c));
    off[0] = take(mx);                  // per-layer workspace (zero-filled: decode accumulators)
    off[1] = take(2 * M * B->inter);    // g / h
    off[2] = take(2 * M * B->inter);    // u
    off[3] = 0;
  }
  *total = bytes;
}

}  // namespace tnl

using namespace tnl;

extern "C" {

int tnl_abi_version(void) { return TNL_ABI_VERSION; }
const char* tnl_last_error(void) { return g_err.c_str(); }
int64_t tnl_launch_count(int32_t reset) { return launch_count(reset != 0); }

tnl_status tnl_stack_workspace_size(const tnl_plan* const* plans, int32_t n, int64_t m, size_t* bytes) {
  if (!plans || n < 1 || !bytes) return fail(TNL_ERR_ARG, "null argument");
  for (int i = 0; i < n; ++i)
    if (!plans[i]) return fail(TNL_ERR_ARG, "null plan %d", i);
  *bytes = stack_ws_bytes(plans, n, m);
  return TNL_OK;
}

static tnl_status stack_forward_impl(const tnl_plan* const* plans, int32_t n, const void* x, int64_t m, int64_t ldx,
                                     void* y, int64_t ldy, void* ws, size_t ws_bytes, void* stream, bool host_io);

tnl_status tnl_stack_forward(const tnl_plan* const* plans, int32_t n, const void* x, int64_t m,
                             int64_t ldx, void* y, int64_t ldy, void* ws, size_t ws_bytes, void* stream) {
  return stack_forward_impl(plans, n, x, m, ldx, y, ldy, ws, ws_bytes, stream, false);
}

tnl_status tnl_stack_forward_host(const tnl_plan* const* plans, int32_t n, const void* x_host, int64_t m, int64_t ldx,
                                  void* y_host, int64_t ldy, void* ws, size_t ws_bytes, void* stream) {
  for (const void* p : {x_host, static_cast<const void*>(y_host)}) {
    cudaPointerAttributes at;
    if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type == cudaMemoryTypeUnregistered ||
        at.type == cudaMemoryTypeDevice) {
      cudaGetLastError();
      return fail(TNL_ERR_ARG, "stack_forward_host: x and y must be pinned host buffers");
    }
  }
  return stack_forward_impl(plans, n, x_host, m, ldx, y_host, ldy, ws, ws_bytes, stream, true);
}

static tnl_status stack_forward_impl(const tnl_plan* const* plans, int32_t n, const void* x, int64_t m, int64_t ldx,
                                     void* y, int64_t ldy, void* ws, size_t ws_bytes, void* stream, bool host_io) {
  if (!plans || n < 1 || !x || !y) return fail(TNL_ERR_ARG, "null argument");
  for (int i = 0; i < n; ++i)
    if (!plans[i]) return fail(TNL_ERR_ARG, "null plan %d", i);
  for (int i = 0; i + 1 < n; ++i)
    if (plans[i]->row_end - plans[i]->row_begin != plans[i + 1]->cols)
      return fail(TNL_ERR_SHAPE, "stack link %d: %lld outputs feed %lld inputs", i,
                  (long long)(plans[i]->row_end - plans[i]->row_begin), (long long)plans[i + 1]->cols);
  if (m == 0) return TNL_OK;
  const size_t need = stack_ws_bytes(plans, n, m);
  if (ws_bytes < need) return fail(TNL_ERR_ARG, "stack workspace %zu < required %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tnl_plan* const* Pv = const_cast<tnl_plan* const*>(plans);
  if (host_io) {
    // The zero-copy loads read whole 64-column k-blocks of x (4 per CTA, register buffered) and
    // the stores write 8-row uint4 chunks of y: reject shapes those kernels would over-read or
    // over-write instead of bounds-checking the hot loop.
    const tnl_plan* P0 = plans[0];
    const tnl_plan* PL = plans[n - 1];
    const int64_t rows_l = PL->row_end - PL->row_begin;
    if (P0->cols % 64 || rows_l % 8 || ldx < P0->cols || ldy < rows_l)
      return fail(TNL_ERR_UNSUPPORTED,
                  "stack_forward_host: needs cols %% 64 == 0 (got %lld), rows %% 8 == 0 (got %lld), ldx >= cols, "
                  "ldy >= rows",
                  (long long)P0->cols, (long long)rows_l);
  }
  if (!stack_fusable(plans, n, m) || (reinterpret_cast<uintptr_t>(y) & 15) || ldy % 8 ||
      (reinterpret_cast<uintptr_t>(x) & 15) || ldx % 8) {
    if (host_io) return fail(TNL_ERR_UNSUPPORTED, "stack_forward_host: needs the fused decode stack (M <= 64)");
    // generic chain: per-layer forwards through two activation buffers in the workspace
    size_t layer_ws = 0;
    int64_t width = 0;
    for (int i = 0; i < n; ++i) {
      size_t a, b, c;
      layer_ws = std::max(layer_ws, ws_layout(plans[i], std::max<int64_t>(m, 1), &a, &b, &c));
      width = std::max(width, plans[i]->row_end - plans[i]->row_begin);
    }
    char* base = static_cast<char*>(ws);
    void* buf[2] = {base + layer_ws, base + layer_ws + round_up(2 * m * width, 256)};
    const void* cur = x;
    int64_t ldc = ldx;
    for (int i = 0; i < n; ++i) {
      const bool last = i + 1 == n;
      void* out = last ? y : buf[i & 1];
      const int64_t ldo = last ? ldy : width;
      tnl_status s = tnl_forward(plans[i], cur, m, ldc, out, ldo, ws, layer_ws, stream);
      if (s) return s;
      cur = out;
      ldc = ldo;
    }
    return TNL_OK;
  }
  char* base = static_cast<char*>(ws);
  // three rotating zero-at-rest accumulators: boundary l reads T_l = tacc[l % 3], reduces into
  // T_{l+1} = tacc[(l+1) % 3] and zeroes T_{l-1} = tacc[(l+2) % 3], which only boundary l-1 read.
  // They are the accumulators of the workspace's three decode slots (and the last phase B uses
  // slot 2's counter), so a stack can share a workspace with single-layer decode calls and MLP
  // blocks without ever overlapping their scratch.
  float* tacc[3] = {reinterpret_cast<float*>(base), reinterpret_cast<float*>(base + kDecSlotBytes),
                    reinterpret_cast<float*>(base + 2 * kDecSlotBytes)};
  unsigned int* cnt = reinterpret_cast<unsigned int*>(base + 2 * kDecSlotBytes + kDecHeadBytes);
  const int bn = pick_bn(m);
  int err = 0;
  // layer 0, phase A
  {
    tnl_plan* P = Pv[0];
    CUtensorMap tw, tx;
    if ((err = get_tmap(P, &tw, P->bin, P->cols, P->r_pad, P->cols, 128)) ||
        (err = host_io ? 0 : get_tmap(P, &tx, x, P->cols, m, ldx, bn)))
      return fail(TNL_ERR_CUDA, "tensor map (stack phase A) failed: %d", err);
    if (host_io) tx = tw;  // unused: the kernel reads x from host memory
    DecArgs a;
    memset(&a, 0, sizeof a);
    a.M_rows = (int32_t)P->r_pad;
    a.tokens = (int32_t)m;
    a.K = (int32_t)P->cols;
    const int total_kb = (int)((P->cols + 63) / 64);
    a.kb_per_split = 4;
    const int splits = (total_kb + 3) / 4;
    a.out = tacc[0];
    a.ldo_i = 64;
    a.ldo_j = 1;
    a.out_f32_atomic = 1;
    a.trace = P->trace;
    if (host_io) {
      a.x_host = static_cast<const __nv_bfloat16*>(x);
      a.ldx_host = ldx;
    }
    if ((err = launch_dec_a(tw, tx, a, splits, st)))
      return fail(TNL_ERR_CUDA, "stack phase A launch: %s", cudaGetErrorString((cudaError_t)err));
  }
  // boundaries l | l+1
  for (int l = 0; l + 1 < n; ++l) {
    tnl_plan* P = Pv[l];
    tnl_plan* Q = Pv[l + 1];
    CUtensorMap two, tt, twi;
    if ((err = get_tmap(P, &two, P->aout, P->r_pad, P->rows, P->r_pad, 128)) ||
        (err = get_tmap2(P, &tt, tacc[l % 3], true, 64, P->r_pad, 64, bn, 64, 0)) ||
        (err = get_tmap(Q, &twi, Q->bin, Q->cols, Q->r_pad, Q->cols, 128)))
      return fail(TNL_ERR_CUDA, "tensor map (stack boundary) failed: %d", err);
    FusedArgs f;
    memset(&f, 0, sizeof f);
    f.tokens = (int32_t)m;
    f.rows = (int32_t)P->rows;
    f.kB = (int32_t)P->r_pad;
    f.nA = (int32_t)Q->r_pad;
    f.t_in = tacc[l % 3];
    f.cnt_in = nullptr;
    f.t_out = tacc[(l + 1) % 3];
    f.t_zero = l >= 1 ? tacc[(l + 2) % 3] : nullptr;
    f.zero_elems = l >= 1 ? 64 * Pv[l - 1]->r_pad : 0;
    f.trace = P->trace ? P->trace + 16 * 1024 : nullptr;
    // (griddepcontrol.wait handoff and one CTA per 128 rows: a flag handoff and a CTA-pair
    // boundary kernel were built and measured slower, profiles/r02/ab_decode_flags_pair.jsonl)
    static const int ksplit_env = getenv("TNL_DEC_KSPLIT") ? atoi(getenv("TNL_DEC_KSPLIT")) : 0;  // A/B
    f.ksplit = (ksplit_env == 2 && f.nA > 128) ? 2 : 1;
    if ((err = launch_dec_fused(two, tt, twi, f, (int)(P->rows / 128) * f.ksplit, st)))
      return fail(TNL_ERR_CUDA, "stack boundary launch: %s", cudaGetErrorString((cudaError_t)err));
  }
  // last layer, phase B
  {
    const int l = n - 1;
    tnl_plan* P = Pv[l];
    const int64_t rows_local = P->row_end - P->row_begin;
    CUtensorMap tw2, tt, ty;
    if ((err = get_tmap(P, &tw2, P->aout, P->r_pad, rows_local, P->r_pad, 128)) ||
        (err = get_tmap2(P, &tt, tacc[l % 3], true, 64, P->r_pad, 64, bn, 64, 0)) ||
        (err = host_io ? 0 : get_tmap2(P, &ty, y, false, rows_local, m, ldy, 128, bn, 0)))
      return fail(TNL_ERR_CUDA, "tensor map (stack phase B) failed: %d", err);
    if (host_io) ty = tw2;  // unused: the kernel writes y to host memory
    DecArgs b;
    memset(&b, 0, sizeof b);
    b.M_rows = (int32_t)rows_local;
    b.tokens = (int32_t)m;
    b.K = (int32_t)P->r_pad;
    b.kb_per_split = (int32_t)((P->r_pad + 63) / 64);
    b.act_f32 = tacc[l % 3];
    b.act_ld = 64;
    b.out = y;
    b.ldo_i = 1;
    b.ldo_j = ldy;
    b.counter = cnt;  // the last CTA re-zeroes T_{n-1}
    b.zero_elems = 64 * P->r_pad;
    if (l >= 1) {  // T_{n-2}, read only by the last boundary kernel
      b.zero_prev = tacc[(l + 2) % 3];
      b.zero_prev_elems = 64 * Pv[l - 1]->r_pad;
    }
    b.trace = P->trace ? P->trace + 16 * 1024 : nullptr;
    if (host_io) {
      b.y_host = static_cast<__nv_bfloat16*>(y);
      b.ldy_host = ldy;
    }
    if ((err = launch_dec_b(tw2, tt, ty, b, st)))
      return fail(TNL_ERR_CUDA, "stack phase B launch: %s", cudaGetErrorString((cudaError_t)err));
  }
  return TNL_OK;
}


// Decode MLP block in three launches: (1) T_gu = [B_g; B_u] x (stacked phase A, split-K fp32
// reductions into decode slot 0), (2) the gated boundary kernel: per 128 intermediate rows,
// g = A_g T_g and u = A_u T_u (tcgen05, TMEM), h = silu(g) * u on chip, T_d += B_d[:, rows] h
// (reductions into slot 1), (3) down's phase B (re-zeroes T_d, zeroes T_gu). h never leaves the
// SM; the path replaces gate/up phase B, the SiLU*mul kernel and down's phase A.
static tnl_status mlp_decode_gated(tnl_mlp* B, const void* x, int64_t m, int64_t ldx, void* y, int64_t ldy,
                                   char* head, cudaStream_t st) {
  const int64_t rgu = B->rg + B->ru;
  tnl_plan* D = B->d;
  float* t0 = reinterpret_cast<float*>(head);
  float* t1 = reinterpret_cast<float*>(head + kDecSlotBytes);
  unsigned int* cnt = reinterpret_cast<unsigned int*>(head + kDecSlotBytes + kDecHeadBytes);
  const int bn = pick_bn(m);
  int err;
  {
    CUtensorMap tw, tx;
    if ((err = get_tmap(B->g, &tw, B->bgu, B->hidden, rgu, B->hidden, 128)) ||
        (err = get_tmap(B->g, &tx, x, B->hidden, m, ldx, bn)))
      return fail(TNL_ERR_CUDA, "tensor map (MLP decode phase A) failed: %d", err);
    DecArgs a;
    memset(&a, 0, sizeof a);
    a.M_rows = (int32_t)rgu;
    a.tokens = (int32_t)m;
    a.K = (int32_t)B->hidden;
    a.kb_per_split = 4;
    const int splits = (int)(((B->hidden + 63) / 64 + 3) / 4);
    a.out = t0;
    a.ldo_i = 64;
    a.ldo_j = 1;
    a.out_f32_atomic = 1;
    if ((err = launch_dec_a(tw, tx, a, splits, st)))
      return fail(TNL_ERR_CUDA, "MLP decode phase A launch: %s", cudaGetErrorString((cudaError_t)err));
  }
  {
    CUtensorMap two, tt, twi;
    if ((err = get_tmap(B->g, &two, B->agu, rgu, B->inter, rgu, 128)) ||
        (err = get_tmap2(B->g, &tt, t0, true, 64, rgu, 64, bn, 64, 0)) ||
        (err = get_tmap(D, &twi, D->bin, B->inter, D->r_pad, B->inter, 128)))
      return fail(TNL_ERR_CUDA, "tensor map (MLP gated boundary) failed: %d", err);
    FusedArgs f;
    memset(&f, 0, sizeof f);
    f.tokens = (int32_t)m;
    f.rows = (int32_t)B->inter;
    f.kB = (int32_t)rgu;
    f.nA = (int32_t)D->r_pad;
    f.t_in = t0;
    f.t_out = t1;
    f.kg = (int32_t)(B->rg / 64);
    if ((err = launch_dec_fused(two, tt, twi, f, (int)(B->inter / 128), st)))
      return fail(TNL_ERR_CUDA, "MLP gated boundary launch: %s", cudaGetErrorString((cudaError_t)err));
  }
  {
    CUtensorMap tw2, tt, ty;
    if ((err = get_tmap(D, &tw2, D->aout, D->r_pad, D->rows, D->r_pad, 128)) ||
        (err = get_tmap2(D, &tt, t1, true, 64, D->r_pad, 64, bn, 64, 0)) ||
        (err = get_tmap2(D, &ty, y, false, D->rows, m, ldy, 128, bn, 0)))
      return fail(TNL_ERR_CUDA, "tensor map (MLP decode phase B) failed: %d", err);
    DecArgs b;
    memset(&b, 0, sizeof b);
    b.M_rows = (int32_t)D->rows;
    b.tokens = (int32_t)m;
    b.K = (int32_t)D->r_pad;
    b.kb_per_split = (int32_t)((D->r_pad + 63) / 64);
    b.act_f32 = t1;
    b.act_ld = 64;
    b.out = y;
    b.ldo_i = 1;
    b.ldo_j = ldy;
    b.counter = cnt;  // the last CTA re-zeroes T_d
    b.zero_elems = 64 * D->r_pad;
    b.zero_prev = t0;  // T_gu, read only by the gated boundary kernel
    b.zero_prev_elems = 64 * rgu;
    if ((err = launch_dec_b(tw2, tt, ty, b, st)))
      return fail(TNL_ERR_CUDA, "MLP decode phase B launch: %s", cudaGetErrorString((cudaError_t)err));
  }
  return TNL_OK;
}

// ---------------------------------------------------------------------------
// Shared-input groups (tnl_stack.h): plans that read the same activations (a decoder's q, k, v)
// ---------------------------------------------------------------------------
struct tnl_group {
  std::vector<tnl_plan*> p;
  std::vector<int64_t> off;  // column of each plan's cut block in the stacked T
  int64_t cols = 0, r_total = 0;
  bool stacked = false;          // bf16 cut plans: one first-step GEMM over the stacked B_in panels
  __nv_bfloat16* bstack = nullptr;  // [B_in(p0); B_in(p1); ...] (r_total x cols)
};

static size_t group_ws_bytes(const tnl_group* G, int64_t m, size_t* o_t32, size_t* o_t) {
  size_t per = 0, a, b, c;
  for (const tnl_plan* P : G->p) per = std::max(per, ws_layout(P, std::max<int64_t>(m, 1), &a, &b, &c));
  size_t bytes = per;
  *o_t32 = bytes;
  bytes += round_up((int64_t)sizeof(float) * m * G->r_total, 256);
  *o_t = bytes;
  bytes += round_up((int64_t)2 * m * G->r_total, 256);
  return bytes;
}

tnl_status tnl_group_create(const tnl_plan* const* plans, int32_t n, tnl_group** out) {
  if (!plans || n < 1 || !out) return fail(TNL_ERR_ARG, "null argument");
  *out = nullptr;
  std::unique_ptr<tnl_group> G(new tnl_group);
  G->cols = plans[0]->cols;
  bool stack = true;
  for (int i = 0; i < n; ++i) {
    const tnl_plan* P = plans[i];
    if (!P) return fail(TNL_ERR_ARG, "null plan %d", i);
    if (P->cols != G->cols)
      return fail(TNL_ERR_SHAPE, "group plans must share the input width: %lld vs %lld", (long long)P->cols,
                  (long long)G->cols);
    stack = stack && P->compute_dtype == TNL_BF16 && P->plan_large == TNL_PLAN_CUT && P->bin &&
            P->family != TNL_FAMILY_DENSE && !P->tucker_chain;
    G->p.push_back(const_cast<tnl_plan*>(P));
    G->off.push_back(G->r_total);
    G->r_total += P->r_pad;
  }
  G->stacked = stack && n > 1;
  if (G->stacked) {
    CUDA_TRY(dev_alloc(&G->bstack, 2 * G->r_total * G->cols));
    for (int i = 0; i < n; ++i)
      CUDA_TRY(cudaMemcpy(G->bstack + G->off[i] * G->cols, G->p[i]->bin, 2 * G->p[i]->r_pad * G->cols,
                          cudaMemcpyDeviceToDevice));
  }
  *out = G.release();
  return TNL_OK;
}

tnl_status tnl_group_destroy(tnl_group* G) {
  if (!G) return TNL_OK;
  cudaDeviceSynchronize();
  dev_free(G->bstack);
  delete G;
  return TNL_OK;
}

tnl_status tnl_group_workspace_size(const tnl_group* G, int64_t m, size_t* bytes) {
  if (!G || !bytes) return fail(TNL_ERR_ARG, "null argument");
  size_t a, b;
  *bytes = group_ws_bytes(G, m, &a, &b);
  return TNL_OK;
}

tnl_status tnl_group_forward_ex(const tnl_group* Gc, const void* x, int64_t m, int64_t ldx, void* const* ys,
                                const int64_t* ldys, void* ws, size_t ws_bytes, const tnl_fwd_opts* o, void* stream) {
  tnl_group* G = const_cast<tnl_group*>(Gc);
  if (!G || !x || !ys || !ldys) return fail(TNL_ERR_ARG, "null argument");
  const int n = (int)G->p.size();
  size_t o_t32, o_t;
  const size_t need = group_ws_bytes(G, m, &o_t32, &o_t);
  if (ws_bytes < need) return fail(TNL_ERR_ARG, "group workspace %zu < required %zu bytes", ws_bytes, need);
  if (m == 0) return TNL_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool aligned = !(reinterpret_cast<uintptr_t>(x) & 15) && ldx % 8 == 0;
  bool ys_ok = true;
  for (int i = 0; i < n; ++i) ys_ok = ys_ok && ys[i] && !(reinterpret_cast<uintptr_t>(ys[i]) & 15) && ldys[i] % 8 == 0;
  if (!G->stacked || m <= kSwapMaxM || !aligned || !ys_ok || (o && o->accumulate)) {
    if (o && o->rms_fused) return fail(TNL_ERR_UNSUPPORTED, "rms_fused: needs the stacked prefill path");
    for (int i = 0; i < n; ++i) {  // per-plan forwards (decode, or plans that do not stack)
      tnl_status s = (o && (o->accumulate || o->ss_in))
                         ? tnl_forward_ex(G->p[i], x, m, ldx, ys[i], ldys[i], ws, o_t32, o, stream)
                         : tnl_forward(G->p[i], x, m, ldx, ys[i], ldys[i], ws, o_t32, stream);
      if (s) return s;
    }
    return TNL_OK;
  }
  // one first step over x (read once) into the stacked cut activations T (M x r_total)
  char* w = static_cast<char*>(ws);
  float* t32 = reinterpret_cast<float*>(w + o_t32);
  __nv_bfloat16* t = reinterpret_cast<__nv_bfloat16*>(w + o_t);
  tnl_plan* P0 = G->p[0];
  tnl_fwd_opts in_o = {};
  if (o && o->ss_in) {
    if (o->rms_n <= 0) return fail(TNL_ERR_ARG, "rms_n must be > 0");
    in_o.ss_in = o->ss_in;
    in_o.rms_n = o->rms_n;
    in_o.rms_eps = o->rms_eps;
  }
  if (o && o->rms_fused) {
    if (o->rms_n <= 0) return fail(TNL_ERR_ARG, "rms_n must be > 0");
    in_o.rms_fused = 1;
    in_o.rms_n = o->rms_n;
    in_o.rms_eps = o->rms_eps;
  }
  const tnl_fwd_opts* ino = (o && (o->ss_in || o->rms_fused)) ? &in_o : nullptr;
  const int64_t tiles1 = ((m + 127) / 128) * ((G->r_total + 255) / 256);
  const int64_t kb = (G->cols + 63) / 64;
  const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(148 / std::max<int64_t>(tiles1, 1), kb / 8));
  if (o && o->rms_fused && splits > 1)
    return fail(TNL_ERR_UNSUPPORTED, "rms_fused: the stacked first step splits K at M = %lld", (long long)m);
  tnl_status s;
  if (splits > 1) {
    if ((s = tc_step_p(P0, x, ldx, G->bstack, G->cols, m, G->r_total, G->cols, t32, G->r_total, true, splits, st)))
      return s;
    if (ino)
      to_bf16_scaled(t32, t, m, G->r_total, ino, st);
    else
      to_bf16(t32, t, m * G->r_total, st);
  } else if ((s = tc_step_p(P0, x, ldx, G->bstack, G->cols, m, G->r_total, G->cols, t, G->r_total, false, 1, st, 0,
                            ino))) {
    return s;
  }
  // each plan's output step on its block of T
  for (int i = 0; i < n; ++i) {
    tnl_plan* P = G->p[i];
    if ((s = tc_step_p(P, t + G->off[i], G->r_total, P->aout, P->r_pad, m, P->row_end - P->row_begin, P->r_pad, ys[i],
                       ldys[i], false, 1, st)))
      return s;
  }
  return TNL_OK;
}

tnl_status tnl_mlp_create(const tnl_plan* gate, const tnl_plan* up, const tnl_plan* down, int32_t flags,
                          tnl_mlp** out) {
  if (!gate || !up || !down || !out) return fail(TNL_ERR_ARG, "null argument");
  *out = nullptr;
  for (const tnl_plan* P : {gate, up, down})
    if (P->compute_dtype != TNL_BF16 || P->row_begin != 0 || P->row_end != P->rows)
      return fail(TNL_ERR_UNSUPPORTED, "MLP block needs full-row bf16 plans");
  if (gate->rows != up->rows || gate->cols != up->cols || down->cols != gate->rows || down->rows != gate->cols)
    return fail(TNL_ERR_SHAPE, "MLP block shapes: gate %lldx%lld, up %lldx%lld, down %lldx%lld",
                (long long)gate->rows, (long long)gate->cols, (long long)up->rows, (long long)up->cols,
                (long long)down->rows, (long long)down->cols);
  std::unique_ptr<tnl_mlp> B(new tnl_mlp());
  B->g = const_cast<tnl_plan*>(gate);
  B->u = const_cast<tnl_plan*>(up);
  B->d = const_cast<tnl_plan*>(down);
  B->hidden = gate->cols;
  B->inter = gate->rows;
  auto cut = [](const tnl_plan* P) { return P->family != TNL_FAMILY_DENSE && P->bin && P->aout; };
  B->rg = round_up(gate->r_pad, 64);
  B->ru = round_up(up->r_pad, 64);
  B->rd = round_up(down->r_pad, 64);
  B->fused = !(flags & 1) && cut(gate) && cut(up) && cut(down) && B->rg <= 128 && B->ru <= 128 && B->rd <= 256 &&
             B->inter % 64 == 0 && B->hidden % 8 == 0;
  if (B->fused) {
    MlpArgs a;
    memset(&a, 0, sizeof a);
    a.rg = (int32_t)B->rg;
    a.ru = (int32_t)B->ru;
    a.rd = (int32_t)B->rd;
    if (mlp_mid_smem(a) > 227 * 1024) B->fused = false;
  }
  // ranks the on-chip middle kernel cannot hold: gate/up output GEMMs fused with SiLU*mul
  B->dual = !B->fused && !(flags & 1) && cut(gate) && cut(up) && B->inter % 64 == 0 && B->hidden % 8 == 0;
  if (B->dual) {
    DualArgs da;
    memset(&da, 0, sizeof da);
    da.N = (int32_t)B->inter;
    da.kg = (int32_t)gate->r_pad;
    da.ku = (int32_t)up->r_pad;
    B->dual = dual_silu_ok(da);
  }
  CUDA_TRY(cudaStreamCreateWithFlags(&B->side, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&B->ev_fork, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&B->ev_join, cudaEventDisableTiming));
  // gate + up cut <= 256: everything resident; <= 512: down's B_in reuses the gate's A blocks
  // (needs the gate's cut to cover down's input blocks)
  B->gated = !(flags & 1) && cut(gate) && cut(up) && cut(down) && gate->decode_max_m && up->decode_max_m &&
             down->decode_max_m && down->r_pad <= 256 && B->inter % 128 == 0 && B->hidden % 128 == 0 &&
             (B->rg + B->ru <= 256 ||
              (B->rg + B->ru <= 512 && B->rg / 64 >= 2 * ((down->r_pad + 127) / 128)));
  if (B->gated) {
    const int64_t rgu = B->rg + B->ru;
    const size_t bytes = 2 * rgu * B->inter;
    CUDA_TRY(dev_alloc(&B->agu, bytes));
    CUDA_TRY(cudaMemset(B->agu, 0, bytes));
    CUDA_TRY(cudaMemcpy2D(B->agu, 2 * rgu, gate->aout, 2 * gate->r_pad, 2 * gate->r_pad, B->inter,
                          cudaMemcpyDeviceToDevice));
    CUDA_TRY(cudaMemcpy2D(B->agu + B->rg, 2 * rgu, up->aout, 2 * up->r_pad, 2 * up->r_pad, B->inter,
                          cudaMemcpyDeviceToDevice));
  }
  if (B->fused || B->dual || B->gated) {
    const size_t bytes = 2 * (B->rg + B->ru) * B->hidden;
    CUDA_TRY(dev_alloc(&B->bgu, bytes));
    CUDA_TRY(cudaMemset(B->bgu, 0, bytes));
    CUDA_TRY(cudaMemcpy(B->bgu, gate->bin, 2 * gate->r_pad * B->hidden, cudaMemcpyDeviceToDevice));
    CUDA_TRY(cudaMemcpy(B->bgu + B->rg * B->hidden, up->bin, 2 * up->r_pad * B->hidden, cudaMemcpyDeviceToDevice));
  }
  *out = B.release();
  return TNL_OK;
}


tnl_status tnl_mlp_destroy(tnl_mlp* B) {
  if (!B) return TNL_OK;
  cudaDeviceSynchronize();
  dev_free(B->bgu);
  dev_free(B->agu);
  if (B->ev_fork) cudaEventDestroy(B->ev_fork);
  if (B->ev_join) cudaEventDestroy(B->ev_join);
  if (B->side) cudaStreamDestroy(B->side);
  delete B;
  return TNL_OK;
}

int32_t tnl_mlp_is_fused(const tnl_mlp* B) { return B && B->fused ? 1 : 0; }

tnl_status tnl_mlp_workspace_size(const tnl_mlp* B, int64_t m, size_t* bytes) {
  if (!B || !bytes) return fail(TNL_ERR_ARG, "null argument");
  size_t off[4];
  mlp_ws_layout(B, std::max<int64_t>(m, 1), off, bytes);
  return TNL_OK;
}

static tnl_status mlp_forward_impl(const tnl_mlp* Bc, const void* x, int64_t m, int64_t ldx, void* y, int64_t ldy,
                                   void* ws, size_t ws_bytes, void* stream, const tnl_fwd_opts* o);

tnl_status tnl_mlp_forward(const tnl_mlp* Bc, const void* x, int64_t m, int64_t ldx, void* y, int64_t ldy,
                           void* ws, size_t ws_bytes, void* stream) {
  return mlp_forward_impl(Bc, x, m, ldx, y, ldy, ws, ws_bytes, stream, nullptr);
}

tnl_status tnl_mlp_forward_ex(const tnl_mlp* Bc, const void* x, int64_t m, int64_t ldx, void* y, int64_t ldy,
                              void* ws, size_t ws_bytes, const tnl_fwd_opts* opts, void* stream) {
  return mlp_forward_impl(Bc, x, m, ldx, y, ldy, ws, ws_bytes, stream, opts);
}

static tnl_status mlp_forward_impl(const tnl_mlp* Bc, const void* x, int64_t m, int64_t ldx, void* y, int64_t ldy,
                                   void* ws, size_t ws_bytes, void* stream, const tnl_fwd_opts* o) {
  tnl_mlp* B = const_cast<tnl_mlp*>(Bc);
  if (!B || !x || !y) return fail(TNL_ERR_ARG, "null argument");
  // folded RMSNorm of the block input (ss_in) and accumulation into its output
  tnl_fwd_opts in_o = {}, out_o = {};
  const bool fold = o && (o->accumulate || o->ss_in || o->rms_fused);
  if (fold) {
    in_o.ss_in = o->ss_in;
    in_o.rms_fused = o->rms_fused;
    in_o.rms_n = o->rms_n;
    in_o.rms_eps = o->rms_eps;
    out_o.accumulate = o->accumulate;
    if (m <= kSwapMaxM) return fail(TNL_ERR_UNSUPPORTED, "folded residual / RMSNorm: prefill (M > %lld) only", (long long)kSwapMaxM);
    if ((o->ss_in || o->rms_fused) && o->rms_n <= 0) return fail(TNL_ERR_ARG, "rms_n must be > 0");
    // the in-GEMM statistics need the stacked gate/up input step (fused and dual blocks)
    if (o->rms_fused && !(B->fused || B->dual))
      return fail(TNL_ERR_UNSUPPORTED, "rms_fused: needs a fused or dual MLP block");
  }
  if (m == 0) return TNL_OK;
  size_t off[4], need;
  mlp_ws_layout(B, m, off, &need);
  if (ws_bytes < need) return fail(TNL_ERR_ARG, "MLP workspace %zu < required %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  const bool prefill = m > kSwapMaxM;
  if (B->fused && prefill && ((reinterpret_cast<uintptr_t>(y) & 15) || ldy % 8 ||
                              (reinterpret_cast<uintptr_t>(x) & 15) || ldx % 8))
    return fail(TNL_ERR_SHAPE, "fused MLP needs 16-byte aligned x/y with row pitches % 8 == 0");
  if (B->dual && prefill && !((reinterpret_cast<uintptr_t>(x) & 15) || ldx % 8)) {
    // 1. T_gu = x . [B_g; B_u]^T   2. h = silu(T_g A_g^T) * (T_u A_u^T) in one kernel   3. y = down(h)
    const int64_t rgu = B->rg + B->ru;
    void* lws = w + off[0];
    size_t a_, b_, c_;
    const size_t lbytes = ws_layout(B->d, m, &a_, &b_, &c_);
    float* tgu32 = reinterpret_cast<float*>(w + off[1]);
    __nv_bfloat16* tgu = reinterpret_cast<__nv_bfloat16*>(w + off[2]);
    __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(w + off[3]);
    tnl_status s = mlp_tgu(B, x, m, ldx, tgu32, tgu, st, fold ? &in_o : nullptr);
    if (s) return s;
    CUtensorMap tt, tg, tu, th;
    int err;
    if ((err = get_tmap(B->g, &tt, tgu, rgu, m, rgu, 128)) ||
        (err = get_tmap(B->g, &tg, B->g->aout, B->g->r_pad, B->inter, B->g->r_pad, 64)) ||
        (err = get_tmap(B->u, &tu, B->u->aout, B->u->r_pad, B->inter, B->u->r_pad, 64)) ||
        (err = get_tmap2(B->g, &th, h, false, B->inter, m, B->inter, 64, 128, 128)))
      return fail(TNL_ERR_CUDA, "tensor map (MLP dual) failed: %d", err);
    DualArgs da;
    da.M = (int32_t)m;
    da.N = (int32_t)B->inter;
    da.kg = (int32_t)B->g->r_pad;
    da.ku = (int32_t)B->u->r_pad;
    da.u_off = (int32_t)B->rg;
    if ((err = launch_dual_silu(tt, tg, tu, th, da, st)))
      return fail(TNL_ERR_CUDA, "MLP dual kernel launch: %s", cudaGetErrorString((cudaError_t)err));
    if (fold) return forward_tc(B->d, h, m, B->inter, y, ldy, lws, lbytes, st, &out_o);
    return tnl_forward(B->d, h, m, B->inter, y, ldy, lws, lbytes, stream);
  }
  static const bool no_gated = getenv("TNL_MLP_NO_GATED") && atoi(getenv("TNL_MLP_NO_GATED")) == 1;  // A/B
  if (!prefill && B->gated && !no_gated && m <= kDecMaxM && !((reinterpret_cast<uintptr_t>(x) & 15) || ldx % 8) &&
      !((reinterpret_cast<uintptr_t>(y) & 15) || ldy % 8))
    return mlp_decode_gated(B, x, m, ldx, y, ldy, w + off[0], st);
  if (fold && !B->fused) {
    // unfused prefill with folds: gate/up normalise their input, down adds the residual
    void* lws = w + off[0];
    size_t a_, b_, c_, lbytes = 0;
    for (const tnl_plan* P : {B->g, B->u, B->d}) lbytes = std::max(lbytes, ws_layout(P, m, &a_, &b_, &c_));
    __nv_bfloat16* g = reinterpret_cast<__nv_bfloat16*>(w + off[1]);
    __nv_bfloat16* u = reinterpret_cast<__nv_bfloat16*>(w + off[2]);
    tnl_status s;
    if ((s = tnl_forward_ex(B->g, x, m, ldx, g, B->inter, lws, lbytes, &in_o, stream))) return s;
    if ((s = tnl_forward_ex(B->u, x, m, ldx, u, B->inter, lws, lbytes, &in_o, stream))) return s;
    if (launch_pdl(silu_mul_bf16, dim3(grid_for(m * B->inter / 8)), dim3(256), 0, st, g, u, m * B->inter / 8))
      return fail(TNL_ERR_CUDA, "silu_mul launch failed");
    return tnl_forward_ex(B->d, g, m, B->inter, y, ldy, lws, lbytes, &out_o, stream);
  }
  if (!B->fused || !prefill) {
    // unfused: three layer forwards + a SiLU*mul kernel
    void* lws = w + off[0];
    size_t a_, b_, c_, lbytes = 0;
    for (const tnl_plan* P : {B->g, B->u, B->d}) lbytes = std::max(lbytes, ws_layout(P, m, &a_, &b_, &c_));
    __nv_bfloat16* g = reinterpret_cast<__nv_bfloat16*>(w + off[1]);
    __nv_bfloat16* u = reinterpret_cast<__nv_bfloat16*>(w + off[2]);
    // decode: gate and up are independent given x -> up runs on the forked stream with
    // workspace slot 1 (its own zero-at-rest accumulator); TNL_MLP_SERIAL=1 disables
    static const bool serial = getenv("TNL_MLP_SERIAL") && atoi(getenv("TNL_MLP_SERIAL")) == 1;
    const bool fork = !serial && m <= kDecMaxM && B->u->decode_max_m && B->inter % 8 == 0;
    tnl_status su = TNL_OK;
    std::unique_lock<std::mutex> lk(B->fork_mu, std::defer_lock);
    if (fork) lk.lock();
    if (fork) {
      if (cudaEventRecord(B->ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(B->side, B->ev_fork, 0) != cudaSuccess)
        return fail(TNL_ERR_CUDA, "MLP fork failed");
      su = forward_decode(B->u, x, m, ldx, u, B->inter, static_cast<char*>(lws) + kDecSlotBytes, B->side);
      if (cudaEventRecord(B->ev_join, B->side) != cudaSuccess) return fail(TNL_ERR_CUDA, "MLP join failed");
    }
    tnl_status s = su ? su : tnl_forward(B->g, x, m, ldx, g, B->inter, lws, lbytes, stream);
    // join even on failure, so a capturing stream is never left forked
    if (fork && cudaStreamWaitEvent(st, B->ev_join, 0) != cudaSuccess && !s) return fail(TNL_ERR_CUDA, "MLP join failed");
    if (s) return s;
    if (!fork && (s = tnl_forward(B->u, x, m, ldx, u, B->inter, lws, lbytes, stream))) return s;
    if (launch_pdl(silu_mul_bf16, dim3(grid_for(m * B->inter / 8)), dim3(256), 0, st, g, u, m * B->inter / 8))
      return fail(TNL_ERR_CUDA, "silu_mul launch failed");
    return tnl_forward(B->d, g, m, B->inter, y, ldy, lws, lbytes, stream);
  }
  const int64_t rgu = B->rg + B->ru;
  float* tgu32 = reinterpret_cast<float*>(w + off[0]);
  __nv_bfloat16* tgu = reinterpret_cast<__nv_bfloat16*>(w + off[1]);
  float* td32 = reinterpret_cast<float*>(w + off[2]);
  __nv_bfloat16* td = reinterpret_cast<__nv_bfloat16*>(w + off[3]);
  tnl_status s;
  // 0. zero T_d's fp32 accumulator first, so no memset node sits between the T_gu GEMM and the
  //    middle kernel (they stay PDL-chained: the middle kernel's prologue overlaps the GEMM's tail)
  if (cudaMemsetAsync(td32, 0, sizeof(float) * m * B->rd, st) != cudaSuccess) return fail(TNL_ERR_CUDA, "memset");
  // 1. T_gu = x . [B_g; B_u]^T   (rows scaled by 1/rms(x) when the block's RMSNorm is folded)
  if ((s = mlp_tgu(B, x, m, ldx, tgu32, tgu, st, fold ? &in_o : nullptr))) return s;
  // 2. T_d = (silu(T_g A_g^T) * (T_u A_u^T)) B_d^T, h on chip
  MlpArgs a;
  memset(&a, 0, sizeof a);
  a.M = (int32_t)m;
  a.inter = (int32_t)B->inter;
  a.rg = (int32_t)B->rg;
  a.ru = (int32_t)B->ru;
  a.rd = (int32_t)B->rd;
  const bool pair = mlp_pair_ok(a);  // CTA pairs stream half of each weight chunk per CTA
  const int wbox = pair ? 32 : 64, dbox = pair ? (int)B->rd / 2 : (int)B->rd;
  CUtensorMap tt, tag, tau, tbd;
  int err;
  if ((err = get_tmap(B->g, &tt, tgu, rgu, m, rgu, 128)) ||
      (err = get_tmap2(B->g, &tag, B->g->aout, false, B->g->r_pad, B->inter, B->g->r_pad, 64, wbox, 128)) ||
      (err = get_tmap2(B->u, &tau, B->u->aout, false, B->u->r_pad, B->inter, B->u->r_pad, 64, wbox, 128)) ||
      (err = get_tmap2(B->d, &tbd, B->d->bin, false, B->inter, B->d->r_pad, B->inter, 64, dbox, 128)))
    return fail(TNL_ERR_CUDA, "tensor map (MLP) failed: %d", err);
  int64_t tiles_m = (m + 127) / 128;
  if (pair) tiles_m = (tiles_m + 1) / 2 * 2;
  const int64_t nchunks = B->inter / 64;
  // Slice the intermediate so the grid's waves are nearly full: one CTA per SM (smem-bound),
  // each CTA pays ~10 chunk-times of fixed cost (T tile load, pipeline fill, T_d flush) — fitted
  // to the slice sweep at M = 8192 (profiles/r02/mlp_slices_sweep.jsonl: 1 wave of 2 slices
  // 0.147 ms vs 0.161 ms with the earlier 4-chunk estimate, which picked 9 slices / 4 waves).
  int slices = 1;
  {
    int64_t best = INT64_MAX;
    for (int64_t s = 1; s <= nchunks; ++s) {
      const int64_t waves = (tiles_m * s + 147) / 148;
      const int64_t cost = waves * ((nchunks + s - 1) / s + 10);
      if (cost < best) best = cost, slices = (int)s;
    }
    static const int env_slices = getenv("TNL_MLP_SLICES") ? atoi(getenv("TNL_MLP_SLICES")) : 0;  // A/B switch
    if (env_slices > 0) slices = env_slices;
  }
  a.chunks_per_slice = (int32_t)((nchunks + slices - 1) / slices);
  slices = (int)((nchunks + a.chunks_per_slice - 1) / a.chunks_per_slice);
  // CTA pairs, balanced: split the flattened (token pair, chunk) work evenly over 74 pairs (148 SMs)
  // instead of whole slices per token pair (2 slices of 64 token pairs leave 20 SMs idle at M = 8192)
  a.tiles2 = (int32_t)(tiles_m / 2);
  a.per_pair = 0;
  static const bool balance = !(getenv("TNL_MLP_BALANCE") && atoi(getenv("TNL_MLP_BALANCE")) == 0);
  if (pair && balance) {
    const int64_t work = (tiles_m / 2) * nchunks;
    if (work >= 74 * 32) a.per_pair = (work + 73) / 74;
  }
  a.td = td32;
  a.ld_td = B->rd;
  a.trace = B->g->trace;
  if ((err = pair ? launch_mlp_mid_pair(tt, tag, tau, tbd, a, slices, st) : launch_mlp_mid(tt, tag, tau, tbd, a, slices, st)))
    return fail(TNL_ERR_CUDA, "MLP middle kernel launch: %s", cudaGetErrorString((cudaError_t)err));
  to_bf16(td32, td, m * B->rd, st);
  // 3. y = T_d . A_d^T  (+ residual, RMSNorm statistics of y when folded)
  return tc_step_p(B->d, td, B->rd, B->d->aout, B->d->r_pad, m, B->hidden, B->d->r_pad, y, ldy, false, 1, st, 0,
                   nullptr, fold ? &out_o : nullptr);
}

tnl_status tnl_add_rmsnorm(void* x, int64_t ldx, const void* o, int64_t ldo, void* h, int64_t ldh, int64_t m,
                           int64_t n, float eps, void* stream) {
  if (!x || !h) return fail(TNL_ERR_ARG, "null argument");
  if (m < 0 || n <= 0 || n % 8 || n > 8192 || ldx % 8 || ldh % 8 || (o && ldo % 8))
    return fail(TNL_ERR_SHAPE, "add_rmsnorm: m=%lld n=%lld (n % 8 == 0, n <= 8192, pitches % 8 == 0)",
                (long long)m, (long long)n);
  const int err = launch_add_rmsnorm(x, ldx, o, ldo, h, ldh, m, n, eps, static_cast<cudaStream_t>(stream));
  if (err) return fail(TNL_ERR_CUDA, "add_rmsnorm launch: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

tnl_status tnl_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes && (!dst || !src)) return fail(TNL_ERR_ARG, "null argument");
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15)
    return fail(TNL_ERR_ARG, "copy_async: dst and src must be 16-byte aligned");
  for (const void* p : {static_cast<const void*>(dst), src}) {
    cudaPointerAttributes at;
    if (bytes && (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type == cudaMemoryTypeUnregistered)) {
      cudaGetLastError();
      return fail(TNL_ERR_ARG, "copy_async: %p is pageable host memory (the SMs can only reach pinned memory)", p);
    }
  }
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int err = launch_copy16(dst, src, bytes, sms, static_cast<cudaStream_t>(stream));
  if (err) return fail(TNL_ERR_CUDA, "copy_async launch: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

tnl_status tnl_rms_stats(const void* x, int64_t ldx, int64_t m, int64_t n, float* ss, void* stream) {
  if (!x || !ss) return fail(TNL_ERR_ARG, "null argument");
  if (m < 0 || n <= 0 || n % 8 || ldx % 8 || ldx < n || (reinterpret_cast<uintptr_t>(x) & 15))
    return fail(TNL_ERR_SHAPE, "rms_stats: m=%lld n=%lld ldx=%lld (n, ldx %% 8 == 0, 16-byte aligned x)", (long long)m,
                (long long)n, (long long)ldx);
  if (m == 0) return TNL_OK;
  if (launch_pdl(row_sumsq_bf16, dim3((unsigned)((m + 7) / 8)), dim3(256), 0, static_cast<cudaStream_t>(stream),
                 static_cast<const __nv_bfloat16*>(x), ldx, n, m, ss))
    return fail(TNL_ERR_CUDA, "rms_stats launch failed");
  return TNL_OK;
}

tnl_status tnl_jacobi_sweeps(double* work, double* rot, int64_t batch, int64_t n, int64_t m, int64_t nv, double tol,
                             int32_t max_sweeps, int32_t* sweeps, void* stream) {
  if (batch < 0) return fail(TNL_ERR_ARG, "negative batch %lld", (long long)batch);
  if (batch == 0) return TNL_OK;
  if (n < 1 || m < 1 || nv < 0 || n > INT32_MAX || m > INT32_MAX || nv > INT32_MAX)
    return fail(TNL_ERR_SHAPE, "jacobi problem shape n=%lld m=%lld nv=%lld", (long long)n, (long long)m,
                (long long)nv);
  if (!work || (nv > 0 && !rot)) return fail(TNL_ERR_ARG, "null argument");
  if (!(tol >= 0.0) || max_sweeps < 0) return fail(TNL_ERR_ARG, "tol must be >= 0 and max_sweeps >= 0");
  const int err = tnl::launch_jacobi_sweeps(work, rot, batch, (int)n, (int)m, (int)nv, tol, max_sweeps, sweeps,
                                       static_cast<cudaStream_t>(stream));
  if (err) return fail(TNL_ERR_CUDA, "jacobi launch: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

tnl_status tnl_jacobi_sweeps_parallel(double* work, double* rot, int64_t n, int64_t m, int64_t nv, double tol,
                                      int32_t max_sweeps, int32_t* sweeps, void* stream) {
  if (n < 1 || m < 1 || nv < 0 || n > INT32_MAX || m > INT32_MAX || nv > INT32_MAX)
    return fail(TNL_ERR_SHAPE, "jacobi problem shape n=%lld m=%lld nv=%lld", (long long)n, (long long)m,
                (long long)nv);
  if (!work || (nv > 0 && !rot)) return fail(TNL_ERR_ARG, "null argument");
  if (!(tol >= 0.0) || max_sweeps < 0) return fail(TNL_ERR_ARG, "tol must be >= 0 and max_sweeps >= 0");
  int dev = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // grid-barrier words (count, generation, last rotating sweep): a stream-ordered allocation per
  // call, so concurrent calls on different streams never share a barrier
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned int* sync_buf = nullptr;
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&sync_buf), 4 * sizeof(unsigned int), st));
  const int err = tnl::launch_jacobi_parallel(work, rot, (int)n, (int)m, (int)nv, tol, max_sweeps, sweeps, sync_buf,
                                             sms, st);
  cudaFreeAsync(sync_buf, st);
  if (err) return fail(TNL_ERR_CUDA, "jacobi (parallel order) launch: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

tnl_status tnl_svd_finish(const double* work, const double* rot, int64_t batch, int64_t n, int64_t m, double* left,
                          double* values, double* right, double* scratch, void* stream) {
  if (batch < 0) return fail(TNL_ERR_ARG, "negative batch %lld", (long long)batch);
  if (batch == 0) return TNL_OK;
  if (n < 1 || m < n || n > INT32_MAX || m > INT32_MAX)
    return fail(TNL_ERR_SHAPE, "svd problem shape m=%lld n=%lld (needs m >= n >= 1)", (long long)m, (long long)n);
  if (!work || !rot || !left || !values || !right || !scratch) return fail(TNL_ERR_ARG, "null argument");
  const int err = tnl::launch_svd_finish(work, rot, batch, (int)n, (int)m, left, values, right, scratch,
                                         static_cast<cudaStream_t>(stream));
  if (err) return fail(TNL_ERR_CUDA, "svd finish launch: %s", cudaGetErrorString((cudaError_t)err));
  return TNL_OK;
}

tnl_status tnl_plan_set_trace(tnl_plan* plan, void* device_buffer) {
  if (!plan) return fail(TNL_ERR_ARG, "null plan");
  plan->trace = static_cast<unsigned long long*>(device_buffer);
  return TNL_OK;
}

tnl_status tnl_plan_create(const tnl_layer_desc* desc, int32_t compute_dtype, int64_t max_m,
                           int32_t flags, tnl_plan** out) {
  return create_impl(desc, compute_dtype, max_m, flags, 0, 0, out);
}

tnl_status tnl_plan_create_rows(const tnl_layer_desc* desc, int32_t compute_dtype, int64_t max_m,
                                int32_t flags, int64_t row_begin, int64_t row_end,
                                tnl_plan** out) {
  return create_impl(desc, compute_dtype, max_m, flags, row_begin, row_end, out);
}

tnl_status tnl_plan_destroy(tnl_plan* plan) {
  if (!plan) return TNL_OK;
  cudaDeviceSynchronize();  // work of any stream may still read the arena
  dev_free(plan->arena);
  dev_free(plan->stage_x);
  dev_free(plan->stage_y);
  dev_free(plan->stage_ws);
  delete plan;
  return TNL_OK;
}

tnl_status tnl_plan_query(const tnl_plan* P, tnl_plan_info* info) {
  if (!P || !info) return fail(TNL_ERR_ARG, "null argument");
  memset(info, 0, sizeof *info);
  info->rows = P->rows;
  info->cols = P->cols;
  info->r_cut = P->r_cut;
  info->param_count = P->param_count;
  info->chain_flops_per_token = P->chain_flops;
  info->cut_flops_per_token = P->cut_flops;
  info->dense_flops_per_token = 2 * P->rows * P->cols;
  const int64_t es = P->compute_dtype == TNL_BF16 ? 2 : 4;
  const int64_t rows_local = P->row_end - P->row_begin;
  int64_t wb = P->param_count * es;
  if (P->plan_large == TNL_PLAN_CUT && P->family != TNL_FAMILY_DENSE)
    wb = es * P->r_cut * (P->cols + rows_local);
  info->weight_bytes = wb;
  info->decode_weight_bytes = wb;
  info->compute_dtype = P->compute_dtype;
  info->plan_large = P->plan_large;
  info->plan_small = P->plan_small;
  info->decode_max_m = P->decode_max_m;
  info->row_begin = P->row_begin;
  info->row_end = P->row_end;
  return TNL_OK;
}

tnl_status tnl_workspace_size(const tnl_plan* P, int64_t m, size_t* bytes) {
  if (!P || !bytes) return fail(TNL_ERR_ARG, "null argument");
  if (m < 0) return fail(TNL_ERR_SHAPE, "negative token count");
  size_t a, b, c;
  *bytes = ws_layout(P, std::max<int64_t>(m, 1), &a, &b, &c);
  return TNL_OK;
}

tnl_status tnl_forward(const tnl_plan* plan, const void* x, int64_t m, int64_t ldx, void* y,
                       int64_t ldy, void* workspace, size_t workspace_bytes, void* stream) {
  tnl_plan* P = const_cast<tnl_plan*>(plan);
  if (!P) return fail(TNL_ERR_ARG, "null plan");
  if (m < 0) return fail(TNL_ERR_SHAPE, "negative token count");
  if (m == 0) return TNL_OK;
  if (!x || !y) return fail(TNL_ERR_ARG, "null x or y");
  if (ldx < P->cols) return fail(TNL_ERR_SHAPE, "ldx %lld < cols %lld", (long long)ldx, (long long)P->cols);
  if (ldy < P->row_end - P->row_begin) return fail(TNL_ERR_SHAPE, "ldy too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (P->plan_large == TNL_PLAN_GENERIC || P->compute_dtype != TNL_BF16)
    return forward_generic(P, x, m, ldx, y, ldy, workspace, workspace_bytes, st);
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (ldx % 8))
    return fail(TNL_ERR_SHAPE, "tensor-core plan needs 16-byte aligned x with ldx %% 8 == 0");
  return forward_tc(P, x, m, ldx, y, ldy, workspace, workspace_bytes, st);
}

tnl_status tnl_forward_ex(const tnl_plan* plan, const void* x, int64_t m, int64_t ldx, void* y, int64_t ldy,
                          void* workspace, size_t workspace_bytes, const tnl_fwd_opts* opts, void* stream) {
  if (opts && opts->rms_fused)
    return fail(TNL_ERR_UNSUPPORTED, "rms_fused: use tnl_group_forward_ex / tnl_mlp_forward_ex (stacked input steps)");
  if (!opts || (!opts->accumulate && !opts->ss_in))
    return tnl_forward(plan, x, m, ldx, y, ldy, workspace, workspace_bytes, stream);
  tnl_plan* P = const_cast<tnl_plan*>(plan);
  if (!P || !x || !y) return fail(TNL_ERR_ARG, "null argument");
  if (m <= 0) return m == 0 ? TNL_OK : fail(TNL_ERR_SHAPE, "negative token count");
  if (ldx < P->cols || ldy < P->row_end - P->row_begin) return fail(TNL_ERR_SHAPE, "row pitch too small");
  if (opts->ss_in && opts->rms_n <= 0) return fail(TNL_ERR_ARG, "rms_n must be > 0");
  if (P->plan_large == TNL_PLAN_GENERIC || P->compute_dtype != TNL_BF16 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      ldx % 8)
    return fail(TNL_ERR_UNSUPPORTED, "folded residual / RMSNorm: bf16 tensor-core plans only");
  return forward_tc(P, x, m, ldx, y, ldy, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), opts);
}

tnl_status tnl_forward_host(tnl_plan* P, const void* x_host, int64_t m, void* y_host, void* stream) {
  if (!P || !x_host || !y_host) return fail(TNL_ERR_ARG, "null argument");
  if (m <= 0 || m > P->max_m)
    return fail(TNL_ERR_SHAPE, "m=%lld outside host staging capacity %lld", (long long)m,
                (long long)P->max_m);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = P->compute_dtype == TNL_BF16 ? 2 : 4;
  const int64_t rows_local = P->row_end - P->row_begin;
  size_t need = 0;
  tnl_status s = tnl_workspace_size(P, P->max_m, &need);
  if (s) return s;
  if (P->stage_ws_bytes < need) {
    dev_free(P->stage_ws);
    P->stage_ws = nullptr;
    CUDA_TRY(dev_alloc(&P->stage_ws, need));
    CUDA_TRY(cudaMemset(P->stage_ws, 0, need));  // decode accumulator is zero at rest
    P->stage_ws_bytes = need;
  }
  CUDA_TRY(cudaMemcpyAsync(P->stage_x, x_host, es * m * P->cols, cudaMemcpyHostToDevice, st));
  s = tnl_forward(P, P->stage_x, m, P->cols, P->stage_y, rows_local, P->stage_ws, P->stage_ws_bytes,
                  stream);
  if (s) return s;
  CUDA_TRY(cudaMemcpyAsync(y_host, P->stage_y, es * m * rows_local, cudaMemcpyDeviceToHost, st));
  return TNL_OK;
}

tnl_status tnl_reconstruct(const tnl_plan* plan, void* w, int64_t ldw, int32_t out_dtype, void* stream) {
  tnl_plan* P = const_cast<tnl_plan*>(plan);
  if (!P || !w) return fail(TNL_ERR_ARG, "null argument");
  if (out_dtype != TNL_F32 && out_dtype != TNL_BF16) return fail(TNL_ERR_ARG, "bad out dtype");
  const int64_t rows_local = P->row_end - P->row_begin;
  if (ldw < P->cols) return fail(TNL_ERR_SHAPE, "ldw too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // W^T chunk = chain(identity chunk); written transposed into w.
  const int64_t chunk = std::min<int64_t>(P->cols, 512);
  float *eye = nullptr, *ws0 = nullptr, *ws1 = nullptr, *tmp = nullptr;
  const int64_t mst = std::max<int64_t>(P->max_state, 1);
  CUDA_TRY(dev_alloc(&eye, sizeof(float) * chunk * P->cols));
  CUDA_TRY(dev_alloc(&ws0, sizeof(float) * chunk * mst));
  CUDA_TRY(dev_alloc(&ws1, sizeof(float) * chunk * mst));
  CUDA_TRY(dev_alloc(&tmp, sizeof(float) * chunk * P->rows));
  tnl_status ret = TNL_OK;
  const int odt = out_dtype == TNL_BF16 ? DT_BF16 : DT_F32;
  for (int64_t c0 = 0; c0 < P->cols && ret == TNL_OK; c0 += chunk) {
    const int64_t m = std::min(chunk, P->cols - c0);
    identity_f32<<<grid_for(m * P->cols), 256, 0, st>>>(eye, m, P->cols, c0);
    ChainIO io;
    io.in = Operand{eye, DT_F32, P->cols, 1};
    io.out = Operand{tmp, DT_F32, P->rows, 1};
    io.ws[0] = ws0;
    io.ws[1] = ws1;
    std::vector<GStep> steps;
    build_steps(P, SEG_FULL, m, io, steps);
    if (run_steps(steps, st)) ret = fail(TNL_ERR_CUDA, "reconstruct launch failed");
    // tmp[j][i] -> w[i - row_begin][c0 + j]
    copy_2d_any<<<grid_for(m * rows_local), 256, 0, st>>>(tmp + P->row_begin, DT_F32, P->rows, 1,
                                                          static_cast<char*>(w) +
                                                              c0 * (odt == DT_BF16 ? 2 : 4),
                                                          odt, 1, ldw, m, rows_local);
  }
  cudaError_t e = cudaStreamSynchronize(st);
  dev_free(eye);
  dev_free(ws0);
  dev_free(ws1);
  dev_free(tmp);
  if (ret == TNL_OK && e != cudaSuccess) ret = fail(TNL_ERR_CUDA, "reconstruct: %s", cudaGetErrorString(e));
  return ret;
}

}  // extern "C"
