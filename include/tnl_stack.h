/*
 * tnl_stack.h — decoder-stack extensions of libtnl.so (NOT part of the reference's API).
 *
 * include/tnl.h is the drop-in boundary for the reference's TN-linear layer (construct from
 * cores, forward, reconstruct, param counts, the Jacobi kernel). The reference has no decoder,
 * no MLP block and no multi-layer driver; the entry points below exist for the Qwen3-32B-shaped
 * stack driver of SURVEY.md §8(f) rows 1-2 (cfg3 fused MLP block, cfg4 64-layer stack) and for
 * measurement. They operate on tnl_plan objects created through tnl.h, so they add no second
 * path to the layer itself: every layer computes exactly what tnl_forward computes
 * (layer_to_matrix(L) @ x, tn_decompositions.py:364 / sensitivity.py:154-160).
 */
#ifndef TNL_STACK_H_
#define TNL_STACK_H_

#include "tnl.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tnl_mlp tnl_mlp;

/* Decoder-stack folds of the *_ex entry points (prefill, M > 64, bf16 cut plans):
 *   y (+)= f(x'),   x'_m = x_m / sqrt(ss_in[m] / rms_n + rms_eps)   (RMSNorm, no learned scale)
 * ss_in = per-token sum of squares of x (tnl_rms_stats); the cut activations are linear in x, so
 * the normalisation is one scale per token row in the first step's epilogue / conversion.
 * accumulate != 0: y += f(x') — the residual add rides on the last step's TMA store as a bulk
 * reduce-add at L2 (bf16), so the residual stream is updated in place with no extra pass. Together
 * they replace the decoder stack's residual-add + RMSNorm kernel (a read of x and o and a write of
 * x and h per norm) by one statistics read of x. Not part of the reference's API (the reference has
 * no decoder); used by the cfg4 stack driver. Other paths return TNL_ERR_UNSUPPORTED. */
typedef struct {
  int32_t accumulate;
  const float* ss_in;
  int32_t rms_n;
  float rms_eps;
  /* rms_fused != 0 (tnl_group_forward_ex / tnl_mlp_forward_ex only): normalise by the RMS of x
   * without ss_in — the first step, which streams every full row of x through shared memory,
   * sums the squares itself (no separate statistics pass over x). TNL_ERR_UNSUPPORTED when that
   * step would split K; the caller then uses tnl_rms_stats + ss_in. */
  int32_t rms_fused;
} tnl_fwd_opts;

/* ss[i] = sum_j x[i][j]^2 for a bf16 [m][n] matrix (row pitch ldx % 8 == 0, n % 8 == 0). */
TNL_API tnl_status tnl_rms_stats(const void* x, int64_t ldx, int64_t m, int64_t n, float* ss, void* stream);

TNL_API tnl_status tnl_forward_ex(const tnl_plan* plan, const void* x, int64_t m, int64_t ldx, void* y,
                                  int64_t ldy, void* workspace, size_t workspace_bytes, const tnl_fwd_opts* opts,
                                  void* stream);

/* A chain of layers (a decoder's projection stack): y = L_{n-1}(...L_0(x)).
 * For M <= 64 and merged-cut bf16 plans whose widths chain (rows % 128 == 0) this
 * runs ONE fused kernel per layer boundary (phase B of layer l + phase A of layer
 * l+1, the activation never leaves the SM); otherwise it chains tnl_forward.
 * The workspace (tnl_stack_workspace_size) must be zero-filled before first use. */
TNL_API tnl_status tnl_stack_workspace_size(const tnl_plan* const* plans, int32_t n, int64_t m,
                                            size_t* bytes);
TNL_API tnl_status tnl_stack_forward(const tnl_plan* const* plans, int32_t n, const void* x,
                                     int64_t m, int64_t ldx, void* y, int64_t ldy, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* tnl_stack_forward with zero-copy host I/O: x (m x ldx) and y (m x ldy) are PINNED host buffers;
 * the first kernel reads its x slices straight from host memory and the last one writes y straight
 * to it (no copy-engine transfers, no staging kernels). Fused decode stacks only (M <= 64). */
TNL_API tnl_status tnl_stack_forward_host(const tnl_plan* const* plans, int32_t n, const void* x_host, int64_t m,
                                          int64_t ldx, void* y_host, int64_t ldy, void* workspace,
                                          size_t workspace_bytes, void* stream);

/* Qwen3 MLP block of three TN layers: y = down(silu(gate(x)) * up(x)).
 * For merged-cut bf16 plans (gate/up cut <= 128, down cut <= 256) and M > 64 the
 * intermediate h (M x inter) never reaches HBM: one kernel streams chunks of the
 * gate/up output panels and the down input panel, applies SiLU*mul on chip and
 * folds h into down's cut accumulator. Otherwise (or flags & 1) it runs unfused.
 * The plans must outlive the block. */
TNL_API tnl_status tnl_mlp_create(const tnl_plan* gate, const tnl_plan* up, const tnl_plan* down,
                                  int32_t flags, tnl_mlp** out);
TNL_API tnl_status tnl_mlp_destroy(tnl_mlp* mlp);
TNL_API int32_t tnl_mlp_is_fused(const tnl_mlp* mlp);
TNL_API tnl_status tnl_mlp_workspace_size(const tnl_mlp* mlp, int64_t m, size_t* bytes);
TNL_API tnl_status tnl_mlp_forward(const tnl_mlp* mlp, const void* x, int64_t m, int64_t ldx,
                                   void* y, int64_t ldy, void* workspace, size_t workspace_bytes,
                                   void* stream);

/* opts (tnl_fwd_opts): ss_in normalises the block's input, residual / ss_out apply to its output */
TNL_API tnl_status tnl_mlp_forward_ex(const tnl_mlp* mlp, const void* x, int64_t m, int64_t ldx, void* y,
                                      int64_t ldy, void* workspace, size_t workspace_bytes, const tnl_fwd_opts* opts,
                                      void* stream);

/* Decoder-stack plumbing (not part of the reference's TN path; used by the Qwen3 stack driver):
 * x <- x + o (skipped when o == NULL), h <- x / sqrt(mean(x^2) + eps) per row, bf16 [m][n]
 * with row pitches ldx / ldo / ldh (multiples of 8), n % 8 == 0, n <= 8192. One pass. */
TNL_API tnl_status tnl_add_rmsnorm(void* x, int64_t ldx, const void* o, int64_t ldo, void* h, int64_t ldh,
                                   int64_t m, int64_t n, float eps, void* stream);

/* Stream-ordered copy of `bytes` executed by the SMs (H2D / D2H / D2D): either pointer may be
 * pinned host memory (cudaHostAlloc / torch pin_memory — mapped into the unified address
 * space), both 16-byte aligned. PDL-launched, so in a decode graph the next TN kernel prefetches
 * its weights while the activations arrive, and no memcpy node breaks the launch chain. Used for
 * the host I/O of a decode step (the reference has no device path; its forward is host numpy). */
TNL_API tnl_status tnl_copy_async(void* dst, const void* src, size_t bytes, void* stream);

/* Number of libtnl kernel launches issued by this thread since the last reset
 * (evidence counter for benchmarks). */
TNL_API int64_t tnl_launch_count(int32_t reset);

/* Debug: record per-CTA %globaltimer stamps of the decode kernels into a device
 * buffer of >= 2*1024*16 uint64 (phase A at [0, 16K), phase B at [16K, 32K));
 * NULL disables. Not for production use (adds global stores). */
TNL_API tnl_status tnl_plan_set_trace(tnl_plan* plan, void* device_buffer);

/* Shared-input group: plans that read the same activations (a decoder's q, k and v projections of
 * one normalised hidden state). For prefill (M > 64) over bf16 merged-cut plans their B_in panels
 * are stacked at create time, so ONE first-step GEMM reads x once into the concatenated cut
 * activations (folded RMSNorm row scale applied there, opts->ss_in), then each plan's output step
 * writes its own y. Otherwise (decode, other plan kinds) it runs the plans one after another.
 * The plans must outlive the group; opts->accumulate is not supported by the stacked path. */
typedef struct tnl_group tnl_group;
TNL_API tnl_status tnl_group_create(const tnl_plan* const* plans, int32_t n, tnl_group** out);
TNL_API tnl_status tnl_group_destroy(tnl_group* group);
TNL_API tnl_status tnl_group_workspace_size(const tnl_group* group, int64_t m, size_t* bytes);
TNL_API tnl_status tnl_group_forward_ex(const tnl_group* group, const void* x, int64_t m, int64_t ldx, void* const* ys,
                                        const int64_t* ldys, void* workspace, size_t workspace_bytes,
                                        const tnl_fwd_opts* opts, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TNL_STACK_H_ */
