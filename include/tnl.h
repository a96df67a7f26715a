/*
 * tnl.h — C-ABI of the B200-native TN-structured linear layer (libtnl.so).
 *
 * This is the drop-in boundary for the reference's TN-linear forward path
 * (arxiv/paper_2602_01613 "Minima", /root/reference/pkg/src/minima):
 *
 *   reference                                        replaced by
 *   ---------------------------------------------------------------------------
 *   CompressedLayer(...) + validate()                 tnl_plan_create
 *     tn_decompositions.py:66-126                       (validates, packs the
 *                                                        cores into one device
 *                                                        arena, plans kernels)
 *   layer_to_matrix(L) @ x   (the only forward)       tnl_forward /
 *     tn_decompositions.py:364-365 + sensitivity.py:156  tnl_forward_host
 *   SPEC apply_compressed(c, x)  SPEC.md:476-484       tnl_forward
 *   reconstruct(L) / layer_to_matrix(L)                tnl_reconstruct
 *     tn_decompositions.py:346-365
 *   param_count(L)  tn_decompositions.py:368-374       tnl_plan_query
 *   SPEC flop_report / plan_contraction SPEC.md:465-499 tnl_plan_query
 *   minima.errors ShapeError/RankError/NumericsError   tnl_status codes +
 *     errors.py:8-21                                     tnl_last_error()
 *   native-call convention: jacobi_sweeps(work, rot,   caller-owned buffers,
 *     tol, max_sweeps) -> int  _jacobi_cy.pyx:11        int status return
 *
 * Conventions. Row-major, last index fastest (tensor_core.py:3-8). A layer of
 * mode shape ms with row_mode_count rm maps cols = prod(ms[rm:]) inputs to
 * rows = prod(ms[:rm]) outputs. The device API uses the torch orientation
 * y (M x rows) = x (M x cols) . W^T; the reference orientation W @ x with x of
 * shape (cols, M) is the same computation transposed.
 *
 * Ownership / threading. A plan owns an immutable packed copy of the cores and
 * the derived panels. tnl_forward is stream-ordered, allocation-free, does not
 * synchronise the host, and is CUDA-graph capturable; it is reentrant for
 * distinct workspaces. tnl_forward_host uses plan-owned staging buffers and
 * must not be called concurrently on the same plan.
 */
#ifndef TNL_H_
#define TNL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define TNL_API __attribute__((visibility("default")))
#else
#define TNL_API
#endif

#define TNL_ABI_VERSION 1
#define TNL_MAX_MODES 6 /* reshape_to_modes limit, tensor_core.py:72-73 */

typedef enum {
  TNL_OK = 0,
  TNL_ERR_SHAPE = 1,       /* minima.errors.ShapeError        (errors.py:8)  */
  TNL_ERR_RANK = 2,        /* minima.errors.RankError         (errors.py:16) */
  TNL_ERR_NUMERICS = 3,    /* minima.errors.NumericsError     (errors.py:12) */
  TNL_ERR_CUDA = 4,        /* CUDA runtime / driver failure                 */
  TNL_ERR_UNSUPPORTED = 5, /* valid layer, no kernel for this request      */
  TNL_ERR_ARG = 6          /* null pointer / bad enum / workspace too small */
} tnl_status;

typedef enum {
  TNL_FAMILY_DENSE = 0, /* "dense"  tn_decompositions.py:42 */
  TNL_FAMILY_TUCKER = 1,
  TNL_FAMILY_TT = 2,
  TNL_FAMILY_TR = 3
} tnl_family;

typedef enum { TNL_F64 = 0, TNL_F32 = 1, TNL_BF16 = 2 } tnl_dtype;

/* Plan preferences (tnl_plan_create flags). AUTO lets the host planner pick
 * per M bucket; the others force one contraction plan (for tests/benchmarks). */
enum {
  TNL_PLAN_AUTO = 0,
  TNL_PLAN_CUT = 1,     /* merged cut: y = A_out (B_in x), two tensor-core GEMMs */
  TNL_PLAN_CHAIN = 2,   /* core-by-core chain (Tucker-2: U_in, G, U_out; TT/TR:
                           input modes streamed, cut kept on chip)            */
  TNL_PLAN_GENERIC = 4, /* CUDA-core strided chain (exact fp32 FFMA path)     */
  TNL_PLAN_NO_DECODE = 8, /* disable the small-M decode kernels                 */
  TNL_PLAN_GEMV = 16     /* M <= 8: CUDA-core GEMV decode variant (warp per row) */
};

/* Host description of a layer (construct-from-cores, CompressedLayer fields).
 *   dense : arrays[0] = matrix (rows x cols)
 *   tucker: arrays[0] = core (ranks[0..d-1]), arrays[1+k] = factor k (ms[k] x ranks[k])
 *   tt/tr : arrays[k] = core k of shape (ranks[k], ms[k], ranks[k+1]);
 *           TT: ranks[0] = ranks[d] = 1; TR: ranks[d] = ranks[0] (closure).
 * All arrays are C-contiguous host memory of element type src_dtype. */
typedef struct {
  int32_t family;
  int32_t ndim;
  int32_t row_mode_count;
  int32_t src_dtype;
  int64_t mode_shape[TNL_MAX_MODES];
  int64_t ranks[TNL_MAX_MODES + 1];
  const void* arrays[TNL_MAX_MODES + 1];
} tnl_layer_desc;

typedef struct {
  int64_t rows, cols;
  int64_t r_cut;            /* cut dimension (TT r_rm; TR r0*r_rm; Tucker min side) */
  int64_t param_count;      /* == param_count(L), tn_decompositions.py:368-374 */
  int64_t chain_flops_per_token;
  int64_t cut_flops_per_token;
  int64_t dense_flops_per_token; /* 2*rows*cols, labelled, never a roofline */
  int64_t weight_bytes;     /* bytes the chosen large-M plan reads per call */
  int64_t decode_weight_bytes; /* bytes the chosen small-M plan reads per call */
  int32_t compute_dtype;
  int32_t plan_large;       /* TNL_PLAN_* used for M > decode threshold */
  int32_t plan_small;       /* TNL_PLAN_* used for M <= decode threshold */
  int32_t decode_max_m;     /* GEMV kernel threshold */
  int64_t row_begin, row_end; /* output rows this plan computes (sharding) */
} tnl_plan_info;

typedef struct tnl_plan tnl_plan;
typedef struct tnl_mlp tnl_mlp;
typedef struct tnl_chain tnl_chain;

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
} tnl_fwd_opts;

/* ss[i] = sum_j x[i][j]^2 for a bf16 [m][n] matrix (row pitch ldx % 8 == 0, n % 8 == 0). */
TNL_API tnl_status tnl_rms_stats(const void* x, int64_t ldx, int64_t m, int64_t n, float* ss, void* stream);

TNL_API int tnl_abi_version(void);
TNL_API const char* tnl_last_error(void);

/* Validate (same checks as CompressedLayer.validate, tn_decompositions.py:97-126),
 * pack, plan. max_m bounds tnl_forward_host staging (0 = no host staging). */
TNL_API tnl_status tnl_plan_create(const tnl_layer_desc* desc, int32_t compute_dtype, int64_t max_m,
                           int32_t flags, tnl_plan** out);
/* Same, restricted to output rows [row_begin, row_end) — output-mode sharding
 * (the leading output mode i0 of the layer when the range is i0-aligned). */
TNL_API tnl_status tnl_plan_create_rows(const tnl_layer_desc* desc, int32_t compute_dtype, int64_t max_m,
                                int32_t flags, int64_t row_begin, int64_t row_end,
                                tnl_plan** out);
TNL_API tnl_status tnl_plan_destroy(tnl_plan* plan);
TNL_API tnl_status tnl_plan_query(const tnl_plan* plan, tnl_plan_info* info);
TNL_API tnl_status tnl_workspace_size(const tnl_plan* plan, int64_t m, size_t* bytes);

/* y[m, r] (row stride ldy, r in [row_begin,row_end)) = sum_c x[m, c] W[r, c].
 * x, y, workspace: device pointers; element type = the plan's compute dtype.
 * The workspace must be ZERO-FILLED once before its first use: its head holds the
 * small-M (decode) split-K accumulator, which the kernels keep all-zero at rest.
 * Concurrent calls (other streams) need distinct workspaces. */
TNL_API tnl_status tnl_forward(const tnl_plan* plan, const void* x, int64_t m, int64_t ldx, void* y,
                       int64_t ldy, void* workspace, size_t workspace_bytes, void* stream);

TNL_API tnl_status tnl_forward_ex(const tnl_plan* plan, const void* x, int64_t m, int64_t ldx, void* y,
                                  int64_t ldy, void* workspace, size_t workspace_bytes, const tnl_fwd_opts* opts,
                                  void* stream);

/* End-to-end: host x (M x cols) -> H2D -> forward -> D2H -> host y (M x rows_local),
 * asynchronous on `stream` (host buffers should be pinned). m <= max_m. */
TNL_API tnl_status tnl_forward_host(tnl_plan* plan, const void* x_host, int64_t m, void* y_host,
                            void* stream);

/* Dense W (rows_local x cols, row stride ldw) in out_dtype (TNL_F32 / TNL_BF16),
 * computed on the device from the packed cores. */
TNL_API tnl_status tnl_reconstruct(const tnl_plan* plan, void* w, int64_t ldw, int32_t out_dtype,
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

/* Cluster-resident decode of a chain of square bf16 merged-cut layers (D x D, D % 1024 == 0,
 * D <= 6144, cut ranks padded to multiples of 64 <= 256): ONE 16-CTA thread-block cluster walks
 * all n layers for up to 32 tokens; each CTA owns D/16 rows of every layer, the per-layer
 * split-K reduction of the cut activations runs over distributed shared memory (no kernel
 * boundary, no global accumulator, deterministic summation order) and a producer warp streams
 * the weights, pre-swizzled into an arena at create time, ahead of the dependency chain.
 * Independent token groups (other streams) run as independent clusters. No workspace.
 * Same semantics as tnl_stack_forward over the same plans (the reference's forward is
 * layer_to_matrix(L) @ x per layer, tn_decompositions.py:364 / sensitivity.py:154-160).
 * TNL_ERR_UNSUPPORTED when the plans or the device do not qualify. */
TNL_API tnl_status tnl_chain_create(const tnl_plan* const* plans, int32_t n, int32_t flags, tnl_chain** out);
TNL_API tnl_status tnl_chain_forward(const tnl_chain* chain, const void* x, int64_t m, int64_t ldx, void* y,
                                     int64_t ldy, void* stream);
TNL_API tnl_status tnl_chain_destroy(tnl_chain* chain);
/* Debug: per-layer clock64 stamps of the chain kernel into a device buffer of
 * >= 16*256*8 int64 ([cta][layer][event]); NULL disables. */
TNL_API tnl_status tnl_chain_set_trace(tnl_chain* chain, void* device_buffer);

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

/* Batched cyclic one-sided Jacobi sweeps, fp64, in place — the reference's only native
 * component, `_jacobi_cy.jacobi_sweeps(work, rot, tol, max_sweeps) -> int`
 * (pkg/src/minima/_jacobi_cy.pyx:11-53, selected by _backend.py:5-25, called from
 * tensor_core.py:212 inside _jacobi_svd). `work` holds `batch` row-major problems of n rows
 * x m (the columns being orthogonalised), `rot` `batch` problems of n x nv (rotations are
 * accumulated into it); both device pointers, problem b at offset b*n*m / b*n*nv.
 * `sweeps` (device, batch int32, may be NULL) receives each problem's sweep count. Same
 * visiting order, skip rules and rotation formulas as the reference; dot products are
 * summed in a different order (the latitude the reference grants _jacobi_py.py:7-8).
 * Errors: TNL_ERR_SHAPE for n, m < 1 or nv < 0; TNL_ERR_ARG for null pointers, negative
 * tol / max_sweeps. */
TNL_API tnl_status tnl_jacobi_sweeps(double* work, double* rot, int64_t batch, int64_t n, int64_t m,
                                     int64_t nv, double tol, int32_t max_sweeps, int32_t* sweeps,
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

#ifdef __cplusplus
}
#endif
#endif /* TNL_H_ */
