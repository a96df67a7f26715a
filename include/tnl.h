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
  TNL_PLAN_CHAIN = 2,   /* core-by-core chain, every family and shape (bf16:
                           tcgen05 steps; Tucker-2 and a two-mode TT/TR input
                           side in fused kernels with intermediates on chip)  */
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


/* End-to-end: host x (M x cols) -> H2D -> forward -> D2H -> host y (M x rows_local),
 * asynchronous on `stream` (host buffers should be pinned). m <= max_m. */
TNL_API tnl_status tnl_forward_host(tnl_plan* plan, const void* x_host, int64_t m, void* y_host,
                            void* stream);

/* Dense W (rows_local x cols, row stride ldw) in out_dtype (TNL_F32 / TNL_BF16),
 * computed on the device from the packed cores. */
TNL_API tnl_status tnl_reconstruct(const tnl_plan* plan, void* w, int64_t ldw, int32_t out_dtype,
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





/* The same sweeps for ONE large problem (e.g. a 5120 x 640 unfolding) in a parallel order: the
 * Brent-Luk round-robin ordering rotates n/2 disjoint pairs per step, one warp per pair across a
 * persistent cooperative grid, one grid barrier per step. Same skip rules and rotation formulas;
 * the pair ORDER differs from the reference's cyclic order (tensor_core.py:203-212), so results
 * agree with it up to rounding (spectra to <= 1e-10 relative) and the sweep count may differ.
 * Opt-in: the batched cyclic kernel above stays the parity path. `sweeps` (device int32, may be
 * NULL) receives the sweep count. */
TNL_API tnl_status tnl_jacobi_sweeps_parallel(double* work, double* rot, int64_t n, int64_t m, int64_t nv, double tol,
                                              int32_t max_sweeps, int32_t* sweeps, void* stream);

/* The post-processing of _jacobi_svd (tensor_core.py:214-235) on the device, batched, one CTA per
 * problem: values = row norms of the swept `work` (batch x n x m) in stable descending order,
 * left (batch x m x n) = work[order]^T / values, completed for exactly-zero values by the greedy
 * canonical pick of _complete_basis (:185-200), right (batch x n x n) = rot[order]^T, and the sign
 * convention (largest-|.| entry of each left vector positive, right flipped with it). Requires
 * m >= n (the reference transposes wide inputs first; swap left/right for them). `scratch`:
 * device buffer of batch * (2n + 2m) doubles. All pointers device memory, row-major. */
TNL_API tnl_status tnl_svd_finish(const double* work, const double* rot, int64_t batch, int64_t n, int64_t m,
                                  double* left, double* values, double* right, double* scratch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TNL_H_ */
