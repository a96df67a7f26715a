// decode.cuh — small-M (decode) kernels for the merged-cut plan.
//
// A layer at decode is y = A_out (B_in x) with M <= 64 tokens. Both steps are
// weight-streaming: the weights sit on the MMA M side ("swap-AB"), the tokens
// on N. Two launches per layer, chained with programmatic dependent launch:
//
//   phase A  T_acc[k][m] += sum_j B_in[k][j] x[m][j]      split-K over j, fp32
//            vector reductions (red.global.add.v4) into a plan-owned,
//            kappa-major accumulator that is all-zero at rest;
//   phase B  y[m][i] = sum_k A_out[i][k] bf16(T_acc[k][m]) — T_acc is TMA-
//            staged as fp32 and converted to the bf16 SW128 operand by the
//            (otherwise idle) epilogue warps; y leaves through one TMA store;
//            the last CTA to finish reading re-zeroes T_acc.
//
// Weight tiles are TMA-loaded BEFORE griddepcontrol.wait, so the weight
// stream of layer l overlaps the tail of the previous kernel.
//
// For M <= 8 the same protocol runs on CUDA cores (GEMV-like: 16-byte
// vector loads of the weight rows, warp-shuffle reductions).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tnl {

struct DecArgs {
  int32_t M_rows;    // weight rows (MMA M side): r_pad (phase A) or rows (phase B)
  int32_t tokens;    // M (N side)
  int32_t K;         // contraction length
  int32_t kb_per_split;
  // activation operand (phase B): fp32 [tokens][K] with row stride act_ld
  const float* act_f32;
  int64_t act_ld;
  // output
  void* out;
  int64_t ldo_i, ldo_j;  // element (weight-row i, token j)
  int32_t out_f32_atomic; // 1: red.add fp32 (phase A); 0: bf16 store (phase B)
  // last-CTA zeroing of act_f32 (phase B)
  unsigned int* counter;
  int64_t zero_elems;
  // cooperative zeroing (all CTAs, after the dependency wait) of a buffer the previous kernel read
  float* zero_prev;
  int64_t zero_prev_elems;
  // optional timeline (tnl_plan_set_trace): [cta][16] %globaltimer stamps
  unsigned long long* trace;
  // zero-copy host I/O (decode stacks, tnl_stack_forward_host): phase A reads its x slice straight
  // from pinned host memory [tokens][ldx_host] (the epilogue warps fill the operand stages);
  // phase B writes y straight to pinned host memory [tokens][ldy_host]
  const __nv_bfloat16* x_host;
  int64_t ldx_host;
  __nv_bfloat16* y_host;
  int64_t ldy_host;
};

// phase A: weights (TMA map `w`, rows=M_rows, K) x activations (TMA map `x`, bf16 tokens x K)
int launch_dec_a(const CUtensorMap& w, const CUtensorMap& x, const DecArgs& a, int splits,
                 cudaStream_t st);
// phase B: weights (TMA map `w`) x fp32 accumulator (TMA map `t`: kappa-major [K][64] fp32,
// box {BN tokens, 64 kappa}); y via TMA store (map `y`: [tokens][rows] bf16, box {128, BN});
// the last CTA re-zeroes a.act_f32 (a.zero_elems floats)
int launch_dec_b(const CUtensorMap& w, const CUtensorMap& t, const CUtensorMap& y, const DecArgs& a,
                 cudaStream_t st);

// Fused boundary kernel of a decode stack (decode_fused.cu): phase B of layer l
// (A_out^l, accumulator T_l) + phase A of layer l+1 (B_in^{l+1}) in one launch.
struct FusedArgs {
  int32_t tokens;      // M <= 64
  int32_t rows;        // rows of layer l == cols of layer l+1 (multiple of 128)
  int32_t kB;          // r_pad of layer l (<= 256)
  int32_t nA;          // r_pad of layer l+1 (<= 256)
  float* t_in;         // T_l, kappa-major [kB][64]
  unsigned int* cnt_in;  // unused (kept for layout stability)
  float* t_out;        // T_{l+1}, kappa-major [nA][64], fp32 reductions
  int64_t zero_elems;  // floats of t_zero
  float* t_zero;       // T_{l-1} (read by the previous kernel only): zeroed cooperatively, so it is
                       // back at rest before it is accumulated again two boundaries later
                       // (three rotating accumulators; no last-CTA tail, no counters)
  unsigned long long* trace;  // optional per-CTA %globaltimer stamps [cta][16]
  int32_t kg;          // gated MLP boundary (0: plain): the first kg 64-blocks of kappa are the gate's
                       // cut (T_g, A_g), the rest the up projection's; y = silu(A_g T_g) * (A_u T_u)
  int32_t ksplit;      // plain boundaries with nA > 128: 2 CTAs per row tile, one kappa' half each
                       // (grid = 2 * rows / 128); 0/1: one CTA per row tile
};
// wo: A_out^l map (box {64, 128}, SW128); t: T_l fp32 map (box {BN, 64}); wi: B_in^{l+1}
// map (box {64, 128}, SW128). grid = rows / 128.
int launch_dec_fused(const CUtensorMap& wo, const CUtensorMap& t, const CUtensorMap& wi,
                     const FusedArgs& a, int grid, cudaStream_t st);

// CUDA-core GEMV variants (tokens <= 8): warp per weight row, no atomics.
// T is fp32 [tokens][ldt] (plain stores, no zero-at-rest requirement).
int launch_gemv_a(const __nv_bfloat16* w, int64_t ldw, int rows, int K, const __nv_bfloat16* x,
                  int64_t ldx, int tokens, float* t, int64_t ldt, cudaStream_t st);
int launch_gemv_b(const __nv_bfloat16* w, int64_t ldw, int rows, int K, const float* t, int64_t ldt,
                  int tokens, __nv_bfloat16* y, int64_t ldy, cudaStream_t st);

}  // namespace tnl
