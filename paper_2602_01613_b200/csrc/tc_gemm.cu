// tc_gemm.cu — warp-specialised tcgen05 GEMM step (see tc_gemm.cuh).
//
// CTA = 6 warps: warp 0 issues TMA loads into a STAGES-deep smem ring, warp 1
// allocates TMEM and (one elected lane) issues tcgen05.mma kind::f16 128xBNx16,
// warps 2-5 drain the fp32 accumulator (tcgen05.ld 32x32b) and store. The
// mbarrier protocol: full[s] (TMA -> MMA, tx-count), empty[s] (MMA commit ->
// TMA), done (last MMA commit -> epilogue).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <mutex>

#include "common.cuh"
#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tnl {

namespace {

constexpr int BM = 128, BK = 64;
constexpr uint32_t A_STAGE = BM * BK * 2;

template <int BN>
constexpr uint32_t tmem_cols() {
  return BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
}

template <int BN, int STAGES>
constexpr size_t smem_bytes() {
  return 1024 + (size_t)STAGES * (A_STAGE + (size_t)BN * BK * 2) + 256;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const TcGemmArgs args) {
  constexpr uint32_t B_STAGE = BN * BK * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tile_m = blockIdx.x, tile_n = blockIdx.y;
  const int total_kb = (args.K + BK - 1) / BK;
  const int kb0 = blockIdx.z * args.kb_per_split;
  const int kb1 = min(total_kb, kb0 + args.kb_per_split);
  const int nkb = kb1 - kb0;
  const uint32_t warp = warp_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<tmem_cols<BN>()>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  pdl_wait();
  pdl_launch_dependents();

  if (nkb > 0) {
    if (warp == 0) {
      if (elect_one()) {
        for (int i = 0; i < nkb; ++i) {
          const int s = i % STAGES;
          if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
          tma_load_2d(sA + s * A_STAGE, &tmA, &full[s], (kb0 + i) * BK, tile_m * BM);
          tma_load_2d(sB + s * B_STAGE, &tmB, &full[s], (kb0 + i) * BK, tile_n * BN);
        }
      }
    } else if (warp == 1) {
      if (elect_one()) {
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
        for (int i = 0; i < nkb; ++i) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          tc_fence_after();
          const uint64_t adesc = smem_desc_sw128(smem_u32(sA + s * A_STAGE));
          const uint64_t bdesc = smem_desc_sw128(smem_u32(sB + s * B_STAGE));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance the start address by 32 B (16 bf16) inside the 128 B swizzle row
            mma_bf16_ss(tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (i | k) != 0);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(done);
      }
      __syncwarp();
    } else {
      // epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
      mbar_wait(done, 0);
      tc_fence_after();
      const uint32_t q = warp & 3;
      const int row = tile_m * BM + q * 32 + lane_id();
      const bool row_ok = row < args.M;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((q * 32) << 16) + c, v);
        const int col0 = tile_n * BN + c;
        if (!row_ok || col0 >= args.N) continue;
        const int ncol = min(16, args.N - col0);
        if (args.out_mode == TC_OUT_BF16) {
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(args.out) + (int64_t)row * args.ldo_i +
                             (int64_t)col0 * args.ldo_j;
          if (args.ldo_j == 1 && ncol == 16 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
            uint4 p0, p1;
            p0.x = pack_bf16x2(v[0], v[1]);
            p0.y = pack_bf16x2(v[2], v[3]);
            p0.z = pack_bf16x2(v[4], v[5]);
            p0.w = pack_bf16x2(v[6], v[7]);
            p1.x = pack_bf16x2(v[8], v[9]);
            p1.y = pack_bf16x2(v[10], v[11]);
            p1.z = pack_bf16x2(v[12], v[13]);
            p1.w = pack_bf16x2(v[14], v[15]);
            reinterpret_cast<uint4*>(o)[0] = p0;
            reinterpret_cast<uint4*>(o)[1] = p1;
          } else {
            #pragma unroll
            for (int e = 0; e < 16; ++e)
              if (e < ncol) o[(int64_t)e * args.ldo_j] = __float2bfloat16_rn(v[e]);
          }
        } else {
          float* o = static_cast<float*>(args.out) + (int64_t)row * args.ldo_i +
                     (int64_t)col0 * args.ldo_j;
          if (args.out_mode == TC_OUT_F32_ATOMIC) {
            if (args.ldo_j == 1 && ncol == 16 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
              for (int e = 0; e < 16; e += 4) red_add_v4(o + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
            } else {
              #pragma unroll
              for (int e = 0; e < 16; ++e)
                if (e < ncol) atomicAdd(o + (int64_t)e * args.ldo_j, v[e]);
            }
          } else {
            #pragma unroll
            for (int e = 0; e < 16; ++e)
              if (e < ncol) o[(int64_t)e * args.ldo_j] = v[e];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<tmem_cols<BN>()>(tmem);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

template <int BN, int STAGES>
int launch_impl(const CUtensorMap& a, const CUtensorMap& b, const TcGemmArgs& args, int splits,
                bool pdl, cudaStream_t stream) {
  constexpr size_t smem = smem_bytes<BN, STAGES>();
  static AttrOnce attr_set;  // benign race: idempotent attribute set
  int attr_dev = 0;
  if (attr_set.needed(&attr_dev)) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    attr_set.done(attr_dev);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((args.M + BM - 1) / BM, (args.N + BN - 1) / BN, splits);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, STAGES>, a, b, args);
  count_launch();
  return (int)e;
}

}  // namespace

int make_tmap_bf16(CUtensorMap* map, const void* base, int64_t k, int64_t rows, int64_t ld,
                   int box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return (int)cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 2) % 16) return (int)cudaErrorInvalidValue;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

int make_tmap_2d(CUtensorMap* map, const void* base, bool f32, int64_t inner, int64_t outer,
                 int64_t ld, int box_inner, int box_outer, int swizzle_bytes) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return (int)cudaErrorNotSupported;
  const int64_t es = f32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * es) % 16) return (int)cudaErrorInvalidValue;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                  : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                        : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

int launch_tc_gemm(const CUtensorMap& a, const CUtensorMap& b, const TcGemmArgs& args, int bn,
                   int splits, bool pdl, cudaStream_t stream) {
  switch (bn) {
    case 16:
      return launch_impl<16, 6>(a, b, args, splits, pdl, stream);
    case 32:
      return launch_impl<32, 6>(a, b, args, splits, pdl, stream);
    case 64:
      return launch_impl<64, 6>(a, b, args, splits, pdl, stream);
    case 128:
      return launch_impl<128, 5>(a, b, args, splits, pdl, stream);
    case 256:
      return launch_impl<256, 4>(a, b, args, splits, pdl, stream);
    default:
      return (int)cudaErrorInvalidValue;
  }
}

}  // namespace tnl
