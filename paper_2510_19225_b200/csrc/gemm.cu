// K2: tcgen05 + TMA GEMMs for the dense projections of the decode step.
//
//   C[M, N] = A[M, K] . B[N, K]^T      (A = activations, B = weights; both K-major bf16)
//
// One CTA computes one 128 x BN tile.  Warp roles (256 threads):
//   warp 0     one elected lane issues TMA loads (A 128x64, B BNx64, 128B swizzle)
//              into a STAGES-deep smem ring guarded by full/empty mbarriers;
//   warp 1     one elected lane issues tcgen05.mma (M=128, N=BN, K=16) into a
//              TMEM fp32 accumulator and frees smem stages with tcgen05.commit;
//   warp 2     allocates / frees the TMEM columns;
//   warps 4-7  epilogue: tcgen05.ld 32 lanes x 16 columns -> registers -> fused
//              op (bias / fp32 residual add / SwiGLU / fp32 store) -> global.
//
// Batch invariance (SURVEY.md §7 hard part 2): an output row depends only on
// its A row and on B; the K loop order is fixed and there is no split-K, so a
// token row gets bit-identical results whether it runs in a 512-row decode
// batch or inside a 16k-row varlen prefill chunk.  Migration resume relies on
// this.
#include "internal.h"

namespace rlb {

constexpr int BM = 128;
constexpr int BK = 64;

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
};

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + expf(-g)); }

template <int BN, int EPI>
__global__ void __launch_bounds__(256, 1)
    gemm_bf16_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 GemmParams p) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_blk = blockIdx.y;
  const int n_blk = blockIdx.x;
  const int nk = p.K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(tfull), 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::STAGES;
        const uint32_t ph = (kb / C::STAGES) & 1;
        mbar_wait(smem_u32(&empty[s]), ph ^ 1);
        mbar_expect_tx(smem_u32(&full[s]), C::STAGE_BYTES);
        tma_load_2d(smem_u32(sA + s * C::A_BYTES), &tmA, smem_u32(&full[s]), kb * BK, m_blk * BM);
        tma_load_2d(smem_u32(sB + s * C::B_BYTES), &tmB, smem_u32(&full[s]), kb * BK, n_blk * BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::STAGES;
        const uint32_t ph = (kb / C::STAGES) & 1;
        mbar_wait(smem_u32(&full[s]), ph);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * C::A_BYTES));
        const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * C::B_BYTES));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          // +32 bytes per K=16 step inside the 128 B swizzle atom (encoded >> 4)
          umma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
        }
        umma_commit(smem_u32(&empty[s]));
      }
      umma_commit(smem_u32(tfull));
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int m = m_blk * BM + row;
    const bool live = m < p.M;
    mbar_wait(smem_u32(tfull), 0);
    tc_fence_after();
    const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16);
    if constexpr (EPI == EPI_SWIGLU) {
      bf16* out = reinterpret_cast<bf16*>(p.out);
#pragma unroll 1
      for (int g = 0; g < BN / 128; ++g) {
#pragma unroll 1
        for (int jc = 0; jc < 64; jc += 16) {
          uint32_t rg[16], ru[16];
          tmem_ld16(tbase + g * 128 + jc, rg);
          tmem_ld16(tbase + g * 128 + 64 + jc, ru);
          tmem_ld_wait();
          const int col = n_blk * (BN / 2) + g * 64 + jc;
          if (live && col < p.N / 2) {
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float a0 = silu_f(__uint_as_float(rg[2 * i])) * __uint_as_float(ru[2 * i]);
              const float a1 =
                  silu_f(__uint_as_float(rg[2 * i + 1])) * __uint_as_float(ru[2 * i + 1]);
              pk[i] = pack_bf2(a0, a1);
            }
            uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(m) * p.ldo + col);
            dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
        }
      }
    } else if constexpr (EPI == EPI_ARGMAX) {
      // greedy head: per (row, N-tile) max and its lowest column index; the
      // full-vocab fp32 logits never reach HBM.
      float best = -INFINITY;
      int bidx = 0x7fffffff;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        tmem_ld16(tbase + c, r);
        tmem_ld_wait();
        const int n = n_blk * BN + c;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float v = __uint_as_float(r[i]);
          if (n + i < p.N && v > best) {
            best = v;
            bidx = n + i;
          }
        }
      }
      if (live) {
        float2* part = reinterpret_cast<float2*>(p.out) + static_cast<size_t>(m) * p.ldo + n_blk;
        *part = make_float2(best, __int_as_float(bidx));
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        tmem_ld16(tbase + c, r);
        tmem_ld_wait();
        const int n = n_blk * BN + c;
        if (!live || n >= p.N) continue;
        if constexpr (EPI == EPI_BF16) {
          bf16* out = reinterpret_cast<bf16*>(p.out);
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
          if (p.bias != nullptr) {
            const uint4* bp = reinterpret_cast<const uint4*>(p.bias + n);
            const uint4 b0 = bp[0], b1 = bp[1];
            const uint32_t bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              v[2 * i] += bf_lo(bb[i]);
              v[2 * i + 1] += bf_hi(bb[i]);
            }
          }
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) pk[i] = pack_bf2(v[2 * i], v[2 * i + 1]);
          uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(m) * p.ldo + n);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        } else if constexpr (EPI == EPI_RESADD) {
          float4* h = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) +
                                                static_cast<size_t>(m) * p.ldo + n);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float4 x = h[i];
            x.x += __uint_as_float(r[4 * i]);
            x.y += __uint_as_float(r[4 * i + 1]);
            x.z += __uint_as_float(r[4 * i + 2]);
            x.w += __uint_as_float(r[4 * i + 3]);
            h[i] = x;
          }
        } else {  // EPI_F32
          float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) +
                                                static_cast<size_t>(m) * p.ldo + n);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            o[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                               __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host --

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(ptr);
  }
  return fn;
}

int make_kmajor_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int box_rows) {
  PFN_encodeTiled_t enc = encode_fn();
  RLB_CHECK(enc != nullptr, RLB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  RLB_CHECK(k % BK == 0, RLB_ERR_ARG, "GEMM K must be a multiple of 64");
  RLB_CHECK((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, RLB_ERR_ARG, "TMA base not 16B aligned");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(k * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RLB_CHECK(r == CUDA_SUCCESS, RLB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return RLB_OK;
}

template <int BN, int EPI>
static int set_attr() {
  RLB_CUDA(cudaFuncSetAttribute(gemm_bf16_tc<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                GemmCfg<BN>::SMEM));
  return RLB_OK;
}

template <int BN>
static int set_attr_bn() {
  int rc;
  if ((rc = set_attr<BN, EPI_BF16>()) || (rc = set_attr<BN, EPI_RESADD>()) ||
      (rc = set_attr<BN, EPI_F32>()) || (rc = set_attr<BN, EPI_ARGMAX>()))
    return rc;
  if constexpr (BN >= 128) return set_attr<BN, EPI_SWIGLU>();
  return RLB_OK;
}

int gemm_prepare() {
  static bool done[64] = {false};
  int dev = 0;
  RLB_CUDA(cudaGetDevice(&dev));
  if (done[dev & 63]) return RLB_OK;
  int rc;
  if ((rc = set_attr_bn<64>()) || (rc = set_attr_bn<128>()) || (rc = set_attr_bn<256>())) return rc;
  done[dev & 63] = true;
  return RLB_OK;
}

template <int BN, int EPI>
static int launch_one(const CUtensorMap& a, const CUtensorMap& b, const GemmParams& p,
                      cudaStream_t st) {
  using C = GemmCfg<BN>;
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM);
  gemm_bf16_tc<BN, EPI><<<grid, 256, C::SMEM, st>>>(a, b, p);
  RLB_CUDA(cudaGetLastError());
  return RLB_OK;
}

template <int BN>
static int launch_bn(const CUtensorMap& a, const CUtensorMap& b, int epi, const GemmParams& p,
                     cudaStream_t st) {
  switch (epi) {
    case EPI_BF16: return launch_one<BN, EPI_BF16>(a, b, p, st);
    case EPI_RESADD: return launch_one<BN, EPI_RESADD>(a, b, p, st);
    case EPI_SWIGLU:
      if constexpr (BN >= 128) return launch_one<BN, EPI_SWIGLU>(a, b, p, st);
      break;
    case EPI_F32: return launch_one<BN, EPI_F32>(a, b, p, st);
    case EPI_ARGMAX: return launch_one<BN, EPI_ARGMAX>(a, b, p, st);
  }
  set_error("bad epilogue");
  return RLB_ERR_ARG;
}

int gemm_launch(const CUtensorMap& a, const CUtensorMap& b, int block_n, int epi,
                const GemmParams& p, cudaStream_t st) {
  if (p.M <= 0) return RLB_OK;
  RLB_CHECK(p.K % BK == 0 && p.N % 16 == 0, RLB_ERR_ARG, "GEMM shape not tileable");
  RLB_CHECK(epi != EPI_SWIGLU || (block_n % 128 == 0 && p.N % 128 == 0), RLB_ERR_ARG,
            "SwiGLU GEMM needs 128-column gate/up tiles");
  switch (block_n) {
    case 64: return launch_bn<64>(a, b, epi, p, st);
    case 128: return launch_bn<128>(a, b, epi, p, st);
    case 256: return launch_bn<256>(a, b, epi, p, st);
  }
  set_error("block_n must be 64, 128 or 256");
  return RLB_ERR_ARG;
}

}  // namespace rlb

extern "C" int rlb_gemm(int device, int32_t M, int32_t N, int32_t K, const void* A, const void* B,
                        const void* bias, void* Cout, int32_t epilogue, int32_t block_n) {
  using namespace rlb;
  RLB_CUDA(cudaSetDevice(device));
  int rc = gemm_prepare();
  if (rc) return rc;
  CUtensorMap ma, mb;
  rc = make_kmajor_map(&ma, A, M, K, BM);
  if (rc) return rc;
  rc = make_kmajor_map(&mb, B, N, K, block_n);
  if (rc) return rc;
  GemmParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.bias = static_cast<const bf16*>(bias);
  p.out = Cout;
  p.ldo = epilogue == EPI_SWIGLU ? N / 2 : N;
  rc = gemm_launch(ma, mb, block_n, epilogue, p, 0);
  if (rc) return rc;
  RLB_CUDA(cudaDeviceSynchronize());
  return RLB_OK;
}
