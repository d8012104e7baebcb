// Per-SM streaming probe (research, not product): how fast can one CTA pull
// bytes from HBM into shared memory, and how does the rate scale with the
// number of streaming CTAs?  Three load paths over the same bytes:
//   tma2d  -- cp.async.bulk.tensor 2D boxes of 128 rows x 128 B (the GEMM
//             weight-operand pattern: 128 separate 128-byte row segments)
//   bulk1d -- cp.async.bulk 1D copies of 16 KB contiguous chunks (a
//             pre-tiled weight layout would allow this)
//   ldg    -- 256 threads, 16-byte loads, 8 in flight per thread
// Each CTA streams its own contiguous region (HBM resident, > L2 in total).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_stream scripts/probe_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

constexpr int CHUNK = 16384;
constexpr int STAGES = 16;   // ring slots (runtime `stages` <= STAGES are used)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(b),
      "r"(ph)
      : "memory");
}

// mode 0: tma 2D (128 rows x 64 bf16 per box), mode 1: bulk 1D 16 KB,
// mode 3: two 64-row boxes per 16 KB stage (the 64-column QKV weight tile),
// mode 4: one 64-row weight box + one 128-row box of a 1-row activation
//         tensor (127 rows zero-filled out of bounds) per stage -- the
//         few-row decode GEMM's operand pattern (8 KB of weights per stage)
__global__ void __launch_bounds__(128) stream_async(const __grid_constant__ CUtensorMap tm,
                                                    const __grid_constant__ CUtensorMap tm64,
                                                    const __grid_constant__ CUtensorMap tma1,
                                                    const __grid_constant__ CUtensorMap tma128,
                                                    const __grid_constant__ CUtensorMap tma1r8,
                                                    const __grid_constant__ CUtensorMap tma32,
                                                    const __grid_constant__ CUtensorMap tmw, int box_rows,
                                                    const __grid_constant__ CUtensorMap tm3,
                                                    const uint8_t* base, size_t per_cta,
                                                    int rows_per_cta, int kcols, int mode,
                                                    int stages, int stage_bytes,
                                                    unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(su32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // modes 0-3 stream 16 KB of weights per stage; mode 4 streams 8 KB
  const int nchunks = static_cast<int>(per_cta / (mode == 9 ? box_rows * 256 : mode == 8 ? box_rows * 128
                                                   : mode >= 4 ? 8192 : CHUNK));
  const uint8_t* src = base + per_cta * blockIdx.x;
  const int kblocks = kcols / 64;   // 64 bf16 = 128 B per box row
  auto issue = [&](int c) {
    const int s = c % stages;
    const uint32_t dst = su32(smem + s * stage_bytes);
    if (mode < 8)
      mbar_expect(su32(&full[s]), mode == 6 ? 8192 + 1024 : mode == 7 ? 8192 + 4096
                                  : mode >= 4 ? 8192 + 16384 : CHUNK);
    if (mode == 9) {   // 3D box: box_rows rows x 2 K blocks (two stacked 2D tiles)
      const int kb2 = c % (kblocks / 2), rb = c / (kblocks / 2);
      mbar_expect(su32(&full[s]), box_rows * 256);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tm3)), "r"(0), "r"(blockIdx.x * rows_per_cta + rb * box_rows),
          "r"(kb2 * 2), "r"(su32(&full[s]))
          : "memory");
      return;
    }
    if (mode == 8) {
      // one box of box_rows rows x 128 B: chunk c = K block (c % kblocks) of
      // row block (c / kblocks)
      const int kb = c % kblocks, rb = c / kblocks;
      mbar_expect(su32(&full[s]), box_rows * 128);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tmw)), "r"(kb * 64), "r"(blockIdx.x * rows_per_cta + rb * box_rows),
          "r"(su32(&full[s]))
          : "memory");
      return;
    }
    if (mode >= 3) {
      const int kb = c % kblocks, rb = c / kblocks;
      const int y = blockIdx.x * rows_per_cta + rb * 64;
      if (mode == 3) {
        // two consecutive K blocks of the same 64 rows: 16 KB per stage
        for (int h = 0; h < 2; ++h)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst + h * 8192),
              "l"(reinterpret_cast<uint64_t>(&tm64)), "r"(((2 * c + h) % kblocks) * 64),
              "r"(blockIdx.x * rows_per_cta + ((2 * c + h) / kblocks) * 64), "r"(su32(&full[s]))
              : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(&tm64)), "r"(kb * 64), "r"(y), "r"(su32(&full[s]))
            : "memory");
        const CUtensorMap* am = mode == 4 ? &tma1 : mode == 5 ? &tma128 : mode == 6 ? &tma1r8 : &tma32;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst + 8192),
            "l"(reinterpret_cast<uint64_t>(am)), "r"(kb * 64), "r"(0), "r"(su32(&full[s]))
            : "memory");
      }
    } else if (mode == 1) {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "l"(src + static_cast<size_t>(c) * CHUNK), "r"(CHUNK), "r"(su32(&full[s]))
          : "memory");
    } else {
      // chunk c = K block (c % kblocks) of row block (c / kblocks) of this CTA
      const int kb = c % kblocks, rb = c / kblocks;
      const int x = kb * 64, y = blockIdx.x * rows_per_cta + rb * 128;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(su32(&full[s]))
          : "memory");
    }
  };
  for (int c = 0; c < stages && c < nchunks; ++c) issue(c);
  unsigned long long acc = 0;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % stages;
    mbar_wait(su32(&full[s]), (c / stages) & 1);
    acc += smem[s * stage_bytes + (c & 1023)];
    if (c + stages < nchunks) issue(c + stages);
  }
  if (acc == 0xdeadbeefULL) *sink = acc;
}

__global__ void __launch_bounds__(256) stream_ldg(const uint4* base, size_t per_cta_vec,
                                                  unsigned long long* sink) {
  const uint4* src = base + per_cta_vec * blockIdx.x;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < per_cta_vec; i += 256 * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t j = i + static_cast<size_t>(u) * 256;
      v[u] = j < per_cta_vec ? __ldcs(src + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0xdeadbeefu) *sink = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  const size_t per_cta = 8u << 20;   // 8 MB per CTA
  const int max_ctas = 296;
  const int kcols = 4096;            // matrix row = 8 KB (like a 7B weight row)
  const int rows_per_cta = static_cast<int>(per_cta / (kcols * 2));
  uint8_t* buf = nullptr;
  uint8_t* evict = nullptr;
  unsigned long long* sink = nullptr;
  CK(cudaMalloc(&evict, 512u << 20));
  CK(cudaMalloc(&buf, per_cta * max_ctas));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(buf, 1, per_cta * max_ctas));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(kcols),
                        static_cast<cuuint64_t>(rows_per_cta) * max_ctas};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(kcols) * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  if (reinterpret_cast<EncodeFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box,
                                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    std::printf("tensor map encode failed\n");
    return 1;
  }
  CUtensorMap tm64 = tm, tma1;
  cuuint32_t box64[2] = {64, 64};
  reinterpret_cast<EncodeFn>(fn)(&tm64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box64,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t dims1[2] = {static_cast<cuuint64_t>(kcols), 1};
  reinterpret_cast<EncodeFn>(fn)(&tma1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, evict, dims1, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap tma128, tma1r8;
  cuuint64_t dims128[2] = {static_cast<cuuint64_t>(kcols), 128};
  reinterpret_cast<EncodeFn>(fn)(&tma128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, evict, dims128, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint32_t box8[2] = {64, 8};
  reinterpret_cast<EncodeFn>(fn)(&tma1r8, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, evict, dims1, strides, box8,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap tma32;
  cuuint32_t box32[2] = {64, 32};
  reinterpret_cast<EncodeFn>(fn)(&tma32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, evict, dims128, strides, box32,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 200 * 1024;
  CK(cudaFuncSetAttribute(stream_async, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int counts[] = {1, 36, 74, 148};
  const char* names[] = {"tma2d", "bulk1d", "ldg", "tma64x2", "w+a1oob", "w+a128x8", "w+a1box8",
                         "w+a32x16", "box"};
  CUtensorMap tmw[3];
  const int brs[3] = {64, 128, 256};
  for (int i = 0; i < 3; ++i) {
    cuuint32_t bx[2] = {64, static_cast<cuuint32_t>(brs[i])};
    reinterpret_cast<EncodeFn>(fn)(&tmw[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, bx,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  // 3D view of the weights: (64 elements, rows, K blocks), strides (row, 128 B)
  CUtensorMap tm3;
  {
    cuuint64_t d3[3] = {64, static_cast<cuuint64_t>(rows_per_cta) * max_ctas,
                        static_cast<cuuint64_t>(kcols / 64)};
    cuuint64_t s3[2] = {static_cast<cuuint64_t>(kcols) * 2, 128};
    cuuint32_t b3[3] = {64, 64, 2};
    cuuint32_t e3[3] = {1, 1, 1};
    if (reinterpret_cast<EncodeFn>(fn)(&tm3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      std::printf("3d map failed\n");
  }
  // (box rows, stages, mode): 2D 64 / 128-row boxes vs a 3D 64-row x 2-K-block box
  const int cfgs[4][3] = {{64, 16, 8}, {128, 8, 8}, {64, 8, 9}, {256, 4, 8}};
  for (int ci = 0; ci < 4; ++ci) {
    const int mode = cfgs[ci][2];
    const int bi = cfgs[ci][0] == 64 ? 0 : cfgs[ci][0] == 128 ? 1 : 2;
    const int stages = cfgs[ci][1];
    const int stage_bytes = cfgs[ci][0] * 128 * (mode == 9 ? 2 : 1);
    std::printf("%s box %d rows x %d stages (%d KB in flight)\n", mode == 9 ? "3D(2 K blocks)" : "2D",
                cfgs[ci][0], stages, stages * stage_bytes / 1024);
    for (int n : counts) {
      float best = 1e30f;
      for (int it = 0; it < 5; ++it) {
        // evict: write 512 MB elsewhere first (L2 is 126 MB)
        CK(cudaMemsetAsync(evict, it, 512u << 20));
        CK(cudaEventRecord(e0));
        if (mode != 2)
          stream_async<<<n, 128, smem>>>(tm, tm64, tma1, tma128, tma1r8, tma32, tmw[bi], cfgs[ci][0], tm3, buf,
                                         per_cta, rows_per_cta, kcols, mode, stages, stage_bytes, sink);
        else
          stream_ldg<<<n, 256>>>(reinterpret_cast<const uint4*>(buf), per_cta / 16, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      const double gbs = static_cast<double>(per_cta) * n / (best * 1e-3) / 1e9;
      std::printf("%-7s ctas=%4d  %9.1f GB/s total  %7.1f GB/s per CTA\n", names[mode], n, gbs, gbs / n);
    }
  }
  return 0;
}
