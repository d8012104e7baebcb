// K3 row kernel: residual stream -> RMSNorm -> bf16 input of the next GEMM.
// The projections add their (cluster-reduced) split-K sums into h in their
// epilogues, so the engine runs this with S = 0; S > 0 reduces fp32 partials
// [S][M][N] in split order first (kept for partial-producing callers).
#define RLB_PDL_CLASS 4
#include "internal.h"

namespace rlb {

constexpr int NORM_MAX_PER_THREAD = 16;   // hidden <= 4096 with 256 threads

// Row r (= src_rows[i] when gathering): x = h[r] + sum_z part[z][r], written
// back to h when write_h, then xn[i] = x * rsqrt(mean(x^2) + eps) * w (bf16).
template <int S>
__global__ void __launch_bounds__(256) resid_norm_kernel(
    float* __restrict__ h, const float* __restrict__ part, int Mp,
    const int* __restrict__ src_rows, const bf16* __restrict__ w, int H, float eps,
    bf16* __restrict__ xn, int write_h) {
  __shared__ float red[8];
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x;
  const int r = src_rows ? src_rows[i] : i;
  float* hr = h + static_cast<size_t>(r) * H;
  const size_t slab = static_cast<size_t>(Mp) * H;
  const float* pr = part + static_cast<size_t>(r) * H;
  float x[NORM_MAX_PER_THREAD];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < NORM_MAX_PER_THREAD; ++k) {
    const int c = threadIdx.x + k * 256;
    if (c < H) {
      float p[S > 0 ? S : 1];
#pragma unroll
      for (int z = 0; z < S; ++z) p[z] = pr[z * slab + c];
      float acc = 0.f;
      if constexpr (S > 0) {
        acc = p[0];
#pragma unroll
        for (int z = 1; z < S; ++z) acc += p[z];
      }
      x[k] = hr[c] + acc;
    }
  }
#pragma unroll
  for (int k = 0; k < NORM_MAX_PER_THREAD; ++k) {
    const int c = threadIdx.x + k * 256;
    if (c < H) {
      ss = __fmaf_rn(x[k], x[k], ss);
      if (S > 0 && write_h) hr[c] = x[k];
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) tot += red[k];
  const float inv = rsqrtf(tot / static_cast<float>(H) + eps);
  bf16* orow = xn + static_cast<size_t>(i) * H;
#pragma unroll
  for (int k = 0; k < NORM_MAX_PER_THREAD; ++k) {
    const int c = threadIdx.x + k * 256;
    if (c < H) orow[c] = __float2bfloat16_rn((x[k] * inv) * __bfloat162float(w[c]));
  }
}

int resid_norm_launch(float* h, const float* part, int S, int Mp, const int* src_rows, int R,
                      const bf16* w, int H, float eps, bf16* xn, bool write_h, cudaStream_t st) {
  if (R <= 0) return RLB_OK;
  RLB_CHECK(H <= 256 * NORM_MAX_PER_THREAD, RLB_ERR_ARG, "hidden size too large for RMSNorm");
  const int wh = write_h ? 1 : 0;
#define RN_CASE(s) \
  case s:                                                                                        \
    RLB_CUDA(launch_k(resid_norm_kernel<s>, dim3(R), dim3(256), 0, st, h, part, Mp, src_rows, w, H, \
                      eps, xn, wh));                                                              \
    break;
  switch (S) {
    RN_CASE(0) RN_CASE(1) RN_CASE(2) RN_CASE(3) RN_CASE(4) RN_CASE(5) RN_CASE(6) RN_CASE(7)
    RN_CASE(8)
    default: RLB_CHECK(false, RLB_ERR_ARG, "split-K factor must be <= 8");
  }
#undef RN_CASE
  return RLB_OK;
}

}  // namespace rlb
