// K3 row kernel: residual stream -> RMSNorm -> bf16 input of the next GEMM.
// S > 0: first sum the S fp32 split-K partials [S][M][N] of the projection
// that precedes it in split order and add them to h (the O projection at
// decode, the down projection in prefill chunks); S = 0 when the projection
// already added its (cluster-reduced) sum into h in its epilogue.
#define RLB_PDL_CLASS 4
#include "internal.h"

namespace rlb {

// Row r (= src_rows[i] when gathering): x = h[r] + sum_z part[z][r], written
// back to h when write_h, then xn[i] = x * rsqrt(mean(x^2) + eps) * w (bf16).
// One CTA per row; each thread owns V float4 column groups (t, t + T, ...),
// so every load is 16 bytes and all of a thread's loads are in flight at once.
template <int S, int V>
__global__ void __launch_bounds__(256) resid_norm_kernel(
    float* __restrict__ h, const float* __restrict__ part, int Mp,
    const int* __restrict__ src_rows, const bf16* __restrict__ w, int H, float eps,
    bf16* __restrict__ xn, int write_h) {
  __shared__ float red[8];
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x;
  const int r = src_rows ? src_rows[i] : i;
  const int T = blockDim.x, H4 = H >> 2;
  float4* hr = reinterpret_cast<float4*>(h + static_cast<size_t>(r) * H);
  const size_t slab4 = static_cast<size_t>(Mp) * H4;
  const float4* pr = reinterpret_cast<const float4*>(part + static_cast<size_t>(r) * H);
  float4 x[V];
  float ss = 0.f;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c = threadIdx.x + v * T;
    if (c < H4) {
      float4 p[S > 0 ? S : 1];
#pragma unroll
      for (int z = 0; z < S; ++z) p[z] = pr[z * slab4 + c];
      const float4 hv = hr[c];
      if constexpr (S > 0) {
        float4 acc = p[0];
#pragma unroll
        for (int z = 1; z < S; ++z) {
          acc.x += p[z].x;
          acc.y += p[z].y;
          acc.z += p[z].z;
          acc.w += p[z].w;
        }
        x[v] = make_float4(hv.x + acc.x, hv.y + acc.y, hv.z + acc.z, hv.w + acc.w);
      } else {
        x[v] = hv;
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c = threadIdx.x + v * T;
    if (c < H4) {
      ss = __fmaf_rn(x[v].x, x[v].x, ss);
      ss = __fmaf_rn(x[v].y, x[v].y, ss);
      ss = __fmaf_rn(x[v].z, x[v].z, ss);
      ss = __fmaf_rn(x[v].w, x[v].w, ss);
      if (S > 0 && write_h) hr[c] = x[v];
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int k = 0; k < (T >> 5); ++k) tot += red[k];
  const float inv = rsqrtf(tot / static_cast<float>(H) + eps);
  uint2* orow = reinterpret_cast<uint2*>(xn + static_cast<size_t>(i) * H);
  const uint2* w2 = reinterpret_cast<const uint2*>(w);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c = threadIdx.x + v * T;
    if (c < H4) {
      const uint2 wv = w2[c];
      orow[c] = make_uint2(pack_bf2((x[v].x * inv) * bf_lo(wv.x), (x[v].y * inv) * bf_hi(wv.x)),
                           pack_bf2((x[v].z * inv) * bf_lo(wv.y), (x[v].w * inv) * bf_hi(wv.y)));
    }
  }
}

template <int V>
static int resid_norm_v(float* h, const float* part, int S, int Mp, const int* src_rows, int R,
                        const bf16* w, int H, float eps, bf16* xn, int wh, cudaStream_t st) {
  const int threads = ((H / 4 + V - 1) / V + 31) / 32 * 32;
#define RN_CASE(s)                                                                                 \
  case s:                                                                                          \
    RLB_CUDA(launch_k(resid_norm_kernel<s, V>, dim3(R), dim3(threads), 0, st, h, part, Mp,         \
                      src_rows, w, H, eps, xn, wh));                                               \
    break;
  switch (S) {
    RN_CASE(0) RN_CASE(1) RN_CASE(2) RN_CASE(3) RN_CASE(4) RN_CASE(5) RN_CASE(6) RN_CASE(7)
    RN_CASE(8)
    default: RLB_CHECK(false, RLB_ERR_ARG, "split-K factor must be <= 8");
  }
#undef RN_CASE
  return RLB_OK;
}

int resid_norm_launch(float* h, const float* part, int S, int Mp, const int* src_rows, int R,
                      const bf16* w, int H, float eps, bf16* xn, bool write_h, cudaStream_t st) {
  if (R <= 0) return RLB_OK;
  RLB_CHECK(H % 4 == 0 && H <= 4 * 256 * 4, RLB_ERR_ARG, "hidden size unsupported by RMSNorm");
  const int wh = write_h ? 1 : 0;
  // <= 256 threads, 1 / 2 / 4 float4 groups each (1536 -> 192 x 2, 3584 -> 224 x 4)
  if (H / 4 <= 256) return resid_norm_v<1>(h, part, S, Mp, src_rows, R, w, H, eps, xn, wh, st);
  if (H / 4 <= 512) return resid_norm_v<2>(h, part, S, Mp, src_rows, R, w, H, eps, xn, wh, st);
  return resid_norm_v<4>(h, part, S, Mp, src_rows, R, w, H, eps, xn, wh, st);
}

}  // namespace rlb
