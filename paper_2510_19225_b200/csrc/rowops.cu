// Row-wise consumers of the split-K projections (K3).  The QKV, O and down
// GEMMs write fp32 partials [S][M][N]; these kernels reduce them in split
// order (z = 0..S-1, the same for every row and every batch composition) and
// fuse the reduction with the work that follows it anyway:
//   qkv_rope    sum + bias -> RoPE(q, k) -> q buffer, K/V into the paged cache
//   resid_norm  h += sum (residual) -> RMSNorm -> bf16 input of the next GEMM
// S is a template parameter so every partial load of a thread is in flight
// at once (the kernels are L2-latency bound otherwise).
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

// x = sum_z part[z][r] + bias (fp32).  q heads: rotated into qout; k heads:
// rotated and written to the slot's KV page; v heads: copied to the page.
// rope[pos][j] = (cos, sin) of pos * theta^(-2j/D).  Thread = rotation pair.
template <int S>
__global__ void __launch_bounds__(256) qkv_rope_kernel(
    const float* __restrict__ part, int Mp, const bf16* __restrict__ bias,
    const int* __restrict__ row_slot, const int* __restrict__ row_pos,
    const float2* __restrict__ rope, int NQ, int NKV, int D, bf16* __restrict__ qout, int ldq,
    bf16* __restrict__ kv, const int* __restrict__ block_table, int bt_stride) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int half = D / 2;
  const int N = (NQ + 2 * NKV) * D;
  const int pos = row_pos[r];
  const int page = block_table[static_cast<size_t>(row_slot[r]) * bt_stride + pos / PAGE];
  const size_t head_stride = static_cast<size_t>(2) * PAGE * D;
  bf16* kv_page = kv + static_cast<size_t>(page) * head_stride * NKV +
                  static_cast<size_t>(pos % PAGE) * D;
  const size_t slab = static_cast<size_t>(Mp) * N;
  const float* pr = part + static_cast<size_t>(r) * N;
  const float2* cs = rope + static_cast<size_t>(pos) * half;
  const int total = (NQ + 2 * NKV) * half;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int head = i / half, j = i % half;
    const int c1 = head * D + j, c2 = c1 + half;
    float p1[S], p2[S];
#pragma unroll
    for (int z = 0; z < S; ++z) {
      p1[z] = pr[z * slab + c1];
      p2[z] = pr[z * slab + c2];
    }
    float x1 = p1[0], x2 = p2[0];
#pragma unroll
    for (int z = 1; z < S; ++z) {
      x1 += p1[z];
      x2 += p2[z];
    }
    x1 += __bfloat162float(bias[c1]);
    x2 += __bfloat162float(bias[c2]);
    if (head < NQ + NKV) {
      const float2 c = cs[j];
      const float y1 = __fmaf_rn(x1, c.x, -x2 * c.y);
      const float y2 = __fmaf_rn(x2, c.x, x1 * c.y);
      bf16* o = head < NQ ? qout + static_cast<size_t>(r) * ldq + head * D
                          : kv_page + static_cast<size_t>(head - NQ) * head_stride;
      o[j] = __float2bfloat16_rn(y1);
      o[j + half] = __float2bfloat16_rn(y2);
    } else {
      bf16* o = kv_page + static_cast<size_t>(head - NQ - NKV) * head_stride +
                static_cast<size_t>(PAGE) * D;
      o[j] = __float2bfloat16_rn(x1);
      o[j + half] = __float2bfloat16_rn(x2);
    }
  }
}

int qkv_rope_launch(const float* part, int S, int Mp, const bf16* bias, const int* row_slot,
                    const int* row_pos, int R, const float2* rope, int NQ, int NKV, int D,
                    bf16* qout, int ldq, bf16* kv, const int* block_table, int bt_stride,
                    cudaStream_t st) {
  if (R <= 0) return RLB_OK;
#define QR_CASE(s)                                                                           \
  case s:                                                                                    \
    RLB_CUDA(launch_k(qkv_rope_kernel<s>, dim3(R), dim3(256), 0, st, part, Mp, bias, row_slot, \
                      row_pos, rope, NQ, NKV, D, qout, ldq, kv, block_table, bt_stride));     \
    break;
  switch (S) {
    QR_CASE(1) QR_CASE(2) QR_CASE(3) QR_CASE(4) QR_CASE(5) QR_CASE(6) QR_CASE(7) QR_CASE(8)
    default: RLB_CHECK(false, RLB_ERR_ARG, "split-K factor must be 1..8");
  }
#undef QR_CASE
  return RLB_OK;
}

}  // namespace rlb
