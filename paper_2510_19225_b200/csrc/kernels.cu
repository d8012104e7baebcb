// K3 small fused kernels, K5 compaction, K6
// response-buffer append.  Every kernel works on "token rows": a row is
// (slot, position, token).  A decode step is one row per executing slot; a
// varlen prefill (initial prompt or migration resume) is many rows per slot.
// Each row's arithmetic depends only on the row's own inputs and its slot's
// KV prefix -- never on which other rows share the launch -- so a sequence
// rebuilt by prefill on another GPU continues bit-identically (SURVEY.md §7
// hard part 2).
#include "internal.h"

namespace rlb {

// -------------------------------------------------------------- embed ----
__global__ void embed_kernel(const bf16* __restrict__ embed, int H, const int* __restrict__ tok,
                             float* __restrict__ h) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const bf16* e = embed + static_cast<size_t>(tok[r]) * H;
  float* o = h + static_cast<size_t>(r) * H;
  for (int i = threadIdx.x; i < H; i += blockDim.x) o[i] = __bfloat162float(e[i]);
}

int embed_launch(const bf16* embed, int H, const int* tok, int R, float* h, cudaStream_t st) {
  if (R <= 0) return RLB_OK;
  RLB_CUDA(launch_k(embed_kernel, dim3(R), dim3(256), 0, st, embed, H, tok, h));
  return RLB_OK;
}


// ---------------------------------------------- argmax + response append --
// Greedy token (lowest index on ties) of each logits row, appended to the
// slot's device sequence buffer (K6) and to this step's row of the token ring
// that the host flushes with one D2H copy.
// Input: per (row, lm_head N-tile) (max, lowest argmax index) partials written
// by the EPI_ARGMAX GEMM epilogue.
__global__ void __launch_bounds__(512) argmax_append_kernel(
    const float2* __restrict__ part, int ntiles, const int* __restrict__ logit_slot,
    int32_t* __restrict__ seq_tokens, int32_t* __restrict__ seq_len,
    const int32_t* __restrict__ seq_target, int max_seq, int32_t* __restrict__ ring,
    const int32_t* __restrict__ ring_cur, int max_slots) {
  __shared__ float sv[16];
  __shared__ int si[16];
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const float2* row = part + static_cast<size_t>(r) * ntiles;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = threadIdx.x; i < ntiles; i += 512) {
    const float2 v = row[i];
    const int vi = __float_as_int(v.y);
    if (v.x > best || (v.x == best && vi < idx)) {
      best = v.x;
      idx = vi;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, off);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
    if (ov > best || (ov == best && oi < idx)) {
      best = ov;
      idx = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < 16; ++k)
      if (sv[k] > best || (sv[k] == best && si[k] < idx)) {
        best = sv[k];
        idx = si[k];
      }
    const int s = logit_slot[r];
    const int len = seq_len[s];
    RLB_DEV_CHECK(s >= 0 && s <= max_slots, "argmax_append: slot");
    if (len < seq_target[s]) {
      RLB_DEV_CHECK(len >= 0 && len < max_seq, "argmax_append: sequence length");
      seq_tokens[static_cast<size_t>(s) * max_seq + len] = idx;
      seq_len[s] = len + 1;
      ring[static_cast<size_t>(*ring_cur) * max_slots + s] = idx;
    }
  }
}

int argmax_append_launch(const float2* part, int ntiles, int L, const int* logit_slot,
                         int32_t* seq_tokens, int32_t* seq_len, const int32_t* seq_target,
                         int max_seq, int32_t* ring, const int32_t* ring_cur, int max_slots,
                         cudaStream_t st) {
  if (L <= 0) return RLB_OK;
  RLB_CUDA(launch_k(argmax_append_kernel, dim3(L), dim3(512), 0, st, part, ntiles, logit_slot,
                    seq_tokens, seq_len, seq_target, max_seq, ring, ring_cur, max_slots));
  return RLB_OK;
}

// ------------------------------------------------------ decode prepare --
__global__ void decode_prepare_kernel(const int* __restrict__ dec_slots, int R,
                                      const int32_t* __restrict__ seq_tokens,
                                      const int32_t* __restrict__ seq_len, int max_seq,
                                      int* row_tok, int* row_pos, int* row_slot, int* logit_src,
                                      int* logit_slot, int32_t* ring_ctr, int32_t* ring_cur) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *ring_cur = (*ring_ctr)++;
  if (i >= R) return;
  const int s = dec_slots[i];
  const int len = seq_len[s];
  RLB_DEV_CHECK(len >= 1 && len <= max_seq, "decode_prepare: sequence length");
  row_tok[i] = seq_tokens[static_cast<size_t>(s) * max_seq + len - 1];
  row_pos[i] = len - 1;
  row_slot[i] = s;
  logit_src[i] = i;
  logit_slot[i] = s;
}

int decode_prepare_launch(const int* dec_slots, int R, const int32_t* seq_tokens,
                          const int32_t* seq_len, int max_seq, int* row_tok, int* row_pos,
                          int* row_slot, int* logit_src, int* logit_slot, int32_t* ring_ctr,
                          int32_t* ring_cur, cudaStream_t st) {
  RLB_CUDA(launch_k(decode_prepare_kernel, dim3((R + 255) / 256), dim3(256), 0, st, dec_slots, R,
                    seq_tokens, seq_len, max_seq, row_tok, row_pos, row_slot, logit_src, logit_slot,
                    ring_ctr, ring_cur));
  return RLB_OK;
}

// Prefill rows carry the request's prompt + prefix ids: copy them into the
// slot's device sequence buffer (the response buffer the decode reads from).
__global__ void seed_tokens_kernel(const int* __restrict__ row_tok, const int* __restrict__ row_pos,
                                   const int* __restrict__ row_slot, int R,
                                   int32_t* __restrict__ seq_tokens, int max_seq) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < R) {
    RLB_DEV_CHECK(row_pos[i] >= 0 && row_pos[i] < max_seq, "seed_tokens: position");
    seq_tokens[static_cast<size_t>(row_slot[i]) * max_seq + row_pos[i]] = row_tok[i];
  }
}

int seed_tokens_launch(const int* row_tok, const int* row_pos, const int* row_slot, int R,
                       int32_t* seq_tokens, int max_seq, cudaStream_t st) {
  if (R <= 0) return RLB_OK;
  RLB_CUDA(launch_k(seed_tokens_kernel, dim3((R + 255) / 256), dim3(256), 0, st, row_tok, row_pos,
                    row_slot, R, seq_tokens, max_seq));
  return RLB_OK;
}

__global__ void ring_advance_kernel(int32_t* ring_ctr, int32_t* ring_cur) {
  pdl_trigger();
  pdl_wait();
  *ring_cur = (*ring_ctr)++;
}

int ring_advance_launch(int32_t* ring_ctr, int32_t* ring_cur, cudaStream_t st) {
  RLB_CUDA(launch_k(ring_advance_kernel, dim3(1), dim3(1), 0, st, ring_ctr, ring_cur));
  return RLB_OK;
}

// ---------------------------------------------------- K5 compaction ------
// Gather each slot's prompt+generated ids into one contiguous varlen buffer
// at the exclusive-scan offsets cu[i].
__global__ void gather_seqs_kernel(const int* __restrict__ slots, const int64_t* __restrict__ cu,
                                   const int32_t* __restrict__ seq_tokens, int max_seq,
                                   int32_t* __restrict__ out) {
  const int i = blockIdx.x;
  const int64_t beg = cu[i], len = cu[i + 1] - cu[i];
  RLB_DEV_CHECK(len >= 0 && len <= max_seq, "gather_seqs: length");
  const int32_t* src = seq_tokens + static_cast<size_t>(slots[i]) * max_seq;
  for (int64_t k = threadIdx.x; k < len; k += blockDim.x) out[beg + k] = src[k];
}

int gather_seqs_launch(const int* slots, const int64_t* cu, int n, const int32_t* seq_tokens,
                       int max_seq, int32_t* out, cudaStream_t st) {
  if (n <= 0) return RLB_OK;
  gather_seqs_kernel<<<n, 256, 0, st>>>(slots, cu, seq_tokens, max_seq, out);
  RLB_CUDA(cudaGetLastError());
  return RLB_OK;
}

}  // namespace rlb
