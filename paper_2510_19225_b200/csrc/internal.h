// Internal declarations shared by the librlb translation units.
#pragma once
#include "../../include/rlb.h"
#include "common.cuh"

#include <vector>

namespace rlb {

constexpr int PAGE = 64;      // tokens per KV page

enum Epi { EPI_BF16 = 0, EPI_RESADD = 1, EPI_SWIGLU = 2, EPI_F32 = 3, EPI_ARGMAX = 4,
           EPI_PARTIAL = 5, EPI_ROPE = 6, EPI_SUMRES = 7 };
// Split-K epilogues reduced inside a (1,1,splits) thread-block cluster
// through distributed shared memory (BN = 128): RESADD (h += sum) and ROPE.
constexpr bool cluster_epi(int epi) { return epi == EPI_RESADD || epi == EPI_ROPE; }

// EPI_ROPE destination: q rows, the layer's paged KV cache, RoPE table.
struct RopeDst {
  const int* row_slot;
  const int* row_pos;
  const float2* rope;        // [pos][D/2] (cos, sin)
  bf16* q;
  int ldq;
  bf16* kv;                  // this layer's pages [page][kv_head][K|V][PAGE][D]
  const int* block_table;
  int bt_stride;
  int nq, nkv, d;
  int num_pages = 1 << 30;   // (checked build) page ids must be below it
};

struct GemmParams {
  int M, N, K;
  const bf16* bias;
  void* out;
  int ldo;
  int splits;     // split-K factor (1 = no split)
  float* ws;      // EPI_PARTIAL: fp32 partials [splits][M][N]; EPI_SUMRES: per-CTA
                  // running-sum tiles [CTA][128][256] (out = the fp32 residual h)
  unsigned long long* dbg;  // optional: globaltimer stamps of CTA 0 (latency breakdown)
  RopeDst rope;   // EPI_ROPE only
  int sum_tmem = 0;   // EPI_SUMRES: running sum in TMEM (short splits), else in L2 scratch
};

int make_kmajor_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int box_rows);
int gemm_prepare();  // set smem attributes of every GEMM variant on the current device
int gemm_launch(const CUtensorMap& a, const CUtensorMap& b, int block_n, int epi,
                const GemmParams& p, cudaStream_t st, int block_m = 256, int a_multicast = 1,
                int kps = 1);
int make_kmajor_map3(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int box_rows,
                     int kps);
// The KV pool as rows of head_dim bf16 ([layer][page][kv head][K|V][64 tok])
// in 16-token x head_dim boxes (3D, 128B swizzle) for the decode attention
int make_kv_map(CUtensorMap* map, const void* kv, int64_t rows, int head_dim);
int gemm_launch_pairp(const CUtensorMap& a, const CUtensorMap& b128, int epi, const GemmParams& p,
                      cudaStream_t st);
int pairp_units(int epi, int M, int N, int splits);   // work units of one pair-GEMM launch
size_t pairp_sumres_scratch(int splits);              // EPI_SUMRES scratch (floats)

// ---- elementwise / attention launchers (kernels.cu) ----
struct AttnArgs {
  const bf16* q;  int ldq;          // rotated q rows [R][NQ*D]
  const bf16* kv;                   // layer base [page][NKV][2][PAGE][D]
  const int* block_table; int bt_stride;
  const int* row_slot; const int* row_pos;
  int R, NQ, NKV, D, max_splits;
  float* ws;                        // [R][NQ][max_splits][D+2]
  bf16* out; int ldo;
  // prefill row pairs split by length (row_pairs mode): pair_ids[0, n_short)
  // hold pairs whose rows all have <= 2 pages of context (a 2-warp kernel),
  // pair_ids[n_short, n_short + n_long) the rest; null = every pair, 4 warps
  const int* pair_ids = nullptr;
  int n_short = 0, n_long = 0;
  int pair_off = 0;                 // (set by the launcher) first pair id of a launch
  // prefill rows in groups of 16 consecutive positions of one sequence
  // (first row of each), served per query head by attn_head16_kernel; their
  // pairs are in neither pair list
  const int* head16_ids = nullptr;
  int n_head16 = 0;
  // decode K/V loads through TMA: a 3D tensor map over the whole KV pool
  // (make_kv_map) and this layer's first row in it; null = cp.async
  const CUtensorMap* kv_map = nullptr;
  int64_t kv_row0 = 0;
  int num_pages = 1 << 30;          // (checked build) page ids must be below it
};
int attention_launch(const AttnArgs& a, cudaStream_t st, bool row_pairs = false);
int attention_windows(int max_seq);   // CTA windows per row (AttnArgs.max_splits)
int attention_window_positions();     // positions per CTA window (numerics plan)
int attention_warps();                // warps per attention item (numerics plan)

int embed_launch(const bf16* embed, int H, const int* tok, int R, float* h, cudaStream_t st);
int resid_norm_launch(float* h, const float* part, int S, int Mp, const int* src_rows, int R,
                      const bf16* w, int H, float eps, bf16* xn, bool write_h, cudaStream_t st);
int argmax_append_launch(const float2* part, int ntiles, int L, const int* logit_slot,
                         int32_t* seq_tokens, int32_t* seq_len, const int32_t* seq_target,
                         int max_seq, int32_t* ring, const int32_t* ring_cur, int max_slots,
                         cudaStream_t st);
int decode_prepare_launch(const int* dec_slots, int R, const int32_t* seq_tokens,
                          const int32_t* seq_len, int max_seq, int* row_tok, int* row_pos,
                          int* row_slot, int* logit_src, int* logit_slot, int32_t* ring_ctr,
                          int32_t* ring_cur, cudaStream_t st);
int seed_tokens_launch(const int* row_tok, const int* row_pos, const int* row_slot, int R,
                       int32_t* seq_tokens, int max_seq, cudaStream_t st);
int ring_advance_launch(int32_t* ring_ctr, int32_t* ring_cur, cudaStream_t st);
int gather_seqs_launch(const int* slots, const int64_t* cu, int n, const int32_t* seq_tokens,
                       int max_seq, int32_t* out, cudaStream_t st);

// ---- weight pull (pull.cu) ----
struct Segment { int32_t hf; int64_t src_off, dst_off, bytes; };
void relayout_segments(const rlb_model_cfg& m, std::vector<Segment>* out);
int64_t arena_bytes(const rlb_model_cfg& m);
int32_t hf_count(const rlb_model_cfg& m);
int relayout_copy(const rlb_model_cfg& m, const void* const* hf_ptrs, int32_t n, void* dst,
                  cudaStream_t st);
int copy_bytes(void* dst, const void* src, int64_t nbytes, cudaStream_t st);

}  // namespace rlb
