// The rollout instance: one per GPU, behind the rlb_* C ABI (include/rlb.h).
//
// It replaces the reference's simulated rollout instance -- GenUnit's
// continuous-batching state, the FIFO prefill lane and the analytic decode
// rate (pkg/src/spotrl/sim/engine.py:63-83,699-811,
// pkg/src/spotrl/sim/models.py:39-48) -- with a real Qwen2-shape decoder:
//
//   * requests live in device slots: token buffer [max_slots][max_seq]
//     (prompt + generated = the response buffer, K6), length, target, and a
//     page table into a paged KV pool (64-token pages, allocated for the whole
//     request at admission);
//   * admission runs one varlen prefill (K4) over prompt + prefix tokens of
//     every newly admitted request -- resume after migration is the same call
//     (the `generate{prompt_tokens, prefix_tokens}` message,
//     pkg/src/spotrl/protocol.py:75-81);
//   * a decode step is [prepare rows -> 28 x (RMSNorm, QKV GEMM+bias, RoPE+KV
//     append, split-K paged attention, O GEMM+residual, RMSNorm, gate_up GEMM
//     +SwiGLU, down GEMM+residual) -> final norm -> lm_head -> argmax+append],
//     captured `graph_steps` steps per CUDA graph;
//   * new token ids land in a [steps][slots] ring flushed with one D2H copy per
//     rlb_step call, which the host turns into bulk on_tokens(count=k)
//     (pkg/src/spotrl/manager.py:295-314).
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <unordered_map>

// Programmatic dependent launch per kernel class (1 GEMM, 2 attention, 4 row
// kernels, 8 small kernels), RLB_PDL_MASK (default 11: all but the RMSNorm
// row kernels); RLB_NO_PDL=1 turns it off.  Every kernel waits
// (griddepcontrol.wait) before touching memory its predecessors write; the
// GEMM producer streams its first weight stages before waiting.  Measured on
// B200 (1.5B shape): decode step at 512 rows 3.50 -> 3.37 ms with PDL, tokens
// bit-identical to the non-PDL build; launching the RMSNorms without it (so
// they do not take SM slots while the GEMM before them drains, the GEMM after
// them still launches early) -0.57% decode over 5 A/B pairs
// (scripts/r2_gpu_au.sh, r2_gpu_av.sh).
bool pdl_enabled(int cls) {
  static const int mask = [] {
    const char* off = std::getenv("RLB_NO_PDL");
    if (off && off[0] == '1') return 0;
    const char* m = std::getenv("RLB_PDL_MASK");
    return m ? std::atoi(m) : 11;
  }();
  return (mask & cls) != 0;
}

namespace rlb {

thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

struct Req {
  uint64_t key = 0;
  std::vector<int32_t> tokens;  // prompt + generated (host mirror, exact after each rlb_step)
  int32_t n_prompt = 0;
  int32_t target_len = 0;       // generated tokens at completion (prefix included)
  int32_t slot = -1;
  int32_t reported = 0;         // generated tokens already handed to the caller
  bool prefilled = false;
  int32_t generated() const { return static_cast<int32_t>(tokens.size()) - n_prompt; }
  bool complete() const { return generated() >= target_len; }
};

struct LayerW {
  bf16 *ln1, *wqkv, *bqkv, *wo, *ln2, *wgu, *wdown;
  CUtensorMap m_qkv, m_qkv64, m_qkv64x2, m_o, m_ox2, m_gu, m_gu_small, m_down;
};

// GEMM tile widths per projection (N-tile of the 128 x BN UMMA tile).  A
// forward of at most SMALL_ROWS rows (the rollout tail) runs gate_up and
// lm_head with 128-wide tiles instead: twice the CTAs for the same weight
// stream.  The N tiling does not change any output bit (a row's K loop is
// the same), so batch invariance holds across the switch.
constexpr int BN_QKV = 128, BN_O = 128, BN_GU = 256, BN_DOWN = 128, BN_LM = 256;
constexpr int BN_SMALL = 128;
constexpr int SMALL_ROWS = 256;

// Tile shape of each projection for a forward of R rows.  Measured on B200
// (scripts/gemm_small_m.py): at <= 256 rows 128-row tiles (and for gate_up
// 128-wide N tiles) win, because a 256-row tile half empty still streams the
// same weights through half the CTAs; large prefill chunks want 256-row QKV
// tiles.  None of these choices changes a bit of any row's result.
struct TilePlan {
  int bm_qkv, bm_o, bn_gu, bm_gu, bm_down;
  bool cl_down;   // down: cluster residual add (else fp32 partials + RMSNorm sum)
  int bn_qkv;     // 64 (twice the CTAs, whole RoPE pairs per tile) or 128
};
constexpr int RING_ROWS = 512;

// Split-K factor of an [N, K] projection: the largest divisor d of the K
// blocks with (N-tiles x 2 row tiles of a 512-row decode step) x d <= max_ctas
// and >= 4 K blocks per split.  Depends on the weight shape only.  The short-K
// O projection stops at half the SMs: each extra split adds an fp32 partial
// that the row consumer must read (measured: 100.4k vs 98.7k tok/s for O /
// down splits 3/5 vs 6/5 on config 2).
// Small-batch floor on the split: at one 128-row tile a CTA streams
// N x K x 2 / (N-tiles x S) weight bytes; above ~512 KB per CTA the decode of
// a few rows is bound by too few CTAs (7B o / down / qkv).  Raise S (a divisor
// of the K blocks, <= 8, >= 4 K blocks per split) until it fits.
static int small_batch_splits(int N, int K, int bn, int s0) {
  const int nk = K / 64;
  const double per_tile = 2.0 * N * K / ((N + bn - 1) / bn);
  int s = s0;
  for (int d = s0; d <= 8 && d <= nk / 4; ++d) {
    if (nk % d) continue;
    s = d;
    if (per_tile / d <= 512.0 * 1024) break;
  }
  return std::max(s, s0);
}

static int pick_splits(int N, int K, int bn, int max_ctas) {
  const int nk = K / 64;
  const int tiles = ((N + bn - 1) / bn) * 2;
  int best = 1;
  for (int d = 1; d <= nk; ++d)
    if (nk % d == 0 && nk / d >= 4 && tiles * d <= max_ctas && d <= 8) best = d;
  return best;
}

template <typename T>
static int dalloc(T** p, size_t n) {
  RLB_CUDA(cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
  return RLB_OK;
}

}  // namespace rlb

using namespace rlb;

struct rlb_instance {
  int device = 0;
  rlb_model_cfg m{};
  rlb_engine_cfg e{};
  cudaStream_t st = nullptr;
  int NQ = 0, NKV = 0, D = 0, H = 0, F = 0, V = 0, QKV = 0;
  int max_slots = 0, max_seq = 0, pps = 0, num_pages = 0, max_rows = 0, max_splits = 0;
  int prefill_rows = 0;
  // weights
  uint8_t* arena = nullptr;
  int64_t arena_bytes = 0;
  uint64_t version = 0;
  bool has_weights = false;
  bf16 *embed = nullptr, *norm = nullptr, *lm_head = nullptr;
  std::vector<LayerW> L;
  CUtensorMap m_lm, m_lm_small;
  // double-buffered weights: version v+1 is pulled into
  // the shadow arena on the copy stream while v serves; rlb_swap_weights
  // exchanges the two sets at a step boundary.
  struct WeightSet {
    uint8_t* arena = nullptr;
    uint64_t version = 0;
    bool has = false;
    bf16 *embed = nullptr, *norm = nullptr, *lm_head = nullptr;
    std::vector<LayerW> L;
    CUtensorMap m_lm, m_lm_small;
  } shadow;
  int shadow_state = 0;               // 0 empty, 1 copy enqueued, 2 filled
  bool shadow_timed = false;          // ev_s0/ev_s1 bracket an internal copy
  cudaStream_t st_copy = nullptr;
  cudaEvent_t ev_shadow = nullptr, ev_s0 = nullptr, ev_s1 = nullptr;
  void swap_sets() {
    std::swap(arena, shadow.arena);
    std::swap(version, shadow.version);
    std::swap(has_weights, shadow.has);
    std::swap(embed, shadow.embed);
    std::swap(norm, shadow.norm);
    std::swap(lm_head, shadow.lm_head);
    std::swap(L, shadow.L);
    std::swap(m_lm, shadow.m_lm);
    std::swap(m_lm_small, shadow.m_lm_small);
  }
  int ensure_shadow();
  // KV
  bf16* kv = nullptr;
  size_t layer_stride = 0;  // elements
  int* d_bt = nullptr;
  std::vector<int> h_bt;
  std::vector<int> free_pages;
  // slots
  int32_t *d_seq_tokens = nullptr, *d_seq_len = nullptr, *d_seq_target = nullptr;
  std::vector<int32_t> h_seq_len, h_seq_target;
  std::vector<int> free_slots;
  std::vector<Req*> slot_req;
  bool slots_dirty = true;
  // rows
  int *d_row_tok = nullptr, *d_row_pos = nullptr, *d_row_slot = nullptr, *d_logit_src = nullptr,
      *d_logit_slot = nullptr, *d_dec_slots = nullptr;
  int* h_stage = nullptr;  // pinned: prefill row staging
  size_t stage_cap = 0;
  float* d_h = nullptr;
  bf16 *d_xn = nullptr, *d_qkv = nullptr, *d_q = nullptr, *d_attn = nullptr, *d_act = nullptr;
  float* d_logits = nullptr;
  float* d_ws = nullptr;
  CUtensorMap m_xn, m_attn, m_act;
  CUtensorMap m_xn_x2;    // 3D view of xn: 128-row x 2-K-block boxes (64-column QKV tiles)
  CUtensorMap m_attn_x2;  // 3D view of the attention output (O projection, 128-row tiles)
  bool o_kps2 = true;     // RLB_O_KPS=1: one K block per stage
  int o_partials(const TilePlan& tp, const LayerW& w, int R) {
    if (o_kps2 && tp.bm_o == 128 && BN_O == 128) {
      GemmParams p{R, H, NQ * D, nullptr, nullptr, 0, sp_o < 1 ? 1 : sp_o, d_part};
      p.dbg = d_dbg;
      return gemm_launch(m_attn_x2, w.m_ox2, BN_O, EPI_PARTIAL, p, st, 128, 1, 2);
    }
    return proj(m_attn, w.m_o, BN_O, sp_o, EPI_PARTIAL, R, H, NQ * D, nullptr, nullptr, 0,
                tp.bm_o);
  }
  bool qkv_kps2 = true;   // RLB_QKV_KPS=1: one K block per stage
  int qkv_launch(const TilePlan& tp, const LayerW& w, const GemmParams& pq) {
    // prefill chunks: persistent 2-SM tiles with the same RoPE / KV epilogue
    if ((pairp & 16) && pq.M > 512 && QKV % 256 == 0)
      return gemm_launch_pairp(m_xn, w.m_qkv, EPI_ROPE, pq, st);
    if (tp.bn_qkv == 64 && qkv_kps2)
      return gemm_launch(m_xn_x2, w.m_qkv64x2, 64, EPI_ROPE, pq, st, tp.bm_qkv, 1, 2);
    return gemm_launch(m_xn, tp.bn_qkv == 64 ? w.m_qkv64 : w.m_qkv, tp.bn_qkv, EPI_ROPE, pq, st,
                       tp.bm_qkv);
  }
  int32_t *d_ring = nullptr, *d_ring_ctr = nullptr, *d_ring_cur = nullptr, *h_ring = nullptr;
  // K5 export scratch (rlb_export_partials)
  int* d_exp_slots = nullptr;
  // prefill row pairs split by context length (short: <= 2 pages, 2-warp
  // attention CTAs); set per chunk by admit_and_prefill (RLB_ATTN_SPLIT=0: off)
  int* d_pairs = nullptr;
  int* d_head16 = nullptr;      // first rows of the 16-row prefill runs (K1h)
  std::vector<int> h_head16;
  int head16_n = 0;
  bool attn_head16 = true;      // RLB_ATTN_HEAD16=0: every pair on the pair kernel (A/B)
  // decode attention K/V through TMA boxes of the whole pool (RLB_ATTN_TMA=0
  // at instance creation: per-lane cp.async -- the same bits, the A/B
  // reference of tests/test_gpu_engine.py)
  bool attn_tma = true;
  CUtensorMap kv_map{};
  std::vector<int> h_pairs;
  int pairs_short = 0, pairs_long = 0;
  bool attn_split = true;
  int64_t* d_exp_cu = nullptr;
  int32_t* d_exp_out = nullptr;
  float2* d_rope = nullptr;
  // requests
  std::deque<Req*> pending;
  std::unordered_map<uint64_t, Req*> reqs;
  std::vector<int> dec_list;
  // decode graphs per (rows, weight arena): kernel parameters hold the arena
  std::map<std::pair<int, const uint8_t*>, cudaGraphExec_t> graphs;
  int graph_built_for_version = -1;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evA = nullptr, evB = nullptr;
  // measured decode profile: device time per batch size,
  // from CUDA events around every constant-batch burst of decode steps
  struct ProfAcc {
    int64_t steps = 0;
    double ms = 0.0, ctx_sum = 0.0;   // ctx_sum: sum over steps of the mean context
  };
  std::map<int, ProfAcc> prof;
  struct Burst {
    int R, steps;
    double ctx;
    size_t e0, e1;
  };
  std::vector<Burst> bursts;
  std::vector<cudaEvent_t> burst_ev;
  size_t n_burst_ev = 0;
  int burst_event(size_t* idx) {
    if (n_burst_ev == burst_ev.size()) {
      cudaEvent_t e;
      RLB_CUDA(cudaEventCreate(&e));
      burst_ev.push_back(e);
    }
    *idx = n_burst_ev++;
    RLB_CUDA(cudaEventRecord(burst_ev[*idx], st));
    return RLB_OK;
  }
  int collect_bursts() {   // after the stream has been synchronized
    for (const Burst& b : bursts) {
      float ms = 0.f;
      RLB_CUDA(cudaEventElapsedTime(&ms, burst_ev[b.e0], burst_ev[b.e1]));
      ProfAcc& a = prof[b.R];
      a.steps += b.steps;
      a.ms += ms;
      a.ctx_sum += b.ctx * b.steps;
    }
    bursts.clear();
    n_burst_ev = 0;
    return RLB_OK;
  }
  rlb_stats stats{};
  int last_R = 0;  // rows of the last decode step (for rlb_profile_kernel)
  unsigned long long* d_dbg = nullptr;   // RLB_GEMM_DBG: CTA-0 timestamps of profiled GEMMs
  // split-K factors of the small-N projections: a property of the model
  // shape only (never of M or of the engine config), so every instance of
  // the same model reduces every row identically.
  int sp_qkv = 1, sp_o = 1, sp_down = 1;
  // rows per GEMM CTA: QKV uses 128-row tiles instead of split-K (twice the
  // CTAs, and its RoPE / KV-append epilogue runs straight from TMEM); the
  // others share each weight stage between two 128-row accumulators
  int bm_qkv = 128, bm_o = 128, bm_gu = 256, bm_down = 256;   // decode batch (> 256 rows)
  // persistent 2-SM tiles writing split-K partials for down above the
  // small-batch plans (bit 4) and for O in prefill chunks (bit 8): a third
  // less operand ingress per SM than the single-SM 256 x 128 tiles, same K
  // partition, same bits.  Measured (scripts/pair_splitk.py, 1.5B shape):
  // down at 512 rows 22.0 us (cluster residual add) -> 14.8 us (+ ~2 us in
  // the RMSNorm that sums the 5 partials); prefill chunk of 16k rows: down
  // 492 -> 310 us, O 147 -> 93 us; O at 512 rows gains nothing (8.6 us).
  bool pair_down(int R) const { return (pairp & 4) && R > SMALL_ROWS; }
  bool pair_o(int R) const { return (pairp & 8) && R > 512; }
  int proj_pairp(const CUtensorMap& a, const CUtensorMap& b128, int splits, int R, int N, int K) {
    GemmParams p{R, N, K, nullptr, nullptr, 0, splits, d_part};
    p.dbg = d_dbg;
    return gemm_launch_pairp(a, b128, EPI_PARTIAL, p, st);
  }
  // Prefill chunks: the pair tile's splits summed on its cluster and added
  // into h (EPI_SUMRES) instead of [S][R][H] partial slabs through HBM and a
  // resid_norm that sums them -- the same adds in the same order, so the
  // same bits (RLB_SUMRES=0 / RLB_SUMRES_ROWS=<min rows> for A/B).
  bool sumres_on = true;
  int sumres_rows = 4096;
  size_t part_floats = 0;   // capacity of d_part
  bool use_sumres(int R, int splits) const {
    return sumres_on && R >= sumres_rows && pairp_sumres_scratch(splits) <= part_floats;
  }
  // Splits of <= 1,024 K (O) keep the running sum in TMEM: their MMAs are
  // shorter than the L2 scratch round trips (RLB_SUMRES_TMEM=0/1 overrides).
  int sumres_tmem = -1;
  int proj_sumres(const CUtensorMap& a, const CUtensorMap& b128, int splits, int R, int N, int K) {
    GemmParams p{R, N, K, nullptr, d_h, N, splits, d_part};
    p.sum_tmem = sumres_tmem >= 0 ? sumres_tmem : (K / splits <= 1024 ? 1 : 0);
    return gemm_launch_pairp(a, b128, EPI_SUMRES, p, st);
  }
  int n_sm = 148;
  bool small_gu_wave = true;   // RLB_SMALL_GU_WAVE=0: 128-wide SwiGLU tiles at <= 128 rows
  bool bm_override = false;   // RLB_BM set: the fixed decode-batch tiles below
  // Between 129 and 512 rows each projection takes the first of its tile
  // shapes (smallest first) whose grid fits in one wave of the SMs, else the
  // one with the fewest waves.  Tile shapes never change a row's bits.  For
  // the 1.5B shape this reproduces the measured plans (128 x 64 QKV, 128 x
  // 128 O, 256 x 128 / 256 x 256 SwiGLU); for 7B at 192 rows it moves O and
  // down to 256-row tiles and gate_up to 256 x 256 (one wave of 148 CTAs).
  int pick_tile(int R, const int (*cand)[2], int n, int N, int S, int* bn) const {
    int best = 0, best_w = 1 << 30;
    for (int i = 0; i < n; ++i) {
      const int ctas = ((R + cand[i][0] - 1) / cand[i][0]) * ((N + cand[i][1] - 1) / cand[i][1]) * S;
      const int w = (ctas + n_sm - 1) / n_sm;
      if (w < best_w) {
        best = i;
        best_w = w;
      }
      if (w == 1) break;
    }
    *bn = cand[best][1];
    return cand[best][0];
  }
  TilePlan plan(int R) const {
    const int bnq = sp_qkv == 1 ? bn_qkv_decode : BN_QKV;
    if (R <= 128) {
      // one row tile: SwiGLU on 128-wide tiles, or 256-wide when that is what
      // fits one wave (7B: 296 -> 148 CTAs)
      const int cg1[2][2] = {{128, BN_SMALL}, {128, BN_GU}};
      int bn_gu = BN_SMALL;
      if (!bm_override && small_gu_wave) pick_tile(R, cg1, 2, 2 * F, 1, &bn_gu);
      return {128, 128, bn_gu, 128, 128, cl_down, bnq};
    }
    // prefill chunks: the DSMEM reduction of thousands of split tiles costs
    // more than writing the partials (both sum the splits in the same order)
    if (R > 512) return {256, 256, BN_GU, bm_gu, bm_down, cl_down_large && !pair_down(R), BN_QKV};
    if (bm_override) {
      if (R <= SMALL_ROWS) return {128, 128, BN_SMALL, 256, 128, cl_down, bnq};
      return {bm_qkv, bm_o, BN_GU, bm_gu, bm_down, cl_down && !pair_down(R),
              bm_qkv == 128 ? bnq : BN_QKV};
    }
    const int cq[3][2] = {{128, bnq}, {128, 128}, {256, 128}};
    const int co[2][2] = {{128, BN_O}, {256, BN_O}};
    const int cg[3][2] = {{128, BN_SMALL}, {256, BN_SMALL}, {256, BN_GU}};
    const int cd[2][2] = {{128, BN_DOWN}, {256, BN_DOWN}};
    TilePlan tp{};
    int bn = 0;
    tp.bm_qkv = pick_tile(R, cq, 3, QKV, sp_qkv, &tp.bn_qkv);
    tp.bm_o = pick_tile(R, co, 2, H, sp_o, &bn);
    tp.bm_gu = pick_tile(R, cg, 3, 2 * F, 1, &tp.bn_gu);
    tp.bm_down = pick_tile(R, cd, 2, H, sp_down, &bn);
    tp.cl_down = cl_down && !pair_down(R);
    return tp;
  }
  int bn_qkv_decode = 64;   // RLB_QKV_BN=128 restores 128-column QKV tiles
  bool attn_pairs = true;   // prefill attention on row pairs (RLB_ATTN_PAIRS=0: one row per CTA)
  bool sort_rows = true;    // decode rows in descending context order (RLB_SORT_ROWS=0: slot order)
  // persistent 2-SM tiles (double-buffered TMEM): bit 1 gate_up, bit 2
  // lm_head, bit 4 down, bit 8 O in prefill (RLB_PAIRP).  Default: lm_head
  // (1188 tiles: the epilogues hide behind the next tile's MMAs, 165 -> 121
  // us), down, O in prefill and gate_up in prefill chunks; at a 512-row
  // decode gate_up has ~2 tiles per cluster and gains nothing.  Same bits as
  // the single-SM kernels.
  int pairp = 2 | 4 | 8 | 16;   // + bit 16: QKV (RoPE epilogue) in prefill chunks
  bool pairp_prefill = true;
  bool cl_down_large = false;
  bool last_cl_down = true;   // the last forward's down output is already in h (else the
                              // head sums its partials)
  bool down_summed = true;
  // split-K O / down: sum the splits inside a cluster and add into h in the
  // GEMM epilogue (true), or write fp32 partials that the following RMSNorm
  // kernel sums in split order (false)
  // (measured on B200, 1.5B shape, 512 rows: cluster for down (5 splits),
  // partials for O (3 splits); scripts/sweep_bm.sh)
  bool cl_o = false, cl_down = true;
  int pending_rows = 0;     // partial mode: rows whose last down partials await the head
  float* d_part = nullptr;  // split-K partials [splits][max_rows][H] (partial mode)
  int64_t launches_per_forward(int R_logits) const {
    // embed + first norm + per layer (4 GEMMs, attention [+window combine],
    // 2 norms; the last layer's second one is the head's) + head (norm,
    // lm_head, argmax)
    const int per_layer = 7 + (max_splits > 1 ? 1 : 0);
    return 2 + static_cast<int64_t>(m.layers) * per_layer - 1 + (R_logits > 0 ? 3 : 0);
  }
  int proj(const CUtensorMap& a, const CUtensorMap& b, int bn, int splits, int epi, int R, int N,
           int K, const bf16* bias, void* out, int ldo, int bm = 256);
  // KV target of rlb_profile_kernel's qkv timing (clobbers the last
  // layer's entries of the current positions: only for a throw-away rollout)
  bf16* kv_scratch() const { return kv + layer_stride * (m.layers - 1); }

  ~rlb_instance();
  int init();
  int bind_arena();
  // prefill: rows come grouped by sequence (attention serves row pairs)
  int forward_layers(int R, bool prefill = false);
  int head(int Lrows, bool append);
  int decode_step_launch(int R);
  int admit_and_prefill(int* rows_run);
  int run_decode(int steps, int* steps_run);
  int flush(rlb_token_batch* out);
  int upload_slots();
  bool gs_enabled() const { return e.graph_steps > 0; }
  // decode batch buckets: exact up to 16 rows, then multiples of 16 / 32 / 64
  int decode_bucket(int R) const {
    int b = R;
    if (R > 512) b = (R + 63) / 64 * 64;
    else if (R > 128) b = (R + 31) / 32 * 32;
    else if (R > 16) b = (R + 15) / 16 * 16;
    return std::min(b, (max_slots + 127) / 128 * 128);
  }
  void release(Req* r);
  // row pairs (2p, 2p+1) of a prefill chunk (positions pos[0..n)): those
  // whose rows all see <= 2 pages of context first (2-warp attention CTAs),
  // then the rest in row order; the lists belong to the next forward only
  // row pairs (2p, 2p+1) of a prefill chunk (positions pos[0..n)): those
  // whose rows all see <= 2 pages of context first (2-warp attention CTAs),
  // then the rest in row order; the lists belong to the next forward only
  // Rows in runs of 16 consecutive positions of one sequence go to the
  // head-packed kernel (K1h, one CTA per 16 rows x query head); the other
  // pairs to the pair kernel: short ones (<= 2 pages) first, then the rest.
  int build_pairs(const int* pos, size_t n) {
    pairs_short = pairs_long = head16_n = 0;
    if (!(attn_pairs && attn_split)) return RLB_OK;
    const int np = static_cast<int>((n + 1) / 2);
    h_pairs.resize(np);
    h_head16.clear();
    int lo = 0, hi = np;
    auto run16 = [&](int z) {      // rows 2z .. 2z+15: consecutive positions
      const size_t a0 = 2 * static_cast<size_t>(z);
      if (a0 + 16 > n) return false;
      for (int k = 1; k < 16; ++k)
        if (pos[a0 + k] != pos[a0 + k - 1] + 1) return false;
      return true;
    };
    for (int z = 0; z < np;) {
      if (attn_head16 && run16(z)) {
        h_head16.push_back(2 * z);
        z += 8;
        continue;
      }
      const size_t a0 = 2 * static_cast<size_t>(z);
      const bool short_pair = pos[a0] < 2 * PAGE && (a0 + 1 >= n || pos[a0 + 1] < 2 * PAGE);
      if (short_pair) h_pairs[lo++] = z;
      else h_pairs[--hi] = z;
      ++z;
    }
    std::reverse(h_pairs.begin() + hi, h_pairs.end());   // long pairs in row order
    pairs_short = lo;
    pairs_long = np - hi;
    if (hi > lo) std::copy(h_pairs.begin() + hi, h_pairs.end(), h_pairs.begin() + lo);
    head16_n = static_cast<int>(h_head16.size());
    const int nl = pairs_short + pairs_long;
    if (nl) {
      RLB_CUDA(cudaMemcpyAsync(d_pairs, h_pairs.data(), nl * sizeof(int), cudaMemcpyHostToDevice, st));
      stats.h2d_bytes += static_cast<int64_t>(nl) * 4;
    }
    if (head16_n) {
      RLB_CUDA(cudaMemcpyAsync(d_head16, h_head16.data(), head16_n * sizeof(int),
                               cudaMemcpyHostToDevice, st));
      stats.h2d_bytes += static_cast<int64_t>(head16_n) * 4;
    }
    const int launches = (pairs_short > 0) + (pairs_long > 0) + (head16_n > 0);
    if (launches > 1) stats.kernel_launches += static_cast<int64_t>(m.layers) * (launches - 1);
    return RLB_OK;
  }
};

rlb_instance::~rlb_instance() {
  cudaSetDevice(device);
  if (st) cudaStreamSynchronize(st);
  for (auto& g : graphs) cudaGraphExecDestroy(g.second);
  void* bufs[] = {arena, kv, d_bt, d_seq_tokens, d_seq_len, d_seq_target, d_row_tok, d_row_pos,
                  d_row_slot, d_logit_src, d_logit_slot, d_dec_slots, d_h, d_xn, d_qkv, d_q,
                  d_attn, d_act, d_logits, d_ws, d_ring, d_ring_ctr, d_ring_cur, d_rope,
                  d_part, d_exp_slots, d_exp_cu, d_exp_out, d_pairs, d_head16};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (shadow.arena) cudaFree(shadow.arena);
  if (st_copy) {
    cudaStreamSynchronize(st_copy);
    cudaStreamDestroy(st_copy);
  }
  for (cudaEvent_t ev : {ev_shadow, ev_s0, ev_s1})
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : burst_ev) cudaEventDestroy(ev);
  if (h_stage) cudaFreeHost(h_stage);
  if (h_ring) cudaFreeHost(h_ring);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (evA) cudaEventDestroy(evA);
  if (evB) cudaEventDestroy(evB);
  if (st) cudaStreamDestroy(st);
  for (auto& kv_ : reqs) delete kv_.second;
}

int rlb_instance::init() {
  NQ = m.n_q_heads;
  NKV = m.n_kv_heads;
  D = m.head_dim;
  H = m.hidden;
  F = m.ffn;
  V = m.vocab;
  QKV = (NQ + 2 * NKV) * D;
  RLB_CHECK(D == 64 || D == 128, RLB_ERR_ARG, "head_dim must be 64 or 128");
  RLB_CHECK(NQ % NKV == 0 && NQ / NKV <= 8, RLB_ERR_ARG, "unsupported GQA group");
  RLB_CHECK(H % 64 == 0 && F % 64 == 0 && (NQ * D) % 64 == 0 && V % 16 == 0 && QKV % 128 == 0,
            RLB_ERR_ARG, "model dims not tileable");
  max_slots = e.max_slots;
  max_seq = e.max_seq_len;
  RLB_CHECK(max_slots > 0 && max_seq > 0, RLB_ERR_ARG, "max_slots/max_seq_len must be positive");
  pps = (max_seq + PAGE - 1) / PAGE;
  // default pool: every slot at max_seq_len, + the scratch slot's page
  num_pages = e.num_pages > 0 ? e.num_pages : max_slots * pps + 1;
  max_splits = attention_windows(max_seq);
  const size_t ws_row = static_cast<size_t>(NQ) * max_splits * (D + 2) * sizeof(float);
  const size_t ws_budget = static_cast<size_t>(1) << 30;
  // Prefill chunks of ~1k rows keep the split-K partials of a chunk L2-resident.
  prefill_rows = e.max_prefill_rows > 0 ? e.max_prefill_rows : 1024;
  prefill_rows = static_cast<int>(std::min<size_t>(prefill_rows, ws_budget / ws_row));
  prefill_rows = std::max(prefill_rows, 128);
  max_rows = std::max(prefill_rows, max_slots);
  max_rows = (max_rows + 255) / 256 * 256;
  // QKV is never split: 64-wide RoPE tiles give it its CTAs.  O / down:
  // measured on B200 for the two shapes the configs use (scripts/sweep_bm.sh,
  // scripts/decode_profile.py --shape; splits of 5+ CTAs per cluster stop
  // packing into the GPCs once there are more than ~24 clusters), the
  // rule-based pick for any other shape.
  sp_qkv = 1;
  sp_o = small_batch_splits(H, NQ * D, BN_O, pick_splits(H, NQ * D, BN_O, 74));
  sp_down = small_batch_splits(H, F, BN_DOWN, pick_splits(H, F, BN_DOWN, 148));
  if (H == 1536 && NQ * D == 1536 && F == 8960) {          // Qwen2.5-1.5B
    sp_o = 3;
    sp_down = 5;
  } else if (H == 3584 && NQ * D == 3584 && F == 18944) {  // Qwen2.5-7B
    sp_o = 4;
    sp_down = 4;
  }
  // the numerics plan of the instance config (not process environment):
  // split factors set the reduction order of a row's dot products
  {
    const int ko = NQ * D / 64, kd = F / 64;
    RLB_CHECK(e.split_o >= 0 && e.split_o <= 8 && (e.split_o == 0 || ko >= 4 * e.split_o) &&
                  e.split_down >= 0 && e.split_down <= 8 && (e.split_down == 0 || kd >= 4 * e.split_down),
              RLB_ERR_ARG, "split_o / split_down: 0 (default) or 1..8 splits of >= 4 K blocks");
    if (e.split_o) sp_o = e.split_o;
    if (e.split_down) sp_down = e.split_down;
  }

  if (const char* ov = std::getenv("RLB_CLUSTER")) {   // "o,down[,down_large]" 0/1 (tuning)
    int a = 0, b = 0, c = 0;
    const int n = std::sscanf(ov, "%d,%d,%d", &a, &b, &c);
    if (n >= 2) {
      cl_o = a != 0;
      cl_down = b != 0;
    }
    if (n == 3) cl_down_large = c != 0;
  }
  if (const char* ov = std::getenv("RLB_QKV_BN")) bn_qkv_decode = std::atoi(ov) == 128 ? 128 : 64;
  if (const char* ov = std::getenv("RLB_ATTN_PAIRS")) attn_pairs = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_ATTN_SPLIT")) attn_split = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_ATTN_TMA")) attn_tma = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_ATTN_HEAD16")) attn_head16 = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_QKV_KPS")) qkv_kps2 = std::atoi(ov) == 2;
  if (const char* ov = std::getenv("RLB_O_KPS")) o_kps2 = std::atoi(ov) == 2;
  if (const char* ov = std::getenv("RLB_SMALL_GU_WAVE")) small_gu_wave = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_SORT_ROWS")) sort_rows = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_PAIRP")) pairp = std::atoi(ov);
  if (const char* ov = std::getenv("RLB_PAIRP_PREFILL")) pairp_prefill = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_SUMRES")) sumres_on = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_SUMRES_ROWS")) sumres_rows = std::atoi(ov);
  if (const char* ov = std::getenv("RLB_SUMRES_TMEM")) sumres_tmem = std::atoi(ov) != 0;
  if (const char* ov = std::getenv("RLB_BM")) {   // "qkv,o,gate_up,down" (tuning; process-wide)
    int a = 0, b = 0, c = 0, d = 0;
    if (std::sscanf(ov, "%d,%d,%d,%d", &a, &b, &c, &d) == 4) {
      for (int v : {a, b, c, d}) RLB_CHECK(v == 128 || v == 256, RLB_ERR_ARG, "RLB_BM: 128 or 256");
      bm_override = true;
      bm_qkv = a;
      bm_o = b;
      bm_gu = c;
      bm_down = d;
    }
  }

  RLB_CUDA(cudaSetDevice(device));
  RLB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
  RLB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  {
    // stream-ordered allocations (the pull's chunk lists) keep their memory in
    // the pool instead of returning it to the driver at every synchronize
    cudaMemPool_t pool;
    RLB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = ~0ull;
    RLB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  RLB_CUDA(cudaEventCreate(&ev0));
  RLB_CUDA(cudaEventCreate(&ev1));
  RLB_CUDA(cudaEventCreate(&evA));
  RLB_CUDA(cudaEventCreate(&evB));

  arena_bytes = rlb::arena_bytes(m);
  int rc;
  if ((rc = dalloc(&arena, arena_bytes))) return rc;
  RLB_CUDA(cudaMemset(arena, 0, arena_bytes));
  layer_stride = static_cast<size_t>(num_pages) * NKV * 2 * PAGE * D;
  if ((rc = dalloc(&kv, layer_stride * m.layers))) return rc;
  // zeroed once: pages never written read as zeros (bytewise KV comparisons,
  // compute-sanitizer initcheck)
  RLB_CUDA(cudaMemset(kv, 0, layer_stride * m.layers * sizeof(bf16)));
  if (attn_tma &&
      (rc = make_kv_map(&kv_map, kv, static_cast<int64_t>(layer_stride / D) * m.layers, D)))
    return rc;
  // + one scratch slot (index max_slots): the padding rows of bucketed decode
  // batches -- length 1, target 1, so it never appends; its one page is
  // reserved from the pool
  if ((rc = dalloc(&d_bt, static_cast<size_t>(max_slots + 1) * pps))) return rc;
  h_bt.assign(static_cast<size_t>(max_slots) * pps, 0);
  RLB_CUDA(cudaMemset(d_bt, 0, sizeof(int) * h_bt.size()));
  RLB_CHECK(num_pages >= 2, RLB_ERR_ARG, "KV pool needs at least 2 pages");
  free_pages.resize(num_pages - 1);                    // page num_pages-1: the scratch slot's
  for (int i = 0; i < num_pages - 1; ++i) free_pages[i] = num_pages - 2 - i;
  if ((rc = dalloc(&d_seq_tokens, static_cast<size_t>(max_slots + 1) * max_seq))) return rc;
  if ((rc = dalloc(&d_seq_len, max_slots + 1))) return rc;
  if ((rc = dalloc(&d_seq_target, max_slots + 1))) return rc;
  h_seq_len.assign(max_slots, 1);
  h_seq_target.assign(max_slots, 0);
  slot_req.assign(max_slots, nullptr);
  for (int s = max_slots - 1; s >= 0; --s) free_slots.push_back(s);
  RLB_CUDA(cudaMemset(d_seq_tokens, 0, sizeof(int32_t) * (max_slots + 1) * static_cast<size_t>(max_seq)));
  {
    const int32_t one = 1, scratch_page = num_pages - 1;
    RLB_CUDA(cudaMemcpy(d_seq_len + max_slots, &one, sizeof(int32_t), cudaMemcpyHostToDevice));
    RLB_CUDA(cudaMemcpy(d_seq_target + max_slots, &one, sizeof(int32_t), cudaMemcpyHostToDevice));
    RLB_CUDA(cudaMemset(d_bt + static_cast<size_t>(max_slots) * pps, 0, sizeof(int) * pps));
    RLB_CUDA(cudaMemcpy(d_bt + static_cast<size_t>(max_slots) * pps, &scratch_page, sizeof(int),
                        cudaMemcpyHostToDevice));
  }

  const size_t R = max_rows;
  if ((rc = dalloc(&d_row_tok, R)) || (rc = dalloc(&d_row_pos, R)) || (rc = dalloc(&d_row_slot, R)) ||
      (rc = dalloc(&d_logit_src, R)) || (rc = dalloc(&d_logit_slot, R)) ||
      (rc = dalloc(&d_dec_slots, max_rows)))
    return rc;
  if ((rc = dalloc(&d_h, R * H)) || (rc = dalloc(&d_xn, R * H)) || (rc = dalloc(&d_qkv, R * QKV)) ||
      (rc = dalloc(&d_q, R * NQ * D)) || (rc = dalloc(&d_attn, R * NQ * D)) ||
      (rc = dalloc(&d_act, R * F)))
    return rc;
  RLB_CUDA(cudaMemset(d_xn, 0, R * H * sizeof(bf16)));
  RLB_CUDA(cudaMemset(d_attn, 0, R * NQ * D * sizeof(bf16)));
  RLB_CUDA(cudaMemset(d_act, 0, R * F * sizeof(bf16)));
  const int logit_rows = (max_slots + 127) / 128 * 128;
  if ((rc = dalloc(&d_logits, static_cast<size_t>(logit_rows) * V))) return rc;
  if ((rc = dalloc(&d_ws, R * ws_row / sizeof(float)))) return rc;
  const size_t part = std::max({static_cast<size_t>(sp_o) * H, static_cast<size_t>(sp_down) * H});
  part_floats = part * R;
  // chunks that run the split-sum epilogue need its per-CTA scratch
  if (sumres_on && R >= static_cast<size_t>(sumres_rows))
    part_floats = std::max({part_floats, pairp_sumres_scratch(sp_o), pairp_sumres_scratch(sp_down)});
  if ((rc = dalloc(&d_part, part_floats))) return rc;
  if ((rc = dalloc(&d_ring, static_cast<size_t>(RING_ROWS) * max_slots))) return rc;
  if ((rc = dalloc(&d_pairs, max_rows / 2 + 1))) return rc;
  if ((rc = dalloc(&d_head16, max_rows / 16 + 1))) return rc;
  if ((rc = dalloc(&d_exp_slots, max_slots)) || (rc = dalloc(&d_exp_cu, max_slots + 1)) ||
      (rc = dalloc(&d_exp_out, static_cast<size_t>(max_slots) * max_seq)))
    return rc;
  if ((rc = dalloc(&d_ring_ctr, 1)) || (rc = dalloc(&d_ring_cur, 1))) return rc;
  RLB_CUDA(cudaMemset(d_ring, 0xff, sizeof(int32_t) * RING_ROWS * max_slots));
  RLB_CUDA(cudaMemset(d_ring_ctr, 0, sizeof(int32_t)));
  RLB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_ring),
                          sizeof(int32_t) * RING_ROWS * static_cast<size_t>(max_slots)));
  stage_cap = static_cast<size_t>(max_slots) * max_seq;
  RLB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_stage), sizeof(int) * 5 * stage_cap));

  // RoPE table in double precision, stored fp32 (cos, sin).
  const int half = D / 2;
  std::vector<float2> rope(static_cast<size_t>(max_seq) * half);
  for (int p = 0; p < max_seq; ++p)
    for (int j = 0; j < half; ++j) {
      const double inv = std::pow(static_cast<double>(m.rope_theta), -2.0 * j / D);
      const double a = static_cast<double>(static_cast<float>(p * inv));
      rope[static_cast<size_t>(p) * half + j] = make_float2(static_cast<float>(std::cos(a)),
                                                            static_cast<float>(std::sin(a)));
    }
  if ((rc = dalloc(&d_rope, rope.size()))) return rc;
  RLB_CUDA(cudaMemcpy(d_rope, rope.data(), rope.size() * sizeof(float2), cudaMemcpyHostToDevice));

  if ((rc = gemm_prepare())) return rc;
  if ((rc = make_kmajor_map(&m_xn, d_xn, R, H, 128))) return rc;
  if ((rc = make_kmajor_map3(&m_xn_x2, d_xn, R, H, 128, 2))) return rc;
  if ((rc = make_kmajor_map3(&m_attn_x2, d_attn, R, NQ * D, 128, 2))) return rc;
  if ((rc = make_kmajor_map(&m_attn, d_attn, R, NQ * D, 128))) return rc;
  if ((rc = make_kmajor_map(&m_act, d_act, R, F, 128))) return rc;
  return bind_arena();
}

int rlb_instance::bind_arena() {
  // carve order: paper_2510_19225_b200/shapes.py engine_layout()
  int64_t off = 0;
  auto put = [&](int64_t elems) {
    bf16* p = reinterpret_cast<bf16*>(arena + off);
    off = (off + 2 * elems + 255) / 256 * 256;
    return p;
  };
  embed = put(static_cast<int64_t>(V) * H);
  L.resize(m.layers);
  int rc;
  for (int i = 0; i < m.layers; ++i) {
    LayerW& w = L[i];
    w.ln1 = put(H);
    w.wqkv = put(static_cast<int64_t>(QKV) * H);
    w.bqkv = put(QKV);
    w.wo = put(static_cast<int64_t>(H) * NQ * D);
    w.ln2 = put(H);
    w.wgu = put(static_cast<int64_t>(2) * F * H);
    w.wdown = put(static_cast<int64_t>(H) * F);
    if ((rc = make_kmajor_map(&w.m_qkv, w.wqkv, QKV, H, BN_QKV))) return rc;
    if ((rc = make_kmajor_map(&w.m_qkv64, w.wqkv, QKV, H, 64))) return rc;
    if ((rc = make_kmajor_map3(&w.m_qkv64x2, w.wqkv, QKV, H, 64, 2))) return rc;
    if ((rc = make_kmajor_map3(&w.m_ox2, w.wo, H, NQ * D, BN_O, 2))) return rc;
    if ((rc = make_kmajor_map(&w.m_o, w.wo, H, NQ * D, BN_O))) return rc;
    if ((rc = make_kmajor_map(&w.m_gu, w.wgu, 2 * F, H, BN_GU))) return rc;
    if ((rc = make_kmajor_map(&w.m_gu_small, w.wgu, 2 * F, H, BN_SMALL))) return rc;
    if ((rc = make_kmajor_map(&w.m_down, w.wdown, H, F, BN_DOWN))) return rc;
  }
  norm = put(H);
  lm_head = m.tied ? embed : put(static_cast<int64_t>(V) * H);
  RLB_CHECK(off == arena_bytes, RLB_ERR_STATE, "arena carve mismatch");
  if ((rc = make_kmajor_map(&m_lm_small, lm_head, V, H, BN_SMALL))) return rc;
  return make_kmajor_map(&m_lm, lm_head, V, H, BN_LM);
}

// Allocate and carve the shadow arena on first use (bind_arena works on the
// active members, so the sets are swapped around it).
int rlb_instance::ensure_shadow() {
  if (shadow.arena) return RLB_OK;
  uint8_t* a = nullptr;
  int rc;
  if ((rc = dalloc(&a, arena_bytes))) return rc;
  RLB_CUDA(cudaMemset(a, 0, arena_bytes));
  RLB_CUDA(cudaStreamCreateWithFlags(&st_copy, cudaStreamNonBlocking));
  RLB_CUDA(cudaEventCreateWithFlags(&ev_shadow, cudaEventDisableTiming));
  RLB_CUDA(cudaEventCreate(&ev_s0));
  RLB_CUDA(cudaEventCreate(&ev_s1));
  shadow.arena = a;
  swap_sets();
  rc = bind_arena();
  swap_sets();
  return rc;
}

int rlb_instance::forward_layers(int R, bool prefill) {
  // Per layer:
  //   qkv  GEMM -> [sum + bias + RoPE -> q, K/V into the paged cache] in its
  //               epilogue (EPI_ROPE; splits reduced in a cluster if split)
  //   attention
  //   o    GEMM -> h += sum (EPI_RESADD, cluster) or fp32 partials that
  //               resid_norm sums in split order -> RMSNorm(ln2) -> xn
  //   gate_up GEMM -> SwiGLU -> act
  //   down GEMM -> as o, then RMSNorm(ln1 of the next layer); the last
  //               layer's partials are summed by the head's norm
  int rc;
  if ((rc = embed_launch(embed, H, d_row_tok, R, d_h, st))) return rc;
  if ((rc = resid_norm_launch(d_h, nullptr, 0, R, nullptr, R, L[0].ln1, H, m.rms_eps, d_xn, false,
                              st)))
    return rc;
  const TilePlan tp = plan(R);
  for (int l = 0; l < m.layers; ++l) {
    const LayerW& w = L[l];
    bf16* kv_l = kv + layer_stride * l;
    GemmParams pq{R, QKV, H, w.bqkv, nullptr, 0, sp_qkv, nullptr};
    pq.rope = RopeDst{d_row_slot, d_row_pos, d_rope, d_q, NQ * D, kv_l, d_bt, pps, NQ, NKV, D,
                      num_pages};
    if ((rc = qkv_launch(tp, w, pq))) return rc;
    AttnArgs a{d_q, NQ * D, kv_l, d_bt, pps, d_row_slot, d_row_pos, R, NQ, NKV, D, max_splits,
               d_ws, d_attn, NQ * D};
    a.num_pages = num_pages;
    if (!prefill && attn_tma) {
      a.kv_map = &kv_map;
      a.kv_row0 = static_cast<int64_t>(layer_stride / D) * l;
    }
    if (prefill && attn_pairs && attn_split && pairs_short + pairs_long + head16_n > 0) {
      a.pair_ids = d_pairs;
      a.n_short = pairs_short;
      a.n_long = pairs_long;
      a.head16_ids = d_head16;
      a.n_head16 = head16_n;
    }
    if ((rc = attention_launch(a, st, prefill && attn_pairs))) return rc;
    if (cl_o && !pair_o(R)) {
      if ((rc = proj(m_attn, w.m_o, BN_O, sp_o, EPI_RESADD, R, H, NQ * D, nullptr, d_h, H,
                     tp.bm_o)) ||
          (rc = resid_norm_launch(d_h, nullptr, 0, R, nullptr, R, w.ln2, H, m.rms_eps, d_xn, false,
                                  st)))
        return rc;
    } else if (pair_o(R) && use_sumres(R, sp_o)) {
      if ((rc = proj_sumres(m_attn, w.m_o, sp_o, R, H, NQ * D)) ||
          (rc = resid_norm_launch(d_h, nullptr, 0, R, nullptr, R, w.ln2, H, m.rms_eps, d_xn, false,
                                  st)))
        return rc;
    } else {
      if ((rc = pair_o(R) ? proj_pairp(m_attn, w.m_o, sp_o, R, H, NQ * D)
                          : o_partials(tp, w, R)) ||
          (rc = resid_norm_launch(d_h, d_part, sp_o, R, nullptr, R, w.ln2, H, m.rms_eps, d_xn, true,
                                  st)))
        return rc;
    }
    {
      GemmParams pg{R, 2 * F, H, nullptr, d_act, F, 1, d_part};
      if (((pairp & 1) || (R > 512 && pairp_prefill)) && tp.bn_gu == BN_GU && tp.bm_gu == 256) {
        if ((rc = gemm_launch_pairp(m_xn, w.m_gu_small, EPI_SWIGLU, pg, st))) return rc;
      } else if ((rc = gemm_launch(m_xn, tp.bn_gu == BN_SMALL ? w.m_gu_small : w.m_gu, tp.bn_gu,
                                   EPI_SWIGLU, pg, st, tp.bm_gu))) {
        return rc;
      }
    }
    const bool last = l + 1 == m.layers;
    down_summed = tp.cl_down || (pair_down(R) && use_sumres(R, sp_down));
    if (down_summed && !tp.cl_down) {
      if ((rc = proj_sumres(m_act, w.m_down, sp_down, R, H, F))) return rc;
      if (!last && (rc = resid_norm_launch(d_h, nullptr, 0, R, nullptr, R, L[l + 1].ln1, H,
                                           m.rms_eps, d_xn, false, st)))
        return rc;
    } else if (tp.cl_down) {
      if ((rc = proj(m_act, w.m_down, BN_DOWN, sp_down, EPI_RESADD, R, H, F, nullptr, d_h, H,
                     tp.bm_down)))
        return rc;
      if (!last && (rc = resid_norm_launch(d_h, nullptr, 0, R, nullptr, R, L[l + 1].ln1, H,
                                           m.rms_eps, d_xn, false, st)))
        return rc;
    } else {
      if ((rc = pair_down(R) ? proj_pairp(m_act, w.m_down, sp_down, R, H, F)
                             : proj(m_act, w.m_down, BN_DOWN, sp_down, EPI_PARTIAL, R, H, F,
                                    nullptr, nullptr, 0, tp.bm_down)))
        return rc;
      // the last layer's partials are summed by the head's norm (its rows only)
      if (!last && (rc = resid_norm_launch(d_h, d_part, sp_down, R, nullptr, R, L[l + 1].ln1, H,
                                           m.rms_eps, d_xn, true, st)))
        return rc;
    }
  }
  pending_rows = R;
  last_cl_down = down_summed;
  return RLB_OK;
}

int rlb_instance::proj(const CUtensorMap& a, const CUtensorMap& b, int bn, int splits, int epi,
                       int R, int N, int K, const bf16* bias, void* out, int ldo, int bm) {
  GemmParams p{R, N, K, bias, out, ldo, splits < 1 ? 1 : splits, d_part};
  p.dbg = d_dbg;   // null outside rlb_profile_kernel's RLB_GEMM_DBG breakdown
  return gemm_launch(a, b, bn, epi, p, st, bm);
}

// Final RMSNorm over the rows listed in d_logit_src, lm_head, and (optionally) argmax + append into the
// slots listed in d_logit_slot.  h is not written, so the head can run over
// several row blocks of one forward.
int rlb_instance::head(int Lrows, bool append) {
  if (Lrows <= 0) return RLB_OK;
  int rc;
  if ((rc = resid_norm_launch(d_h, last_cl_down ? nullptr : d_part, last_cl_down ? 0 : sp_down,
                              pending_rows,
                              d_logit_src, Lrows, norm, H, m.rms_eps, d_xn, false, st)))
    return rc;
  if (!append) return proj(m_xn, m_lm, BN_LM, 1, EPI_F32, Lrows, V, H, nullptr, d_logits, V);
  // lm_head: 128 x 128 tiles between 33 and 128 rows (measured), else 256 x 256
  const bool small = Lrows > 32 && Lrows <= 128;
  const int bn = small ? BN_SMALL : BN_LM;
  const int ntiles = (V + bn - 1) / bn;
  if ((pairp & 2) && Lrows > 128) {
    GemmParams pl{Lrows, V, H, nullptr, d_logits, ntiles, 1, d_part};
    if ((rc = gemm_launch_pairp(m_xn, m_lm_small, EPI_ARGMAX, pl, st))) return rc;
  } else if ((rc = proj(m_xn, small ? m_lm_small : m_lm, bn, 1, EPI_ARGMAX, Lrows, V, H, nullptr,
                        d_logits, ntiles, small ? 128 : 256))) {
    return rc;
  }
  return argmax_append_launch(reinterpret_cast<const float2*>(d_logits), ntiles, Lrows,
                              d_logit_slot, d_seq_tokens, d_seq_len, d_seq_target, max_seq, d_ring,
                              d_ring_cur, max_slots, st);
}

int rlb_instance::decode_step_launch(int R) {
  int rc;
  if ((rc = decode_prepare_launch(d_dec_slots, R, d_seq_tokens, d_seq_len, max_seq, d_row_tok,
                                  d_row_pos, d_row_slot, d_logit_src, d_logit_slot, d_ring_ctr,
                                  d_ring_cur, st)))
    return rc;
  if ((rc = forward_layers(R))) return rc;
  return head(R, true);
}

int rlb_instance::upload_slots() {
  if (!slots_dirty) return RLB_OK;
  RLB_CUDA(cudaMemcpyAsync(d_seq_len, h_seq_len.data(), sizeof(int32_t) * max_slots,
                           cudaMemcpyHostToDevice, st));
  RLB_CUDA(cudaMemcpyAsync(d_seq_target, h_seq_target.data(), sizeof(int32_t) * max_slots,
                           cudaMemcpyHostToDevice, st));
  RLB_CUDA(cudaMemcpyAsync(d_bt, h_bt.data(), sizeof(int) * h_bt.size(), cudaMemcpyHostToDevice, st));
  RLB_CUDA(cudaStreamSynchronize(st));  // host vectors are pageable; keep them stable
  stats.h2d_bytes += static_cast<int64_t>(sizeof(int32_t)) * (2 * max_slots + h_bt.size());
  slots_dirty = false;
  return RLB_OK;
}

void rlb_instance::release(Req* r) {
  if (r->slot >= 0) {
    const int s = r->slot;
    const int total = r->n_prompt + r->target_len;
    const int np = (total + PAGE - 1) / PAGE;
    for (int i = 0; i < np; ++i) free_pages.push_back(h_bt[static_cast<size_t>(s) * pps + i]);
    slot_req[s] = nullptr;
    h_seq_len[s] = 1;
    h_seq_target[s] = 0;
    free_slots.push_back(s);
    slots_dirty = true;
    r->slot = -1;
  }
}

// Admit pending requests (FIFO) into free slots, then run the varlen prefill
// over prompt + prefix of every newly admitted request.
int rlb_instance::admit_and_prefill(int* rows_run) {
  *rows_run = 0;
  std::vector<Req*> admitted;
  while (!pending.empty() && !free_slots.empty()) {
    Req* r = pending.front();
    const int total = r->n_prompt + r->target_len;
    const int np = (total + PAGE - 1) / PAGE;
    if (static_cast<int>(free_pages.size()) < np) break;
    pending.pop_front();
    const int s = free_slots.back();
    free_slots.pop_back();
    r->slot = s;
    slot_req[s] = r;
    for (int i = 0; i < np; ++i) {
      h_bt[static_cast<size_t>(s) * pps + i] = free_pages.back();
      free_pages.pop_back();
    }
    h_seq_len[s] = static_cast<int32_t>(r->tokens.size());
    h_seq_target[s] = total;
    slots_dirty = true;
    if (!r->complete()) admitted.push_back(r);
  }
  int rc;
  if ((rc = upload_slots())) return rc;
  if (admitted.empty()) return RLB_OK;

  // rows: (tok, pos, slot); logits for each sequence's last row.
  size_t total_rows = 0;
  for (Req* r : admitted) total_rows += r->tokens.size();
  RLB_CHECK(total_rows <= stage_cap, RLB_ERR_CAPACITY, "prefill staging overflow");
  int* tok = h_stage;
  int* pos = h_stage + stage_cap;
  int* slot = h_stage + 2 * stage_cap;
  int* lsrc = h_stage + 3 * stage_cap;
  int* lslot = h_stage + 4 * stage_cap;
  size_t at = 0;
  for (Req* r : admitted)
    for (size_t i = 0; i < r->tokens.size(); ++i, ++at) {
      tok[at] = r->tokens[i];
      pos[at] = static_cast<int>(i);
      slot[at] = r->slot;
    }
  size_t beg = 0;
  size_t ri = 0;          // request whose rows are being placed
  size_t rrow = 0;        // rows of admitted[ri] already placed
  // every slot gets exactly one first token during the prefill, so all chunks
  // share one ring row
  if ((rc = ring_advance_launch(d_ring_ctr, d_ring_cur, st))) return rc;
  stats.kernel_launches += 1;
  while (beg < total_rows) {
    const size_t n = std::min<size_t>(prefill_rows, total_rows - beg);
    // logits rows: sequences whose last row falls inside [beg, beg+n)
    int nl = 0;
    size_t cursor = beg;
    while (ri < admitted.size()) {
      const size_t left = admitted[ri]->tokens.size() - rrow;
      if (cursor + left <= beg + n) {
        lsrc[beg + nl] = static_cast<int>(cursor + left - 1 - beg);
        lslot[beg + nl] = admitted[ri]->slot;
        ++nl;
        cursor += left;
        ++ri;
        rrow = 0;
      } else {
        rrow += beg + n - cursor;
        break;
      }
    }
    RLB_CUDA(cudaMemcpyAsync(d_row_tok, tok + beg, n * sizeof(int), cudaMemcpyHostToDevice, st));
    RLB_CUDA(cudaMemcpyAsync(d_row_pos, pos + beg, n * sizeof(int), cudaMemcpyHostToDevice, st));
    RLB_CUDA(cudaMemcpyAsync(d_row_slot, slot + beg, n * sizeof(int), cudaMemcpyHostToDevice, st));
    if (nl) {
      RLB_CUDA(cudaMemcpyAsync(d_logit_src, lsrc + beg, nl * sizeof(int), cudaMemcpyHostToDevice, st));
      RLB_CUDA(cudaMemcpyAsync(d_logit_slot, lslot + beg, nl * sizeof(int), cudaMemcpyHostToDevice, st));
    }
    if ((rc = build_pairs(pos + beg, n))) return rc;
    if ((rc = seed_tokens_launch(d_row_tok, d_row_pos, d_row_slot, static_cast<int>(n), d_seq_tokens,
                                 max_seq, st)))
      return rc;
    rc = forward_layers(static_cast<int>(n), true);
    pairs_short = pairs_long = head16_n = 0;   // the lists belong to this chunk only
    if (rc) return rc;
    if ((rc = head(nl, true))) return rc;
    stats.h2d_bytes += static_cast<int64_t>(n) * 12 + static_cast<int64_t>(nl) * 8;
    stats.kernel_launches += 1 + launches_per_forward(nl);
    beg += n;
  }
  stats.prefill_rows += static_cast<int64_t>(total_rows);
  for (Req* r : admitted) r->prefilled = true;
  *rows_run = static_cast<int>(total_rows);
  return RLB_OK;
}

int rlb_instance::run_decode(int steps, int* steps_run) {
  *steps_run = 0;
  int rc;
  while (*steps_run < steps) {
    dec_list.clear();
    int min_left = 1 << 30;
    for (int s = 0; s < max_slots; ++s) {
      Req* r = slot_req[s];
      if (r && r->prefilled && h_seq_len[s] < h_seq_target[s]) {
        dec_list.push_back(s);
        min_left = std::min(min_left, h_seq_target[s] - h_seq_len[s]);
      }
    }
    const int Rreal = static_cast<int>(dec_list.size());
    if (Rreal == 0) break;
    // longest contexts first: the attention grid dispatches rows in order, so
    // the long rows start in the first wave and the last wave is short rows
    // (every row's arithmetic is independent of its position in the batch)
    if (sort_rows)
      std::stable_sort(dec_list.begin(), dec_list.end(),
                       [&](int x, int y) { return h_seq_len[x] > h_seq_len[y]; });
    // bucketed batch: padding rows of the scratch slot (never append, same
    // bits for the real rows) so a shrinking long-tail batch reuses a few
    // captured graphs instead of capturing one per batch size
    const int R = gs_enabled() ? decode_bucket(Rreal) : Rreal;
    dec_list.resize(R, max_slots);
    RLB_CUDA(cudaMemcpyAsync(d_dec_slots, dec_list.data(), R * sizeof(int), cudaMemcpyHostToDevice, st));
    stats.h2d_bytes += static_cast<int64_t>(R) * 4;
    last_R = R;
    const int gs = e.graph_steps;
    // with graphs, a burst runs whole graphs up to the first row's target
    // rounded up: a row at its target recomputes its last position (identical
    // K/V bits) and never appends (argmax_append checks the target) for the
    // rest of that graph, instead of the burst dropping to eager launches
    int burst = std::min(steps - *steps_run,
                         gs > 0 ? (min_left + gs - 1) / gs * gs : min_left);
    const int64_t per_step = 1 + launches_per_forward(R);
    double ctx0 = 0.0;
    for (int i = 0; i < Rreal; ++i) ctx0 += h_seq_len[dec_list[i]];
    Burst rec{Rreal, burst, ctx0 / Rreal + 0.5 * (burst - 1), 0, 0};
    if ((rc = burst_event(&rec.e0))) return rc;
    while (burst > 0) {
      const int k = (gs > 0 && burst >= gs) ? gs : 1;
      stats.decode_steps += k;
      stats.decode_rows += static_cast<int64_t>(k) * Rreal;
      stats.kernel_launches += k * per_step;
      if (gs > 0 && burst >= gs) {
        const auto gkey = std::make_pair(R, static_cast<const uint8_t*>(arena));
        auto it = graphs.find(gkey);
        if (it == graphs.end()) {
          cudaGraph_t g;
          RLB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
          for (int k = 0; k < gs; ++k)
            if ((rc = decode_step_launch(R))) {
              cudaStreamEndCapture(st, &g);
              return rc;
            }
          RLB_CUDA(cudaStreamEndCapture(st, &g));
          cudaGraphExec_t ge;
          RLB_CUDA(cudaGraphInstantiate(&ge, g, 0));
          RLB_CUDA(cudaGraphDestroy(g));
          it = graphs.emplace(gkey, ge).first;
        }
        RLB_CUDA(cudaGraphLaunch(it->second, st));
        burst -= gs;
        *steps_run += gs;
        for (int i = 0; i < Rreal; ++i) {
          const int sl = dec_list[i];
          h_seq_len[sl] = std::min(h_seq_len[sl] + gs, h_seq_target[sl]);
        }
      } else {
        if ((rc = decode_step_launch(R))) return rc;
        burst -= 1;
        *steps_run += 1;
        for (int i = 0; i < Rreal; ++i) {
          const int sl = dec_list[i];
          h_seq_len[sl] = std::min(h_seq_len[sl] + 1, h_seq_target[sl]);
        }
      }
    }
    if ((rc = burst_event(&rec.e1))) return rc;
    bursts.push_back(rec);
  }
  return RLB_OK;
}

// Pull the token ring to the host, extend each request's host mirror and fill
// the caller's batch.  Completed requests free their slot and pages.
int rlb_instance::flush(rlb_token_batch* out) {
  int32_t rows = 0;
  RLB_CUDA(cudaMemcpyAsync(&rows, d_ring_ctr, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RLB_CUDA(cudaStreamSynchronize(st));
  if (rows > 0) {
    RLB_CUDA(cudaMemcpyAsync(h_ring, d_ring, sizeof(int32_t) * rows * static_cast<size_t>(max_slots),
                             cudaMemcpyDeviceToHost, st));
    RLB_CUDA(cudaMemsetAsync(d_ring, 0xff, sizeof(int32_t) * rows * static_cast<size_t>(max_slots), st));
    RLB_CUDA(cudaMemsetAsync(d_ring_ctr, 0, sizeof(int32_t), st));
    RLB_CUDA(cudaStreamSynchronize(st));
    stats.d2h_bytes += 4 + static_cast<int64_t>(rows) * max_slots * 4;
    for (int row = 0; row < rows; ++row) {
      const int32_t* rr = h_ring + static_cast<size_t>(row) * max_slots;
      for (int s = 0; s < max_slots; ++s)
        if (rr[s] >= 0 && slot_req[s]) slot_req[s]->tokens.push_back(rr[s]);
    }
  }
  // the device length is authoritative; keep the mirror equal to it
  for (int s = 0; s < max_slots; ++s)
    if (slot_req[s]) h_seq_len[s] = static_cast<int32_t>(slot_req[s]->tokens.size());
  int n = 0;
  int64_t nt = 0;
  if (out) {
    // capacity first: on failure no request state has changed and the ids
    // stay in the host mirror for a retry with a larger batch
    int need_n = 0;
    int64_t need_t = 0;
    for (int s = 0; s < max_slots; ++s) {
      const Req* r = slot_req[s];
      if (!r) continue;
      const int newc = r->generated() - r->reported;
      if (newc <= 0 && !r->complete()) continue;
      ++need_n;
      need_t += newc;
    }
    RLB_CHECK(need_n <= out->cap_entries && need_t <= out->cap_tokens, RLB_ERR_CAPACITY,
              "token batch capacity exceeded (" + std::to_string(need_n) + " entries, " +
                  std::to_string(need_t) + " tokens)");
  }
  std::vector<Req*> finished;
  for (int s = 0; s < max_slots; ++s) {
    Req* r = slot_req[s];
    if (!r) continue;
    const int newc = r->generated() - r->reported;
    const bool done = r->complete();
    if (newc <= 0 && !done) continue;
    if (out) {
      out->keys[n] = r->key;
      out->counts[n] = newc;
      out->done[n] = done ? 1 : 0;
      std::memcpy(out->tokens + nt, r->tokens.data() + r->n_prompt + r->reported,
                  sizeof(int32_t) * newc);
    }
    ++n;
    nt += newc;
    r->reported += newc;
    if (done) finished.push_back(r);
  }
  for (Req* r : finished) {
    release(r);
    reqs.erase(r->key);
    delete r;
  }
  if (out) {
    out->n_entries = n;
    out->n_tokens = nt;
  }
  return RLB_OK;
}

// ====================================================================== C ABI

extern "C" {

const char* rlb_last_error(void) { return g_err.c_str(); }

int rlb_instance_create(int device, const rlb_model_cfg* model, const rlb_engine_cfg* engine,
                        rlb_instance** out) {
  RLB_CHECK(model && engine && out, RLB_ERR_ARG, "null argument");
  rlb_instance* h = new rlb_instance();
  h->device = device;
  h->m = *model;
  h->e = *engine;
  const int rc = h->init();
  if (rc) {
    const std::string msg = g_err;
    delete h;
    g_err = msg;
    return rc;
  }
  *out = h;
  return RLB_OK;
}

int rlb_instance_destroy(rlb_instance* h) {
  delete h;
  return RLB_OK;
}

int rlb_kv_pool(rlb_instance* h, void** base, int64_t* bytes) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  if (base) *base = h->kv;
  if (bytes) *bytes = static_cast<int64_t>(h->layer_stride * h->m.layers * sizeof(bf16));
  return RLB_OK;
}

int32_t rlb_numerics_plan(const rlb_instance* h, int32_t* out, int32_t cap) {
  if (!h) return 0;
  const int32_t plan[8] = {2, h->sp_qkv, h->sp_o, h->sp_down, attention_window_positions(),
                           attention_warps(), PAGE, 0};
  for (int i = 0; i < 8 && i < cap && out; ++i) out[i] = plan[i];
  return 8;
}

int rlb_load_weights(rlb_instance* h, const void* const* hf_ptrs, int32_t n_tensors,
                     uint64_t version, void* ready_event, rlb_pull_stats* stats) {
  RLB_CHECK(h && hf_ptrs, RLB_ERR_ARG, "null argument");
  RLB_CHECK(!h->has_weights || version >= h->version, RLB_ERR_ARG,
            "weight version " + std::to_string(version) + " < " + std::to_string(h->version));
  RLB_CHECK(h->reqs.empty(), RLB_ERR_STATE,
            "active weights replaced only at a step boundary (" + std::to_string(h->reqs.size()) +
                " requests on the instance; pull into the shadow arena and swap)");
  RLB_CUDA(cudaSetDevice(h->device));
  if (ready_event) RLB_CUDA(cudaStreamWaitEvent(h->st, static_cast<cudaEvent_t>(ready_event), 0));
  RLB_CUDA(cudaEventRecord(h->ev0, h->st));
  int rc = relayout_copy(h->m, hf_ptrs, n_tensors, h->arena, h->st);
  if (rc) return rc;
  RLB_CUDA(cudaEventRecord(h->ev1, h->st));
  RLB_CUDA(cudaEventSynchronize(h->ev1));
  float ms = 0.f;
  RLB_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (stats) {
    stats->bytes = h->arena_bytes;
    int64_t moved = 0;
    std::vector<Segment> segs;
    relayout_segments(h->m, &segs);
    for (const Segment& s : segs) moved += s.bytes;
    stats->bytes = moved;
    stats->seconds = ms * 1e-3;
  }
  h->version = version;
  h->has_weights = true;
  return RLB_OK;
}

int rlb_weights_arena(rlb_instance* h, void** arena, int64_t* bytes) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  if (arena) *arena = h->arena;
  if (bytes) *bytes = h->arena_bytes;
  return RLB_OK;
}

int rlb_mark_weights(rlb_instance* h, uint64_t version) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  RLB_CHECK(h->reqs.empty(), RLB_ERR_STATE,
            "active weights replaced only at a step boundary (" + std::to_string(h->reqs.size()) +
                " requests on the instance)");
  RLB_CHECK(!h->has_weights || version >= h->version, RLB_ERR_ARG,
            "weight version " + std::to_string(version) + " < " + std::to_string(h->version));
  h->version = version;
  h->has_weights = true;
  return RLB_OK;
}

// ---- double-buffered weights ---------------------------------------------

int rlb_shadow_arena(rlb_instance* h, void** arena, int64_t* bytes) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  RLB_CUDA(cudaSetDevice(h->device));
  int rc = h->ensure_shadow();
  if (rc) return rc;
  if (arena) *arena = h->shadow.arena;
  if (bytes) *bytes = h->arena_bytes;
  return RLB_OK;
}

int rlb_load_shadow(rlb_instance* h, const void* const* hf_ptrs, int32_t n_tensors,
                    uint64_t version, void* ready_event) {
  RLB_CHECK(h && hf_ptrs, RLB_ERR_ARG, "null argument");
  RLB_CHECK(!h->has_weights || version >= h->version, RLB_ERR_ARG,
            "weight version " + std::to_string(version) + " < " + std::to_string(h->version));
  RLB_CUDA(cudaSetDevice(h->device));
  int rc = h->ensure_shadow();
  if (rc) return rc;
  // the previous fill of this arena (if any) and every decode step that read
  // it as the active set are ordered before the overwrite
  RLB_CUDA(cudaEventRecord(h->ev_shadow, h->st));
  RLB_CUDA(cudaStreamWaitEvent(h->st_copy, h->ev_shadow, 0));
  if (ready_event)      // the producer finished writing the source tensors
    RLB_CUDA(cudaStreamWaitEvent(h->st_copy, static_cast<cudaEvent_t>(ready_event), 0));
  RLB_CUDA(cudaEventRecord(h->ev_s0, h->st_copy));
  if ((rc = relayout_copy(h->m, hf_ptrs, n_tensors, h->shadow.arena, h->st_copy))) return rc;
  RLB_CUDA(cudaEventRecord(h->ev_s1, h->st_copy));
  RLB_CUDA(cudaEventRecord(h->ev_shadow, h->st_copy));
  h->shadow.version = version;
  h->shadow.has = true;
  h->shadow_state = 1;
  h->shadow_timed = true;
  return RLB_OK;
}

int rlb_mark_shadow(rlb_instance* h, uint64_t version, void* stream) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  RLB_CHECK(h->shadow.arena, RLB_ERR_STATE, "no shadow arena (rlb_shadow_arena first)");
  RLB_CHECK(!h->has_weights || version >= h->version, RLB_ERR_ARG,
            "weight version " + std::to_string(version) + " < " + std::to_string(h->version));
  RLB_CUDA(cudaSetDevice(h->device));
  RLB_CUDA(cudaEventRecord(h->ev_shadow, static_cast<cudaStream_t>(stream)));
  h->shadow.version = version;
  h->shadow.has = true;
  h->shadow_state = 1;
  h->shadow_timed = false;
  return RLB_OK;
}

int rlb_shadow_status(rlb_instance* h, uint64_t* version, int32_t* state, double* seconds) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  if (h->shadow_state == 1) {
    RLB_CUDA(cudaSetDevice(h->device));
    const cudaError_t q = cudaEventQuery(h->ev_shadow);
    if (q == cudaSuccess) h->shadow_state = 2;
    else if (q != cudaErrorNotReady) RLB_CUDA(q);
  }
  if (version) *version = h->shadow.version;
  if (state) *state = h->shadow_state;
  if (seconds) {
    *seconds = 0.0;
    if (h->shadow_state == 2 && h->shadow_timed) {
      float ms = 0.f;
      RLB_CUDA(cudaEventElapsedTime(&ms, h->ev_s0, h->ev_s1));
      *seconds = ms * 1e-3;
    }
  }
  return RLB_OK;
}

int rlb_swap_weights(rlb_instance* h, uint64_t* version) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  RLB_CHECK(h->shadow.has && h->shadow_state > 0, RLB_ERR_STATE, "shadow arena holds no weights");
  RLB_CHECK(h->reqs.empty(), RLB_ERR_STATE,
            "weights swap only at a step boundary (" + std::to_string(h->reqs.size()) +
                " requests on the instance)");
  RLB_CUDA(cudaSetDevice(h->device));
  // the copy finishes before any later kernel on the compute stream runs;
  // the host does not wait
  RLB_CUDA(cudaStreamWaitEvent(h->st, h->ev_shadow, 0));
  h->swap_sets();
  h->shadow.has = false;              // the old set is free for the next pull
  h->shadow_state = 0;
  if (version) *version = h->version;
  return RLB_OK;
}

static int submit_one(rlb_instance* h, uint64_t key, const int32_t* toks, int32_t n_prompt,
                      int32_t n_total, int32_t target_len) {
  RLB_CHECK(n_prompt >= 1, RLB_ERR_ARG, "empty prompt");
  RLB_CHECK(target_len >= 1 && n_total - n_prompt <= target_len, RLB_ERR_ARG,
            "prefix longer than target_len");
  RLB_CHECK(n_prompt + target_len <= h->max_seq, RLB_ERR_CAPACITY,
            "prompt + target_len exceeds max_seq_len");
  RLB_CHECK(h->reqs.find(key) == h->reqs.end(), RLB_ERR_STATE,
            "duplicate request key " + std::to_string(key));
  for (int32_t i = 0; i < n_total; ++i)
    RLB_CHECK(toks[i] >= 0 && toks[i] < h->V, RLB_ERR_ARG, "token id out of vocabulary");
  Req* r = new Req();
  r->key = key;
  r->tokens.assign(toks, toks + n_total);
  r->n_prompt = n_prompt;
  r->target_len = target_len;
  r->reported = n_total - n_prompt;  // the prefix is already known to the caller
  h->reqs[key] = r;
  h->pending.push_back(r);
  return RLB_OK;
}

int rlb_submit(rlb_instance* h, uint64_t key, const int32_t* prompt, int32_t n_prompt,
               const int32_t* prefix, int32_t n_prefix, int32_t target_len) {
  RLB_CHECK(h && prompt && (n_prefix == 0 || prefix), RLB_ERR_ARG, "null argument");
  std::vector<int32_t> all(prompt, prompt + n_prompt);
  if (n_prefix > 0) all.insert(all.end(), prefix, prefix + n_prefix);
  return submit_one(h, key, all.data(), n_prompt, n_prompt + n_prefix, target_len);
}

int rlb_submit_varlen(rlb_instance* h, int32_t n, const uint64_t* keys, const int32_t* tokens,
                      const int64_t* cu_lens, const int32_t* n_prompt, const int32_t* target_len) {
  RLB_CHECK(h && keys && tokens && cu_lens && n_prompt && target_len, RLB_ERR_ARG, "null argument");
  for (int32_t i = 0; i < n; ++i) {
    const int rc = submit_one(h, keys[i], tokens + cu_lens[i], n_prompt[i],
                              static_cast<int32_t>(cu_lens[i + 1] - cu_lens[i]), target_len[i]);
    if (rc) return rc;
  }
  return RLB_OK;
}

int rlb_step(rlb_instance* h, int32_t n_steps, rlb_token_batch* out) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  RLB_CHECK(h->has_weights, RLB_ERR_STATE, "no weights loaded");
  RLB_CUDA(cudaSetDevice(h->device));
  int rows = 0, steps = 0, rc;
  RLB_CUDA(cudaEventRecord(h->evA, h->st));
  if ((rc = h->admit_and_prefill(&rows))) return rc;
  RLB_CUDA(cudaEventRecord(h->evB, h->st));
  const int max_steps = RING_ROWS - 1 - (rows + h->prefill_rows - 1) / h->prefill_rows;
  if ((rc = h->run_decode(std::min<int>(std::max(n_steps, 0), max_steps), &steps))) return rc;
  RLB_CUDA(cudaEventRecord(h->ev1, h->st));
  if ((rc = h->flush(out))) return rc;
  if ((rc = h->collect_bursts())) return rc;
  float ms_pre = 0.f, ms_dec = 0.f;
  RLB_CUDA(cudaEventElapsedTime(&ms_pre, h->evA, h->evB));
  RLB_CUDA(cudaEventElapsedTime(&ms_dec, h->evB, h->ev1));
  if (rows > 0) h->stats.prefill_ms += ms_pre;
  if (steps > 0) h->stats.decode_ms += ms_dec;
  if (out) {
    out->steps_run = steps;
    out->prefill_rows = rows;
  }
  return RLB_OK;
}

int rlb_decode_profile(rlb_instance* h, int32_t cap, int32_t* batch, int64_t* steps,
                       double* seconds, double* ctx_mean, int32_t* n_out, int32_t reset) {
  RLB_CHECK(h && n_out, RLB_ERR_ARG, "null argument");
  const int n = static_cast<int>(h->prof.size());
  RLB_CHECK(n <= cap || !(batch || steps || seconds || ctx_mean), RLB_ERR_CAPACITY,
            "decode profile has " + std::to_string(n) + " batch sizes");
  int i = 0;
  for (const auto& kv : h->prof) {
    if (batch) batch[i] = kv.first;
    if (steps) steps[i] = kv.second.steps;
    if (seconds) seconds[i] = kv.second.ms * 1e-3;
    if (ctx_mean) ctx_mean[i] = kv.second.steps ? kv.second.ctx_sum / kv.second.steps : 0.0;
    ++i;
  }
  *n_out = n;
  if (reset) h->prof.clear();
  return RLB_OK;
}

int rlb_cancel(rlb_instance* h, uint64_t key, int32_t* out_tokens, int32_t cap, int32_t* out_len) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  auto it = h->reqs.find(key);
  RLB_CHECK(it != h->reqs.end(), RLB_ERR_STATE, "unknown request key " + std::to_string(key));
  Req* r = it->second;
  const int gen = r->generated();
  if (out_len) *out_len = gen;
  if (out_tokens) {
    RLB_CHECK(gen <= cap, RLB_ERR_CAPACITY, "cancel output capacity");
    std::memcpy(out_tokens, r->tokens.data() + r->n_prompt, sizeof(int32_t) * gen);
  }
  if (r->slot < 0) {
    for (auto p = h->pending.begin(); p != h->pending.end(); ++p)
      if (*p == r) {
        h->pending.erase(p);
        break;
      }
  }
  h->release(r);
  h->reqs.erase(it);
  delete r;
  return RLB_OK;
}

int rlb_export_partials(rlb_instance* h, int32_t n, const uint64_t* keys, int32_t* out_tokens,
                        int64_t cap, int64_t* out_cu_lens, int32_t* out_n_prompt) {
  RLB_CHECK(h && keys && out_tokens && out_cu_lens, RLB_ERR_ARG, "null argument");
  RLB_CUDA(cudaSetDevice(h->device));
  std::vector<Req*> rs(n);
  std::vector<int64_t> cu(n + 1, 0);
  for (int32_t i = 0; i < n; ++i) {
    auto it = h->reqs.find(keys[i]);
    RLB_CHECK(it != h->reqs.end(), RLB_ERR_STATE, "unknown request key " + std::to_string(keys[i]));
    rs[i] = it->second;
    cu[i + 1] = cu[i] + static_cast<int64_t>(rs[i]->tokens.size());
    if (out_n_prompt) out_n_prompt[i] = rs[i]->n_prompt;
  }
  RLB_CHECK(cu[n] <= cap, RLB_ERR_CAPACITY, "export output capacity");
  std::memcpy(out_cu_lens, cu.data(), sizeof(int64_t) * (n + 1));
  // device-resident sequences: one gather kernel into a contiguous buffer
  std::vector<int> dslots;
  std::vector<int64_t> dcu(1, 0);
  std::vector<int32_t> didx;
  for (int32_t i = 0; i < n; ++i) {
    if (rs[i]->slot >= 0) {
      dslots.push_back(rs[i]->slot);
      dcu.push_back(dcu.back() + static_cast<int64_t>(rs[i]->tokens.size()));
      didx.push_back(i);
    } else {
      std::memcpy(out_tokens + cu[i], rs[i]->tokens.data(), sizeof(int32_t) * rs[i]->tokens.size());
    }
  }
  if (!dslots.empty()) {
    // persistent device scratch + the pinned staging buffer: no allocation on
    // the migration path
    const int nd = static_cast<int>(dslots.size());
    RLB_CHECK(dcu.back() <= static_cast<int64_t>(h->stage_cap), RLB_ERR_CAPACITY,
              "export exceeds the staging buffer");
    RLB_CUDA(cudaMemcpyAsync(h->d_exp_slots, dslots.data(), nd * sizeof(int), cudaMemcpyHostToDevice,
                             h->st));
    RLB_CUDA(cudaMemcpyAsync(h->d_exp_cu, dcu.data(), (nd + 1) * sizeof(int64_t),
                             cudaMemcpyHostToDevice, h->st));
    int rc = gather_seqs_launch(h->d_exp_slots, h->d_exp_cu, nd, h->d_seq_tokens, h->max_seq,
                                h->d_exp_out, h->st);
    if (rc) return rc;
    RLB_CUDA(cudaMemcpyAsync(h->h_stage, h->d_exp_out, dcu.back() * 4, cudaMemcpyDeviceToHost, h->st));
    RLB_CUDA(cudaStreamSynchronize(h->st));
    for (int k = 0; k < nd; ++k) {
      const int i = didx[k];
      std::memcpy(out_tokens + cu[i], h->h_stage + dcu[k], sizeof(int32_t) * (dcu[k + 1] - dcu[k]));
    }
  }
  return RLB_OK;
}

int rlb_status(rlb_instance* h, int32_t* m_pending, int32_t* m_exec, uint64_t* weight_version) {
  RLB_CHECK(h, RLB_ERR_ARG, "null handle");
  if (m_pending) *m_pending = static_cast<int32_t>(h->pending.size());
  if (m_exec) *m_exec = static_cast<int32_t>(h->reqs.size() - h->pending.size());
  if (weight_version) *weight_version = h->version;
  return RLB_OK;
}

int rlb_get_stats(rlb_instance* h, rlb_stats* out, int32_t reset) {
  RLB_CHECK(h && out, RLB_ERR_ARG, "null argument");
  *out = h->stats;
  if (reset) h->stats = rlb_stats{};
  return RLB_OK;
}

int rlb_profile_kernel(rlb_instance* h, int32_t which, int32_t iters, double* avg_ms,
                       double* work_per_launch) {
  RLB_CHECK(h && avg_ms && work_per_launch && iters > 0, RLB_ERR_ARG, "bad argument");
  RLB_CHECK(h->last_R > 0, RLB_ERR_STATE, "no decode step has run yet");
  RLB_CUDA(cudaSetDevice(h->device));
  const int R = h->last_R;
  const LayerW& w = h->L[0];
  const int NQ = h->NQ, D = h->D, H = h->H, F = h->F;
  double work = 0.0;
  const TilePlan tp = h->plan(R);
  auto launch = [&]() -> int {
    switch (which) {
      case 0: {
        AttnArgs a{h->d_q, NQ * D, h->kv, h->d_bt, h->pps, h->d_row_slot, h->d_row_pos, R, NQ,
                   h->NKV, D, h->max_splits, h->d_ws, h->d_attn, NQ * D};
        if (h->attn_tma) a.kv_map = &h->kv_map;     // layer 0: kv_row0 = 0
        return attention_launch(a, h->st);
      }
      // projections with their fused epilogues, outputs to scratch where the
      // product writes state (fp32 h -> the partial workspace; qkv's K/V go
      // to the last layer's pages: timing only, the rollout that was
      // profiled is discarded)
      case 1: return h->proj(h->m_xn, tp.bn_gu == BN_SMALL ? w.m_gu_small : w.m_gu, tp.bn_gu, 1,
                             EPI_SWIGLU, R, 2 * F, H, nullptr, h->d_act, F, tp.bm_gu);
      case 2:
        if (h->pair_down(R)) return h->proj_pairp(h->m_act, w.m_down, h->sp_down, R, H, F);
        return h->proj(h->m_act, w.m_down, BN_DOWN, h->sp_down,
                       tp.cl_down ? EPI_RESADD : EPI_PARTIAL, R, H, F, nullptr, h->d_part, H,
                       tp.bm_down);
      case 3: {
        GemmParams pq{R, h->QKV, H, w.bqkv, nullptr, 0, h->sp_qkv, nullptr};
        pq.rope = RopeDst{h->d_row_slot, h->d_row_pos, h->d_rope, h->d_q, NQ * D, h->kv_scratch(),
                          h->d_bt, h->pps, NQ, h->NKV, D};
        pq.dbg = h->d_dbg;
        return h->qkv_launch(tp, w, pq);
      }
      case 4:
        if (h->pair_o(R)) return h->proj_pairp(h->m_attn, w.m_o, h->sp_o, R, H, NQ * D);
        if (!h->cl_o) return h->o_partials(tp, w, R);
        return h->proj(h->m_attn, w.m_o, BN_O, h->sp_o, h->cl_o ? EPI_RESADD : EPI_PARTIAL,
                       R, H, NQ * D, nullptr, h->d_part, H, tp.bm_o);
      case 5: {
        if ((h->pairp & 2) && R > 128) {
          GemmParams pl{R, h->V, H, nullptr, h->d_logits, (h->V + BN_LM - 1) / BN_LM, 1, h->d_part};
          return gemm_launch_pairp(h->m_xn, h->m_lm_small, EPI_ARGMAX, pl, h->st);
        }
        return h->proj(h->m_xn, h->m_lm, BN_LM, 1, EPI_ARGMAX, R, h->V, H, nullptr, h->d_logits,
                       (h->V + BN_LM - 1) / BN_LM);
      }
      case 6: return resid_norm_launch(h->d_h, tp.cl_down ? nullptr : h->d_part,
                                       tp.cl_down ? 0 : h->sp_down, R, nullptr, R, w.ln2, H,
                                       h->m.rms_eps, h->d_xn, false, h->st);
    }
    set_error("unknown kernel id");
    return RLB_ERR_ARG;
  };
  switch (which) {
    case 0: {  // K and V of every row's context, q in, attention out (bf16)
      std::vector<int> rows(R);
      RLB_CUDA(cudaMemcpy(rows.data(), h->d_row_pos, 4 * R, cudaMemcpyDeviceToHost));
      double ctx = 0;
      for (int i = 0; i < R; ++i) ctx += rows[i] + 1;
      work = ctx * h->NKV * 2.0 * D * 2.0 + 2.0 * R * NQ * D * 2.0;
      break;
    }
    case 1: work = 2.0 * R * 2.0 * F * H; break;
    case 2: work = 2.0 * R * H * F; break;
    case 3: work = 2.0 * R * h->QKV * H; break;
    case 4: work = 2.0 * R * H * NQ * D; break;
    case 5: work = 2.0 * R * h->V * static_cast<double>(H); break;
    case 6: work = R * H * (4.0 * (tp.cl_down ? 1 : 1 + h->sp_down) + 2.0); break;  // bytes
    default: RLB_CHECK(false, RLB_ERR_ARG, "unknown kernel id");
  }
  int rc = launch();  // warm
  if (rc) return rc;
  if (std::getenv("RLB_GEMM_DBG") && which >= 1 && which <= 5) {   // latency breakdown, 1 launch
    if (!h->d_dbg) RLB_CUDA(cudaMalloc(&h->d_dbg, 8 * sizeof(unsigned long long)));
    RLB_CUDA(cudaMemsetAsync(h->d_dbg, 0, 8 * sizeof(unsigned long long), h->st));
    if ((rc = launch())) return rc;
    unsigned long long t[8];
    RLB_CUDA(cudaMemcpyAsync(t, h->d_dbg, sizeof(t), cudaMemcpyDeviceToHost, h->st));
    RLB_CUDA(cudaStreamSynchronize(h->st));
    std::fprintf(stderr, "kernel %d dbg (ns from CTA start): setup %lld wait %lld mma_done %lld "
                 "epi_start %lld epi_end %lld dealloc %lld\n", which,
                 (long long)(t[1] - t[0]), (long long)(t[2] - t[0]), (long long)(t[3] - t[0]),
                 (long long)(t[4] - t[0]), (long long)(t[6] - t[0]), (long long)(t[5] - t[0]));
    RLB_CUDA(cudaFree(h->d_dbg));
    h->d_dbg = nullptr;
  }
  RLB_CUDA(cudaEventRecord(h->ev0, h->st));
  for (int i = 0; i < iters; ++i)
    if ((rc = launch())) return rc;
  RLB_CUDA(cudaEventRecord(h->ev1, h->st));
  RLB_CUDA(cudaEventSynchronize(h->ev1));
  float ms = 0.f;
  RLB_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  *avg_ms = ms / iters;
  *work_per_launch = work;
  return RLB_OK;
}

int rlb_score(rlb_instance* h, const int32_t* tokens, int32_t n, float* out_logits) {
  RLB_CHECK(h && tokens && out_logits, RLB_ERR_ARG, "null argument");
  RLB_CHECK(h->has_weights, RLB_ERR_STATE, "no weights loaded");
  RLB_CHECK(n >= 1 && n <= h->max_seq, RLB_ERR_CAPACITY, "score length exceeds max_seq_len");
  RLB_CHECK(!h->free_slots.empty(), RLB_ERR_CAPACITY, "no free slot for scoring");
  const int np = (n + PAGE - 1) / PAGE;
  RLB_CHECK(static_cast<int>(h->free_pages.size()) >= np, RLB_ERR_CAPACITY, "no free pages for scoring");
  RLB_CUDA(cudaSetDevice(h->device));
  Req tmp;
  tmp.n_prompt = n;
  tmp.target_len = 0;
  const int s = h->free_slots.back();
  h->free_slots.pop_back();
  tmp.slot = s;
  for (int i = 0; i < np; ++i) {
    h->h_bt[static_cast<size_t>(s) * h->pps + i] = h->free_pages.back();
    h->free_pages.pop_back();
  }
  h->slots_dirty = true;
  int rc = h->upload_slots();
  if (rc) return rc;
  int* tok = h->h_stage;
  int* pos = h->h_stage + h->stage_cap;
  int* slot = h->h_stage + 2 * h->stage_cap;
  int* lsrc = h->h_stage + 3 * h->stage_cap;
  for (int i = 0; i < n; ++i) {
    tok[i] = tokens[i];
    pos[i] = i;
    slot[i] = s;
  }
  for (int beg = 0; beg < n && rc == 0; beg += h->prefill_rows) {
    const int cnt = std::min(h->prefill_rows, n - beg);
    RLB_CUDA(cudaMemcpyAsync(h->d_row_tok, tok + beg, cnt * 4, cudaMemcpyHostToDevice, h->st));
    RLB_CUDA(cudaMemcpyAsync(h->d_row_pos, pos + beg, cnt * 4, cudaMemcpyHostToDevice, h->st));
    RLB_CUDA(cudaMemcpyAsync(h->d_row_slot, slot + beg, cnt * 4, cudaMemcpyHostToDevice, h->st));
    // the same pair lists (2-warp short pairs + 4-warp long pairs) as prefill
    if ((rc = h->build_pairs(pos + beg, cnt))) break;
    rc = h->forward_layers(cnt, true);
    h->pairs_short = h->pairs_long = h->head16_n = 0;
    if (rc) break;
    for (int lb = 0; lb < cnt; lb += h->max_slots) {
      const int ln = std::min(h->max_slots, cnt - lb);
      for (int i = 0; i < ln; ++i) lsrc[i] = lb + i;
      RLB_CUDA(cudaMemcpyAsync(h->d_logit_src, lsrc, ln * 4, cudaMemcpyHostToDevice, h->st));
      if ((rc = h->head(ln, false))) break;
      RLB_CUDA(cudaMemcpyAsync(out_logits + static_cast<size_t>(beg + lb) * h->V, h->d_logits,
                               sizeof(float) * ln * static_cast<size_t>(h->V),
                               cudaMemcpyDeviceToHost, h->st));
      RLB_CUDA(cudaStreamSynchronize(h->st));
    }
  }
  h->release(&tmp);
  if (rc) return rc;
  RLB_CUDA(cudaStreamSynchronize(h->st));
  return RLB_OK;
}

}  // extern "C"
