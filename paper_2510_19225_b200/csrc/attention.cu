// K1: paged decode attention on the tensor cores (mma.sync m16n8k16).
//
// One CTA = (token row, kv head, window of SUPER=2048 positions); for every
// context the configs use (<= 1408 + prefix) that is one CTA per (row, kv head)
// and no combine pass.  The GQA group (G <= 8 query heads sharing the kv head)
// forms the M rows of the MMA, so K and V are read from HBM exactly once.
// Positions are cut into 64-token pages; warp w of the WARPS (2) owns pages
// w, w+WARPS, ... of the window and streams them in 16-token chunks through
// a STAGES-deep ring (TMA boxes of the pool's tensor map, or cp.async;
// XOR-swizzled rows, ldmatrix / ldmatrix.trans fragments):
//     S = Q K^T (fp32) -> scale, mask -> online softmax in chunk order
//     -> P (bf16, the S accumulator layout reused as the A operand) -> O += P V
// The warp partials are merged in warp order, then normalised (or, for
// windows beyond the first, written as (O, m, l) and merged in window order).
//
// Determinism: every reduction order (quad shuffles, chunk order, warp order,
// window order) is a function of the row's context length only, so a row gets
// the same bits as a decode row or as one of the rows of a varlen prefill --
// the property migration resume relies on (SURVEY.md §7 part 2).
#define RLB_PDL_CLASS 2
#include "internal.h"

#include <algorithm>
#include <cstdlib>

namespace rlb {

namespace {

#ifndef ATTN_WARPS
#define ATTN_WARPS 2
#endif
// warps per (row, kv head) item: page p of a window goes to warp p mod WARPS,
// and the partials merge in warp order -- part of the numerics plan.
// Measured (bench.py, one box): 2 warps at 4 decode CTAs / 6 prefill pair
// CTAs per SM beat 4 warps at 2 / 3 (decode attention 67.4 vs 71.2 us at
// context ~770, prefill -4%) and 1 warp at 8 / 12 (73.3 us).
constexpr int WARPS = ATTN_WARPS;
constexpr int CHUNK = 16;              // tokens per pipeline stage
#ifndef ATTN_STAGES
#define ATTN_STAGES 3
#endif
constexpr int STAGES = ATTN_STAGES;    // decode ring depth (timing only, not the bits)
#ifndef ATTN_SUPER
#define ATTN_SUPER 2048
#endif
constexpr int SUPER = ATTN_SUPER;           // positions per CTA window (8 pages per warp)
static_assert(SUPER / PAGE / WARPS <= 32, "page ids of a warp are held one per lane");

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;   // zero-fill past the context end
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// D = A(16x16, rows 8..15 zero) * B(16x8) + D
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

}  // namespace

#ifndef ATTN_MINB
#define ATTN_MINB 4   // resident CTAs per SM the register budget is cut for
#endif

// Everything one (window, kv head, row) item needs before its K/V stream:
// q fragments, the row's length and this lane's page id (each lane holds
// one page of its warp's share).  Loaded ahead of the item by the persistent
// kernel, so the dependent chain row -> slot -> block table -> q is off the
// critical path.
template <int D>
struct AttnItem {
  uint32_t qa[D / 16][2];
  int n = 0;            // context length of the row (0: nothing in this window)
  int my_page = 0;
};

template <int D>
__device__ __forceinline__ void attn_load_item(const AttnArgs& a, int ws_idx, int kvh, int r,
                                               AttnItem<D>& it) {
  constexpr int KSTEPS = D / 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.NQ / a.NKV;
  const int h = lane >> 2;
  const bf16* qrow = a.q + static_cast<size_t>(r) * a.ldq + static_cast<size_t>(kvh * G + h) * D;
#pragma unroll
  for (int kk = 0; kk < KSTEPS; ++kk) {
    const int c = kk * 16 + 2 * (lane & 3);
    it.qa[kk][0] = h < G ? *reinterpret_cast<const uint32_t*>(qrow + c) : 0u;
    it.qa[kk][1] = h < G ? *reinterpret_cast<const uint32_t*>(qrow + c + 8) : 0u;
  }
  const int n = a.row_pos[r] + 1;
  const int w0 = ws_idx * SUPER;
  it.n = w0 >= n ? 0 : n;
  it.my_page = 0;
  if (it.n) {
    const int wn = min(SUPER, n - w0);
    const int npages = (wn + PAGE - 1) / PAGE;
    const int nseg = npages > warp ? (npages - warp + WARPS - 1) / WARPS : 0;
    if (lane < nseg) {
      const int p = w0 / PAGE + warp + lane * WARPS;
      RLB_DEV_CHECK(p < a.bt_stride, "attention: position beyond the block table");
      it.my_page = a.block_table[static_cast<size_t>(a.row_slot[r]) * a.bt_stride + p];
      RLB_DEV_CHECK(it.my_page >= 0 && it.my_page < a.num_pages, "attention: page id");
    }
  }
}

// Byte offset of (token row, 16-byte column chunk ch) inside a K or V chunk
// stage.  cp.async path: 256-byte rows, chunk index XOR (row & 7) (the XOR
// stays inside a 128-byte half).  TMA path: the 128B-swizzled image of a 3D
// box -- D/64 blocks of 16 rows x 128 bytes, 16-byte chunk index XOR
// (row & 7) within each block (the hardware's SWIZZLE_128B pattern).  Both
// keep ldmatrix bank-conflict free.
template <int D, bool TMA>
__device__ __forceinline__ uint32_t kv_off(int row, int ch) {
  if constexpr (TMA)
    return (ch >> 3) * (CHUNK * 128) + row * 128 + (((ch & 7) ^ (row & 7)) << 4);
  else
    return row * (D * 2) + ((ch ^ (row & 7)) << 4);
}

// One item: stream the window's K/V pages through the warps' cp.async rings
// (S = QK^T, online softmax, O += PV on the tensor cores), merge the warp
// partials in warp order, write the row's output (or the window partial).
// Called by every thread of the CTA (it synchronises the CTA).
template <int D, bool TMA = false>
__device__ __forceinline__ void attn_run_item(const AttnArgs& a, int ws_idx, int kvh, int r,
                                              const AttnItem<D>& it, uint8_t* smem,
                                              const CUtensorMap* kvmap = nullptr) {
  constexpr int ROWB = D * 2;            // bytes per token row
  constexpr int CPR = ROWB / 16;         // 16-byte chunks per row
  constexpr int KSTEPS = D / 16;
  constexpr int NT = D / 8;              // output n-tiles
  constexpr int STAGE_BYTES = 2 * CHUNK * ROWB;      // K and V
  constexpr int WARP_SMEM = STAGES * STAGE_BYTES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.NQ / a.NKV;
  const int n = it.n;
  const int w0 = ws_idx * SUPER;
  const int wn = min(SUPER, n - w0);                     // positions in this window
  const float scale = rsqrtf(static_cast<float>(D)) * 1.4426950408889634f;
  const int npages = (wn + PAGE - 1) / PAGE;
  const int nseg = npages > warp ? (npages - warp + WARPS - 1) / WARPS : 0;
  const int my_page = it.my_page;
  // chunk c of this warp: segment c/4 (window page warp + 4*(c/4)), rows 16*(c%4)..
  const int last_seg_tokens = nseg > 0 ? min(PAGE, wn - (warp + (nseg - 1) * WARPS) * PAGE) : 0;
  const int nchunks = nseg > 0 ? (nseg - 1) * (PAGE / CHUNK) + (last_seg_tokens + CHUNK - 1) / CHUNK : 0;

  uint8_t* wsm = smem + warp * WARP_SMEM;
  const uint32_t wsm_u32 = smem_u32(wsm);
  const size_t head_off = static_cast<size_t>(kvh) * (2 * PAGE * D);
  const size_t page_stride = static_cast<size_t>(a.NKV) * (2 * PAGE * D);

  // TMA path: one 3D box (16 token rows x D/64 swizzled 128-byte blocks) for
  // K and one for V per chunk, issued by lane 0 and completed on the stage's
  // mbarrier (tokens past the page's valid ones are loaded as they are --
  // finite K/V of earlier tokens or zeros -- and masked to p = 0 exactly as
  // the zero-filled rows of the cp.async path)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * WARP_SMEM) + warp * STAGES;
  if constexpr (TMA) {
    if (lane == 0) {
      for (int i = 0; i < STAGES; ++i) mbar_init(smem_u32(&bars[i]), 1);
      fence_mbar_init();
    }
    __syncwarp();
  }
  auto issue = [&](int c) {
    const int seg = c >> 2;
    const int page = __shfl_sync(0xffffffffu, my_page, seg);
    if constexpr (TMA) {
      if (lane == 0) {
        const uint32_t st = wsm_u32 + (c % STAGES) * STAGE_BYTES;
        const uint32_t bar = smem_u32(&bars[c % STAGES]);
        // generic-proxy reads of this stage (ldmatrix) precede the async write
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, STAGE_BYTES);
        const int64_t row = a.kv_row0 + (static_cast<int64_t>(page) * a.NKV + kvh) * (2 * PAGE) +
                            (c & 3) * CHUNK;
        tma_load_3d(st, kvmap, bar, static_cast<int32_t>(row), 0);
        tma_load_3d(st + CHUNK * ROWB, kvmap, bar, static_cast<int32_t>(row + PAGE), 0);
      }
      return;
    }
    const int seg_tok = min(PAGE, wn - (warp + seg * WARPS) * PAGE);   // valid tokens in the page
    const bf16* kp = a.kv + static_cast<size_t>(page) * page_stride + head_off;
    const uint32_t st = wsm_u32 + (c % STAGES) * STAGE_BYTES;
#pragma unroll
    for (int i = 0; i < (CHUNK * CPR) / 32; ++i) {
      const int idx = i * 32 + lane;
      const int row = idx / CPR, ch = idx % CPR;
      const int tok = (c & 3) * CHUNK + row;          // token within the page
      const bool ok = tok < seg_tok;
      const bf16* src = kp + static_cast<size_t>(ok ? tok : 0) * D + ch * 8;
      const uint32_t off = row * ROWB + ((ch ^ (row & 7)) << 4);
      cp_async16(st + off, src, ok);
      cp_async16(st + CHUNK * ROWB + off, src + PAGE * D, ok);
    }
  };

  float o[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;

#pragma unroll
  for (int c = 0; c < STAGES - 1; ++c) {
    if (c < nchunks) issue(c);
    cp_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    if (c + STAGES - 1 < nchunks) issue(c + STAGES - 1);
    if constexpr (TMA) {
      mbar_wait(smem_u32(&bars[c % STAGES]), (c / STAGES) & 1);
    } else {
      cp_commit();
      cp_wait<STAGES - 1>();
    }
    __syncwarp();
    const uint32_t ks = wsm_u32 + (c % STAGES) * STAGE_BYTES;
    const uint32_t vs = ks + CHUNK * ROWB;
    const int seg_tok = min(PAGE, wn - (warp + (c >> 2) * WARPS) * PAGE);
    const int tok0 = (c & 3) * CHUNK;
    // ---- S = Q K^T over 16 tokens (two n-tiles of 8)
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    {
      const int mi = lane >> 3, ri = lane & 7;
      const int row = (mi >> 1) * 8 + ri;         // token within the chunk
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        const int ch = 2 * kk + (mi & 1);
        uint32_t b[4];
        ldsm_x4(ks + kv_off<D, TMA>(row, ch), b);
        mma_bf16(s[0], it.qa[kk][0], it.qa[kk][1], b[0], b[1]);
        mma_bf16(s[1], it.qa[kk][0], it.qa[kk][1], b[2], b[3]);
      }
    }
    // ---- online softmax (row = lane/4, columns 2*(lane%4)+{0,1} of each n-tile)
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = tok0 + 8 * j + 2 * (lane & 3) + e;
        s[j][e] = tok < seg_tok ? s[j][e] * scale : -INFINITY;
        mx = fmaxf(mx, s[j][e]);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    const float corr = exp2f(m_run - m_new);
    float p[2][2], rs = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        p[j][e] = exp2f(s[j][e] - m_new);
        rs += p[j][e];
      }
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    rs += __shfl_xor_sync(0xffffffffu, rs, 2);
    l_run = __fmaf_rn(l_run, corr, rs);
    m_run = m_new;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      o[t][0] *= corr;
      o[t][1] *= corr;
    }
    const uint32_t pa0 = pack_bf2(p[0][0], p[0][1]);
    const uint32_t pa2 = pack_bf2(p[1][0], p[1][1]);
    // ---- O += P V   (V^T fragments via ldmatrix.trans)
    {
      const int mi = lane >> 3, ri = lane & 7;
      const int row = (mi & 1) * 8 + ri;          // token within the chunk
#pragma unroll
      for (int dt = 0; dt < NT / 2; ++dt) {
        const int ch = 2 * dt + (mi >> 1);
        uint32_t b[4];
        ldsm_x4_t(vs + kv_off<D, TMA>(row, ch), b);
        mma_bf16(o[2 * dt], pa0, pa2, b[0], b[1]);
        mma_bf16(o[2 * dt + 1], pa0, pa2, b[2], b[3]);
      }
    }
    __syncwarp();
  }
  if constexpr (!TMA) cp_wait<0>();
  __syncthreads();

  // ---- merge the 4 warp partials in warp order
  float* red = reinterpret_cast<float*>(smem);            // [WARPS][8][D]
  float* mls = red + WARPS * 8 * D;                        // [WARPS][8][2]
  {
    const int h = lane >> 2;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int col = t * 8 + 2 * (lane & 3);
      *reinterpret_cast<float2*>(&red[(warp * 8 + h) * D + col]) = make_float2(o[t][0], o[t][1]);
    }
    if ((lane & 3) == 0) {
      mls[(warp * 8 + h) * 2] = m_run;
      mls[(warp * 8 + h) * 2 + 1] = l_run;
    }
  }
  __syncthreads();
  const bool single = n <= SUPER;
  for (int i = threadIdx.x; i < G * D; i += WARPS * 32) {
    const int g = i / D, d = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, mls[(w * 8 + g) * 2]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const float cw = exp2f(mls[(w * 8 + g) * 2] - M);
      L = __fmaf_rn(cw, mls[(w * 8 + g) * 2 + 1], L);
      O = __fmaf_rn(cw, red[(w * 8 + g) * D + d], O);
    }
    const int qh = kvh * G + g;
    if (single) {
      a.out[static_cast<size_t>(r) * a.ldo + qh * D + d] = __float2bfloat16_rn(O / L);
    } else {
      float* wsp = a.ws + ((static_cast<size_t>(r) * a.NQ + qh) * a.max_splits + ws_idx) * (D + 2);
      wsp[d] = O;
      if (d == 0) {
        wsp[D] = M;
        wsp[D + 1] = L;
      }
    }
  }
}

// One CTA per (window, kv head, row).  TMA: the K/V chunks arrive through
// tensor-map boxes of the KV pool (`kvmap`, AttnArgs.kv_row0) instead of
// per-lane cp.async -- the same bytes in the same order, the same bits.
template <int D, bool TMA = false>
__global__ void __launch_bounds__(WARPS * 32, ATTN_MINB)
    attn_mma_kernel(AttnArgs a, const __grid_constant__ CUtensorMap kvmap) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // the 128B-swizzle pattern of a TMA box is a function of the smem address:
  // stages start on 1024-byte boundaries (the launch adds 1 KB of slack)
  uint8_t* smem = TMA ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                   ~static_cast<uintptr_t>(1023))
                      : smem_raw;
  if constexpr (TMA) {
    if (threadIdx.x == 0) tma_prefetch(&kvmap);
  }
  pdl_trigger();
  pdl_wait();   // q and this step's K/V rows come from the previous kernel
  AttnItem<D> it;
  attn_load_item<D>(a, blockIdx.x, blockIdx.y, blockIdx.z, it);
  if (it.n == 0) return;
  attn_run_item<D, TMA>(a, blockIdx.x, blockIdx.y, blockIdx.z, it, smem, &kvmap);
}

// Prefill variant: one CTA serves two consecutive token rows (2p, 2p+1) of
// the same sequence, the second row's GQA group in MMA rows 8..15 (zero in
// the decode kernel), so every K/V chunk is loaded once for both.  Each row
// keeps its own online-softmax state and skips the chunks that hold none of
// its positions -- so it goes through exactly the chunk sequence, masking,
// warp split and merge order of the decode kernel and gets the same bits
// (the varlen-resume invariant).  Rows of different sequences (a pair that
// straddles a sequence boundary) run as two single-row passes.
__device__ __forceinline__ void mma_bf16_full(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                              uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

#ifndef ATTN_PAIR_STAGES
#define ATTN_PAIR_STAGES 2     // prefill rows: a shallower ring, more resident CTAs
#endif
#ifndef ATTN_PAIR_MINB
#define ATTN_PAIR_MINB 6
#endif
// NW = 2 < WARPS (built only when WARPS > 2): the short-pair variant --
// rows with <= 2 pages of context only have pages in warp slots 0 and 1, so
// two physical warps do all the work and the other slots enter the merge as
// the empty partials (m = -inf, l = 0, o = 0) an idle warp of the full
// kernel contributes: the same merge, the same bits, at a smaller footprint.
// With WARPS = 2 (the default) every pair runs on the full kernel.
template <int D, int NW = WARPS>
__global__ void __launch_bounds__(NW * 32, NW == WARPS ? ATTN_PAIR_MINB : 2 * ATTN_PAIR_MINB)
    attn_pair_kernel(AttnArgs a) {
  constexpr int STAGES = ATTN_PAIR_STAGES;   // pipeline depth only: no effect on the bits
  constexpr int ROWB = D * 2;
  constexpr int CPR = ROWB / 16;
  constexpr int KSTEPS = D / 16;
  constexpr int NT = D / 8;
  constexpr int STAGE_BYTES = 2 * CHUNK * ROWB;
  constexpr int WARP_SMEM = STAGES * STAGE_BYTES;
  extern __shared__ __align__(128) uint8_t smem[];

  const int ws_idx = blockIdx.x, kvh = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.NQ / a.NKV;
  pdl_trigger();
  pdl_wait();
  const int rA = 2 * (a.pair_ids ? a.pair_ids[a.pair_off + blockIdx.z]
                                  : static_cast<int>(blockIdx.z));
  const bool hasB = rA + 1 < a.R;
  const bool shared = hasB && a.row_slot[rA] == a.row_slot[rA + 1];
  const float scale = rsqrtf(static_cast<float>(D)) * 1.4426950408889634f;
  const int w0 = ws_idx * SUPER;
  const int h = lane >> 2;

  // pass 0: rows A (and B when it shares A's sequence); pass 1: row B alone
  for (int pass = 0; pass < (hasB && !shared ? 2 : 1); ++pass) {
    const int r0 = rA + pass;                              // MMA rows 0..7
    const bool two = pass == 0 && shared;                  // MMA rows 8..15 = row rA + 1
    const int n0 = a.row_pos[r0] + 1;
    const int n1 = two ? a.row_pos[rA + 1] + 1 : 0;
    const int wn0 = min(SUPER, n0 - w0), wn1 = two ? min(SUPER, n1 - w0) : 0;
    const int wn = max(wn0, wn1);
    if (wn <= 0) continue;

    uint32_t qa[KSTEPS][4];
    {
      const bf16* q0 = a.q + static_cast<size_t>(r0) * a.ldq + static_cast<size_t>(kvh * G + h) * D;
      const bf16* q1 = a.q + static_cast<size_t>(rA + 1) * a.ldq + static_cast<size_t>(kvh * G + h) * D;
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        const int c = kk * 16 + 2 * (lane & 3);
        qa[kk][0] = h < G && wn0 > 0 ? *reinterpret_cast<const uint32_t*>(q0 + c) : 0u;
        qa[kk][2] = h < G && wn0 > 0 ? *reinterpret_cast<const uint32_t*>(q0 + c + 8) : 0u;
        qa[kk][1] = h < G && wn1 > 0 ? *reinterpret_cast<const uint32_t*>(q1 + c) : 0u;
        qa[kk][3] = h < G && wn1 > 0 ? *reinterpret_cast<const uint32_t*>(q1 + c + 8) : 0u;
      }
    }
    const int npages = (wn + PAGE - 1) / PAGE;
    const int nseg = npages > warp ? (npages - warp + WARPS - 1) / WARPS : 0;
    int my_page = 0;
    if (lane < nseg) {
      const int pg = w0 / PAGE + warp + lane * WARPS;
      RLB_DEV_CHECK(pg < a.bt_stride, "pair attention: position beyond the block table");
      my_page = a.block_table[static_cast<size_t>(a.row_slot[r0]) * a.bt_stride + pg];
      RLB_DEV_CHECK(my_page >= 0 && my_page < a.num_pages, "pair attention: page id");
    }
    const int last_seg_tokens = nseg > 0 ? min(PAGE, wn - (warp + (nseg - 1) * WARPS) * PAGE) : 0;
    const int nchunks = nseg > 0 ? (nseg - 1) * (PAGE / CHUNK) + (last_seg_tokens + CHUNK - 1) / CHUNK : 0;
    uint8_t* wsm = smem + warp * WARP_SMEM;
    const uint32_t wsm_u32 = smem_u32(wsm);
    const size_t head_off = static_cast<size_t>(kvh) * (2 * PAGE * D);
    const size_t page_stride = static_cast<size_t>(a.NKV) * (2 * PAGE * D);
    auto issue = [&](int c) {
      const int seg = c >> 2;
      const int page = __shfl_sync(0xffffffffu, my_page, seg);
      const int seg_tok = min(PAGE, wn - (warp + seg * WARPS) * PAGE);
      const bf16* kp = a.kv + static_cast<size_t>(page) * page_stride + head_off;
      const uint32_t st = wsm_u32 + (c % STAGES) * STAGE_BYTES;
#pragma unroll
      for (int i = 0; i < (CHUNK * CPR) / 32; ++i) {
        const int idx = i * 32 + lane;
        const int row = idx / CPR, ch = idx % CPR;
        const int tok = (c & 3) * CHUNK + row;
        const bool ok = tok < seg_tok;
        const bf16* src = kp + static_cast<size_t>(ok ? tok : 0) * D + ch * 8;
        const uint32_t off = row * ROWB + ((ch ^ (row & 7)) << 4);
        cp_async16(st + off, src, ok);
        cp_async16(st + CHUNK * ROWB + off, src + PAGE * D, ok);
      }
    };

    float o[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
#pragma unroll
    for (int c = 0; c < STAGES - 1; ++c) {
      if (c < nchunks) issue(c);
      cp_commit();
    }
    for (int c = 0; c < nchunks; ++c) {
      if (c + STAGES - 1 < nchunks) issue(c + STAGES - 1);
      cp_commit();
      cp_wait<STAGES - 1>();
      __syncwarp();
      const uint32_t ks = wsm_u32 + (c % STAGES) * STAGE_BYTES;
      const uint32_t vs = ks + CHUNK * ROWB;
      const int pstart = (warp + (c >> 2) * WARPS) * PAGE;   // window position of the page
      const int tok0 = (c & 3) * CHUNK;
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      {
        const int mi = lane >> 3, ri = lane & 7;
        const int row = (mi >> 1) * 8 + ri;
#pragma unroll
        for (int kk = 0; kk < KSTEPS; ++kk) {
          const int ch = 2 * kk + (mi & 1);
          uint32_t b[4];
          ldsm_x4(ks + row * ROWB + ((ch ^ (row & 7)) << 4), b);
          mma_bf16_full(s[0], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b[0], b[1]);
          mma_bf16_full(s[1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b[2], b[3]);
        }
      }
      // per row x (0: MMA rows 0-7, 1: rows 8-15): online softmax over the
      // chunk exactly as the decode kernel does, or no update at all when the
      // chunk holds none of the row's positions
      uint32_t pa[2][2];
      float corr[2];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int wnx = x == 0 ? wn0 : wn1;
        const int seg_tok = min(PAGE, wnx - pstart);
        const bool active = pstart + tok0 < wnx;             // a valid position in the chunk
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int tok = tok0 + 8 * j + 2 * (lane & 3) + e;
            s[j][2 * x + e] = tok < seg_tok ? s[j][2 * x + e] * scale : -INFINITY;
            mx = fmaxf(mx, s[j][2 * x + e]);
          }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        float p[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
        corr[x] = 1.f;
        if (active) {
          const float m_new = fmaxf(m_run[x], mx);
          corr[x] = exp2f(m_run[x] - m_new);
          float rs = 0.f;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              p[j][e] = exp2f(s[j][2 * x + e] - m_new);
              rs += p[j][e];
            }
          rs += __shfl_xor_sync(0xffffffffu, rs, 1);
          rs += __shfl_xor_sync(0xffffffffu, rs, 2);
          l_run[x] = __fmaf_rn(l_run[x], corr[x], rs);
          m_run[x] = m_new;
        }
        pa[x][0] = pack_bf2(p[0][0], p[0][1]);
        pa[x][1] = pack_bf2(p[1][0], p[1][1]);
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        o[t][0] *= corr[0];
        o[t][1] *= corr[0];
        o[t][2] *= corr[1];
        o[t][3] *= corr[1];
      }
      {
        const int mi = lane >> 3, ri = lane & 7;
        const int row = (mi & 1) * 8 + ri;
#pragma unroll
        for (int dt = 0; dt < NT / 2; ++dt) {
          const int ch = 2 * dt + (mi >> 1);
          uint32_t b[4];
          ldsm_x4_t(vs + row * ROWB + ((ch ^ (row & 7)) << 4), b);
          mma_bf16_full(o[2 * dt], pa[0][0], pa[1][0], pa[0][1], pa[1][1], b[0], b[1]);
          mma_bf16_full(o[2 * dt + 1], pa[0][0], pa[1][0], pa[0][1], pa[1][1], b[2], b[3]);
        }
      }
      __syncwarp();
    }
    cp_wait<0>();
    __syncthreads();

    // merge the 4 warp partials of each row in warp order
    float* red = reinterpret_cast<float*>(smem);                 // [WARPS][16][D]
    float* mls = red + WARPS * 16 * D;                             // [WARPS][16][2]
    {
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int col = t * 8 + 2 * (lane & 3);
        *reinterpret_cast<float2*>(&red[(warp * 16 + h) * D + col]) = make_float2(o[t][0], o[t][1]);
        *reinterpret_cast<float2*>(&red[(warp * 16 + 8 + h) * D + col]) = make_float2(o[t][2], o[t][3]);
      }
      if ((lane & 3) == 0) {
        mls[(warp * 16 + h) * 2] = m_run[0];
        mls[(warp * 16 + h) * 2 + 1] = l_run[0];
        mls[(warp * 16 + 8 + h) * 2] = m_run[1];
        mls[(warp * 16 + 8 + h) * 2 + 1] = l_run[1];
      }
      if constexpr (NW < WARPS) {   // the idle slots' partials, as the full kernel has them
        for (int w = NW + warp; w < WARPS; w += NW) {
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int col = t * 8 + 2 * (lane & 3);
            *reinterpret_cast<float2*>(&red[(w * 16 + h) * D + col]) = make_float2(0.f, 0.f);
            *reinterpret_cast<float2*>(&red[(w * 16 + 8 + h) * D + col]) = make_float2(0.f, 0.f);
          }
          if ((lane & 3) == 0) {
            mls[(w * 16 + h) * 2] = -INFINITY;
            mls[(w * 16 + h) * 2 + 1] = 0.f;
            mls[(w * 16 + 8 + h) * 2] = -INFINITY;
            mls[(w * 16 + 8 + h) * 2 + 1] = 0.f;
          }
        }
      }
    }
    // per (row, head) slot: the running max over the warps, each warp's
    // rescale factor and the merged denominator, once per slot instead of
    // once per output element (same operations, same order, same bits)
    float* cws = mls + WARPS * 16 * 2;                             // [16][WARPS + 2]
    __syncthreads();
    if (threadIdx.x < 16) {
      const int slot = threadIdx.x;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) M = fmaxf(M, mls[(w * 16 + slot) * 2]);
      float L = 0.f;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const float cw = exp2f(mls[(w * 16 + slot) * 2] - M);
        L = __fmaf_rn(cw, mls[(w * 16 + slot) * 2 + 1], L);
        cws[slot * (WARPS + 2) + w] = cw;
      }
      cws[slot * (WARPS + 2) + WARPS] = M;
      cws[slot * (WARPS + 2) + WARPS + 1] = L;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * G * D; i += NW * 32) {
      const int x = i / (G * D), g = (i / D) % G, d = i % D;
      if (x == 1 && !two) break;
      const int rr = x == 0 ? r0 : rA + 1;
      const int n = x == 0 ? n0 : n1;
      if (w0 >= n) continue;                                   // no positions in this window
      const int slot = x * 8 + g;
      const float* cs = cws + slot * (WARPS + 2);
      const float M = cs[WARPS], L = cs[WARPS + 1];
      float O = 0.f;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) O = __fmaf_rn(cs[w], red[(w * 16 + slot) * D + d], O);
      const int qh = kvh * G + g;
      if (n <= SUPER) {
        a.out[static_cast<size_t>(rr) * a.ldo + qh * D + d] = __float2bfloat16_rn(O / L);
      } else {
        float* wsp = a.ws + ((static_cast<size_t>(rr) * a.NQ + qh) * a.max_splits + ws_idx) * (D + 2);
        wsp[d] = O;
        if (d == 0) {
          wsp[D] = M;
          wsp[D + 1] = L;
        }
      }
    }
    __syncthreads();                                           // smem reused by the next pass
  }
}

// K1h: prefill rows packed by head.  The pair kernel's MMA rows are 2 token
// rows x 8 head slots, of which a GQA group of 6 (7 for the 7B shape) is
// real.  Here a CTA serves 16 consecutive rows of one sequence for ONE query
// head: the MMA rows are the 16 positions, all real, so a chunk's QK^T and
// PV MMAs (and the softmax instructions around them) serve 16 rows instead
// of 12.  Every (row, head) still goes through the decode kernel's sequence:
// the same pages per warp slot, 16-token chunks in order, the same masking,
// online-softmax steps (quad shuffles over the same token columns) and
// warp-order merge -- a row whose positions end before a chunk takes no
// update from it (computed and discarded, so the quad shuffles stay
// converged).  Same bits as K1p and K1.
template <int D>
__global__ void __launch_bounds__(WARPS * 32, ATTN_PAIR_MINB) attn_head16_kernel(AttnArgs a) {
  constexpr int STAGES = ATTN_PAIR_STAGES;
  constexpr int ROWB = D * 2;
  constexpr int CPR = ROWB / 16;
  constexpr int KSTEPS = D / 16;
  constexpr int NT = D / 8;
  constexpr int STAGE_BYTES = 2 * CHUNK * ROWB;
  constexpr int WARP_SMEM = STAGES * STAGE_BYTES;
  extern __shared__ __align__(128) uint8_t smem[];

  const int ws_idx = blockIdx.x, qh = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.NQ / a.NKV;
  const int kvh = qh / G;
  pdl_trigger();
  pdl_wait();
  const int rG = a.head16_ids[blockIdx.z];                 // first of the 16 rows
  const float scale = rsqrtf(static_cast<float>(D)) * 1.4426950408889634f;
  const int w0 = ws_idx * SUPER;
  const int h = lane >> 2;                                  // this lane's rows: rG+h, rG+h+8
  const int wnr[2] = {min(SUPER, a.row_pos[rG + h] + 1 - w0),
                      min(SUPER, a.row_pos[rG + h + 8] + 1 - w0)};
  const int wn = min(SUPER, a.row_pos[rG + 15] + 1 - w0);  // the last row sees the most
  if (wn <= 0) return;                                      // uniform over the CTA

  uint32_t qa[KSTEPS][4];
  {
    const bf16* q0 = a.q + static_cast<size_t>(rG + h) * a.ldq + static_cast<size_t>(qh) * D;
    const bf16* q1 = q0 + static_cast<size_t>(8) * a.ldq;
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
      const int c = kk * 16 + 2 * (lane & 3);
      qa[kk][0] = wnr[0] > 0 ? *reinterpret_cast<const uint32_t*>(q0 + c) : 0u;
      qa[kk][2] = wnr[0] > 0 ? *reinterpret_cast<const uint32_t*>(q0 + c + 8) : 0u;
      qa[kk][1] = wnr[1] > 0 ? *reinterpret_cast<const uint32_t*>(q1 + c) : 0u;
      qa[kk][3] = wnr[1] > 0 ? *reinterpret_cast<const uint32_t*>(q1 + c + 8) : 0u;
    }
  }
  const int npages = (wn + PAGE - 1) / PAGE;
  const int nseg = npages > warp ? (npages - warp + WARPS - 1) / WARPS : 0;
  int my_page = 0;
  if (lane < nseg) {
    const int pg = w0 / PAGE + warp + lane * WARPS;
    RLB_DEV_CHECK(pg < a.bt_stride, "head16 attention: position beyond the block table");
    my_page = a.block_table[static_cast<size_t>(a.row_slot[rG]) * a.bt_stride + pg];
    RLB_DEV_CHECK(my_page >= 0 && my_page < a.num_pages, "head16 attention: page id");
  }
  const int last_seg_tokens = nseg > 0 ? min(PAGE, wn - (warp + (nseg - 1) * WARPS) * PAGE) : 0;
  const int nchunks = nseg > 0 ? (nseg - 1) * (PAGE / CHUNK) + (last_seg_tokens + CHUNK - 1) / CHUNK : 0;
  uint8_t* wsm = smem + warp * WARP_SMEM;
  const uint32_t wsm_u32 = smem_u32(wsm);
  const size_t head_off = static_cast<size_t>(kvh) * (2 * PAGE * D);
  const size_t page_stride = static_cast<size_t>(a.NKV) * (2 * PAGE * D);
  auto issue = [&](int c) {
    const int seg = c >> 2;
    const int page = __shfl_sync(0xffffffffu, my_page, seg);
    const int seg_tok = min(PAGE, wn - (warp + seg * WARPS) * PAGE);
    const bf16* kp = a.kv + static_cast<size_t>(page) * page_stride + head_off;
    const uint32_t st = wsm_u32 + (c % STAGES) * STAGE_BYTES;
#pragma unroll
    for (int i = 0; i < (CHUNK * CPR) / 32; ++i) {
      const int idx = i * 32 + lane;
      const int row = idx / CPR, ch = idx % CPR;
      const int tok = (c & 3) * CHUNK + row;
      const bool ok = tok < seg_tok;
      const bf16* src = kp + static_cast<size_t>(ok ? tok : 0) * D + ch * 8;
      const uint32_t off = row * ROWB + ((ch ^ (row & 7)) << 4);
      cp_async16(st + off, src, ok);
      cp_async16(st + CHUNK * ROWB + off, src + PAGE * D, ok);
    }
  };

  float o[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
#pragma unroll
  for (int c = 0; c < STAGES - 1; ++c) {
    if (c < nchunks) issue(c);
    cp_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    if (c + STAGES - 1 < nchunks) issue(c + STAGES - 1);
    cp_commit();
    cp_wait<STAGES - 1>();
    __syncwarp();
    const uint32_t ks = wsm_u32 + (c % STAGES) * STAGE_BYTES;
    const uint32_t vs = ks + CHUNK * ROWB;
    const int pstart = (warp + (c >> 2) * WARPS) * PAGE;
    const int tok0 = (c & 3) * CHUNK;
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    {
      const int mi = lane >> 3, ri = lane & 7;
      const int row = (mi >> 1) * 8 + ri;
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        const int ch = 2 * kk + (mi & 1);
        uint32_t b[4];
        ldsm_x4(ks + row * ROWB + ((ch ^ (row & 7)) << 4), b);
        mma_bf16_full(s[0], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b[0], b[1]);
        mma_bf16_full(s[1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b[2], b[3]);
      }
    }
    uint32_t pa[2][2];
    float corr[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int wnx = wnr[x];
      const int seg_tok = min(PAGE, wnx - pstart);
      const bool active = pstart + tok0 < wnx;             // per quad: the quad's row
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int tok = tok0 + 8 * j + 2 * (lane & 3) + e;
          s[j][2 * x + e] = tok < seg_tok ? s[j][2 * x + e] * scale : -INFINITY;
          mx = fmaxf(mx, s[j][2 * x + e]);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      // every lane runs the shuffles; an inactive row keeps its state
      const float m_new = fmaxf(m_run[x], mx);
      const float cr = exp2f(m_run[x] - m_new);
      float p[2][2], rs = 0.f;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          p[j][e] = active ? exp2f(s[j][2 * x + e] - m_new) : 0.f;
          rs += p[j][e];
        }
      rs += __shfl_xor_sync(0xffffffffu, rs, 1);
      rs += __shfl_xor_sync(0xffffffffu, rs, 2);
      corr[x] = active ? cr : 1.f;
      if (active) {
        l_run[x] = __fmaf_rn(l_run[x], cr, rs);
        m_run[x] = m_new;
      }
      pa[x][0] = pack_bf2(p[0][0], p[0][1]);
      pa[x][1] = pack_bf2(p[1][0], p[1][1]);
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      o[t][0] *= corr[0];
      o[t][1] *= corr[0];
      o[t][2] *= corr[1];
      o[t][3] *= corr[1];
    }
    {
      const int mi = lane >> 3, ri = lane & 7;
      const int row = (mi & 1) * 8 + ri;
#pragma unroll
      for (int dt = 0; dt < NT / 2; ++dt) {
        const int ch = 2 * dt + (mi >> 1);
        uint32_t b[4];
        ldsm_x4_t(vs + row * ROWB + ((ch ^ (row & 7)) << 4), b);
        mma_bf16_full(o[2 * dt], pa[0][0], pa[1][0], pa[0][1], pa[1][1], b[0], b[1]);
        mma_bf16_full(o[2 * dt + 1], pa[0][0], pa[1][0], pa[0][1], pa[1][1], b[2], b[3]);
      }
    }
    __syncwarp();
  }
  cp_wait<0>();
  __syncthreads();

  // merge the 4 warp partials of each of the 16 rows in warp order
  float* red = reinterpret_cast<float*>(smem);                 // [WARPS][16][D]
  float* mls = red + WARPS * 16 * D;                             // [WARPS][16][2]
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int col = t * 8 + 2 * (lane & 3);
    *reinterpret_cast<float2*>(&red[(warp * 16 + h) * D + col]) = make_float2(o[t][0], o[t][1]);
    *reinterpret_cast<float2*>(&red[(warp * 16 + 8 + h) * D + col]) = make_float2(o[t][2], o[t][3]);
  }
  if ((lane & 3) == 0) {
    mls[(warp * 16 + h) * 2] = m_run[0];
    mls[(warp * 16 + h) * 2 + 1] = l_run[0];
    mls[(warp * 16 + 8 + h) * 2] = m_run[1];
    mls[(warp * 16 + 8 + h) * 2 + 1] = l_run[1];
  }
  float* cws = mls + WARPS * 16 * 2;                             // [16][WARPS + 2]
  __syncthreads();
  if (threadIdx.x < 16) {
    const int slot = threadIdx.x;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, mls[(w * 16 + slot) * 2]);
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const float cw = exp2f(mls[(w * 16 + slot) * 2] - M);
      L = __fmaf_rn(cw, mls[(w * 16 + slot) * 2 + 1], L);
      cws[slot * (WARPS + 2) + w] = cw;
    }
    cws[slot * (WARPS + 2) + WARPS] = M;
    cws[slot * (WARPS + 2) + WARPS + 1] = L;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 16 * D; i += WARPS * 32) {
    const int slot = i / D, d = i % D;
    const int rr = rG + slot;
    const int n = a.row_pos[rr] + 1;
    if (w0 >= n) continue;                                     // no positions in this window
    const float* cs = cws + slot * (WARPS + 2);
    const float M = cs[WARPS], L = cs[WARPS + 1];
    float O = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) O = __fmaf_rn(cs[w], red[(w * 16 + slot) * D + d], O);
    if (n <= SUPER) {
      a.out[static_cast<size_t>(rr) * a.ldo + qh * D + d] = __float2bfloat16_rn(O / L);
    } else {
      float* wsp = a.ws + ((static_cast<size_t>(rr) * a.NQ + qh) * a.max_splits + ws_idx) * (D + 2);
      wsp[d] = O;
      if (d == 0) {
        wsp[D] = M;
        wsp[D + 1] = L;
      }
    }
  }
}

// Merge the per-window partials of rows longer than one window, in order.
__global__ void attn_combine_kernel(AttnArgs a) {
  pdl_trigger();
  pdl_wait();
  const int qh = blockIdx.x, r = blockIdx.y, d = threadIdx.x;
  const int n = a.row_pos[r] + 1;
  const int ns = (n + SUPER - 1) / SUPER;
  if (ns <= 1) return;
  const int D = a.D;
  const float* w = a.ws + (static_cast<size_t>(r) * a.NQ + qh) * a.max_splits * (D + 2);
  float M = -INFINITY;
  for (int s = 0; s < ns; ++s) M = fmaxf(M, w[s * (D + 2) + D]);
  float L = 0.f, O = 0.f;
  for (int s = 0; s < ns; ++s) {
    const float c = exp2f(w[s * (D + 2) + D] - M);
    L = __fmaf_rn(c, w[s * (D + 2) + D + 1], L);
    O = __fmaf_rn(c, w[s * (D + 2) + d], O);
  }
  a.out[static_cast<size_t>(r) * a.ldo + qh * D + d] = __float2bfloat16_rn(O / L);
}

int attention_windows(int max_seq) { return (max_seq + SUPER - 1) / SUPER; }
int attention_window_positions() { return SUPER; }
int attention_warps() { return WARPS; }

template <int D>
static int launch_attn(const AttnArgs& a, cudaStream_t st, bool pairs) {
  constexpr int smem_pipe = WARPS * STAGES * 2 * CHUNK * D * 2;
  constexpr int smem_red = WARPS * 8 * D * 4 + WARPS * 8 * 2 * 4;
  constexpr int smem = smem_pipe > smem_red ? smem_pipe : smem_red;
  constexpr int smem_tma = smem + WARPS * STAGES * 8 + 1024;   // + mbarriers, alignment slack
  constexpr int smem_red2 = WARPS * 16 * D * 4 + WARPS * 16 * 2 * 4 + 16 * (WARPS + 2) * 4;
  constexpr int smem_pipe2 = WARPS * ATTN_PAIR_STAGES * 2 * CHUNK * D * 2;
  constexpr int smem2 = smem_pipe2 > smem_red2 ? smem_pipe2 : smem_red2;
  constexpr int smem_pipe2s = 2 * ATTN_PAIR_STAGES * 2 * CHUNK * D * 2;   // 2-warp short pairs
  constexpr int smem2s = smem_pipe2s > smem_red2 ? smem_pipe2s : smem_red2;
  static bool attr[64] = {false};
  int dev = 0;
  RLB_CUDA(cudaGetDevice(&dev));
  if (!attr[dev & 63]) {
    RLB_CUDA(cudaFuncSetAttribute(attn_mma_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    RLB_CUDA(cudaFuncSetAttribute(attn_mma_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_tma));
    RLB_CUDA(cudaFuncSetAttribute(attn_pair_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem2));
    if constexpr (WARPS > 2)
      RLB_CUDA(cudaFuncSetAttribute(attn_pair_kernel<D, 2>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem2s));
    RLB_CUDA(cudaFuncSetAttribute(attn_head16_kernel<D>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    attr[dev & 63] = true;
  }
  static int n_sm = 0;
  if (!n_sm) RLB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));

  if (pairs && a.pair_ids) {
    if (a.n_head16 > 0)
      RLB_CUDA(launch_k(attn_head16_kernel<D>, dim3(a.max_splits, a.NQ, a.n_head16),
                        dim3(WARPS * 32), smem2, st, a));
    AttnArgs as = a, al = a;
    as.pair_off = 0;
    al.pair_off = a.n_short;
    if constexpr (WARPS > 2) {
      if (a.n_short > 0)
        RLB_CUDA(launch_k(attn_pair_kernel<D, 2>, dim3(a.max_splits, a.NKV, a.n_short), dim3(64),
                          smem2s, st, as));
    } else {                      // no narrower variant: short pairs on the same kernel
      al.pair_off = 0;
      al.n_long = a.n_short + a.n_long;
    }
    if (al.n_long > 0)
      RLB_CUDA(launch_k(attn_pair_kernel<D>, dim3(a.max_splits, a.NKV, al.n_long),
                        dim3(WARPS * 32), smem2, st, al));
  } else if (pairs) {
    RLB_CUDA(launch_k(attn_pair_kernel<D>, dim3(a.max_splits, a.NKV, (a.R + 1) / 2),
                      dim3(WARPS * 32), smem2, st, a));
  } else if (a.kv_map) {
    RLB_CUDA(launch_k(attn_mma_kernel<D, true>, dim3(a.max_splits, a.NKV, a.R), dim3(WARPS * 32),
                      smem_tma, st, a, *a.kv_map));
  } else {
    CUtensorMap none{};
    RLB_CUDA(launch_k(attn_mma_kernel<D, false>, dim3(a.max_splits, a.NKV, a.R), dim3(WARPS * 32),
                      smem, st, a, none));
  }
  return RLB_OK;
}

int attention_launch(const AttnArgs& a, cudaStream_t st, bool row_pairs) {
  if (a.R <= 0) return RLB_OK;
  RLB_CHECK(a.NQ % a.NKV == 0 && a.NQ / a.NKV <= 8, RLB_ERR_ARG, "GQA group must be <= 8");
  int rc;
  if (a.D == 128)
    rc = launch_attn<128>(a, st, row_pairs);
  else if (a.D == 64)
    rc = launch_attn<64>(a, st, row_pairs);
  else
    RLB_CHECK(false, RLB_ERR_ARG, "head_dim must be 64 or 128");
  if (rc) return rc;
  if (a.max_splits > 1) {
    RLB_CUDA(launch_k(attn_combine_kernel, dim3(a.NQ, a.R), dim3(a.D), 0, st, a));
  }
  return RLB_OK;
}

}  // namespace rlb
