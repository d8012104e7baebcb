// K2: tcgen05 + TMA GEMMs for the dense projections.
//
//   C[M, N] = A[M, K] . B[N, K]^T      (A = activations, B = weights; both K-major bf16)
//
// One CTA computes a (128 * NACC) x BN tile: NACC = 2 gives two 128 x BN UMMA
// accumulators in TMEM that share every B stage (a weight tile is read once
// per 256 rows); NACC = 1 gives twice the CTAs for the short projections,
// which are bound by how fast one SM's shared memory can be fed.  BN is 256,
// 128 or (RoPE only) 64.  (A-tile multicast across N-tile pairs and
// non-persistent 2-SM 512 x 256 tiles were measured slower and removed;
// DESIGN.md §9.)
// Warp roles (384 threads):
//   warp 0      one elected lane issues TMA loads: A rows [m, m+128), A rows
//               [m+128, m+256) and B rows [n, n+BN), 64-element (128 B) K
//               slices with the 128B swizzle, into a STAGES-deep smem ring
//               guarded by full/empty mbarriers;
//   warp 1      one elected lane issues tcgen05.mma (M=128, N=BN, K=16) for
//               both halves and releases stages with tcgen05.commit;
//   warp 2      allocates / frees 2*BN TMEM columns;
//   warps 4-11  epilogue: warps 4-7 drain accumulator 0, warps 8-11
//               accumulator 1 (tcgen05.ld 32 lanes x 16 columns) and apply the
//               fused op: bias+bf16 / fp32 residual add / SwiGLU / fp32 /
//               greedy argmax partials.
// Split-K (grid.z = splits) covers the small-N projections of a decode step.
// The S split CTAs of a tile form one (1,1,S) thread-block cluster: each
// stages its fp32 partial tile in its own shared memory, and after a cluster
// barrier CTA z sums rows [z*256/S, (z+1)*256/S) of all S partials through
// distributed shared memory in split order (z = 0..S-1) and applies the
// epilogue -- residual add into h (EPI_RESADD) or bias + RoPE + q / paged
// K,V stores (EPI_ROPE).  No partial reaches HBM and no consumer kernel
// re-reads it.  The split count is a property of the weight matrix (never of
// M), so a token row's result is bit-identical in a 512-row decode batch and
// in a varlen prefill chunk -- migration resume relies on this (SURVEY.md §7
// hard part 2).  EPI_PARTIAL (fp32 partials to a workspace) remains for the
// kernel-level test entry rlb_gemm.
#define RLB_PDL_CLASS 1
#include "internal.h"

#include <cstdio>
#include <cstdlib>

namespace rlb {

constexpr int HM = 128;      // rows per accumulator (UMMA_M)
constexpr int BK = 64;       // K elements per stage (one 128 B swizzle atom)
constexpr int GEMM_THREADS = 384;

// NACC accumulators of 128 rows per CTA: 2 (256-row tiles, the B stage is
// shared by both) or 1 (128-row tiles: twice the CTAs for short-K / small-N
// projections that would otherwise need split-K).
// KPS = K blocks per pipeline stage.  KPS = 2 (the 64-column QKV tiles)
// loads each operand tile as one 3D box of two stacked 64-wide K blocks: a
// TMA-streaming SM's rate grows with the bytes per box (64-row weight boxes
// stream at half the rate of 128-row ones, scripts/probe_stream.cu).
template <int BN, int NACC, int KPS = 1>
struct GemmCfg {
  static constexpr int BMT = HM * NACC;                // rows per CTA
  static constexpr int A_BYTES = HM * BK * 2;          // one accumulator's rows, one K block
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = KPS * (NACC * A_BYTES + B_BYTES);
  static constexpr int STAGES =
      (BN == 256 ? 3 : (NACC == 2 ? 4 : (BN == 64 ? 8 : 6))) / KPS;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = NACC * BN;
};

__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// Generic split-K reduce (kernel-level test entry rlb_gemm only; the engine
// fuses the reduction into its row-wise consumer kernels): sum the fp32
// partials of each row in split order and apply the epilogue.
template <int EPI>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(GemmParams p) {
  const int m = blockIdx.x;
  const size_t slab = static_cast<size_t>(p.M) * p.N;
#pragma unroll 1
  for (int n = threadIdx.x * 4; n < p.N; n += 1024) {
    const float* src = p.ws + static_cast<size_t>(m) * p.N + n;
    float4 acc = __ldcg(reinterpret_cast<const float4*>(src));
    for (int z = 1; z < p.splits; ++z) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(src + z * slab));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if constexpr (EPI == EPI_BF16) {
      if (p.bias) {
        acc.x += __bfloat162float(p.bias[n]);
        acc.y += __bfloat162float(p.bias[n + 1]);
        acc.z += __bfloat162float(p.bias[n + 2]);
        acc.w += __bfloat162float(p.bias[n + 3]);
      }
      *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(p.out) + static_cast<size_t>(m) * p.ldo + n) =
          make_uint2(pack_bf2(acc.x, acc.y), pack_bf2(acc.z, acc.w));
    } else if constexpr (EPI == EPI_RESADD) {
      float4* h = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) +
                                            static_cast<size_t>(m) * p.ldo + n);
      float4 x = *h;
      x.x += acc.x;
      x.y += acc.y;
      x.z += acc.z;
      x.w += acc.w;
      *h = x;
    } else if constexpr (EPI == EPI_F32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + static_cast<size_t>(m) * p.ldo + n) =
          acc;
    }
  }
}

constexpr int EPI_LDS = 128 + 4;   // padded fp32 row of a staged 128-column tile

// Engine QKV layout (pull.cu relayout_segments): within a head, each 64-row
// block holds 32 rows of the first rotation half and their partners, i.e.
// physical column c of a head (block t = c / 64, b = c % 64) is head column
// t*32 + b for b < 32 and t*32 + (b - 32) + D/2 otherwise.  The head column
// of the first half of the block holding physical column gcol:
__device__ __forceinline__ int rope_j0(int gcol, int D) { return ((gcol % D) / 64) * 32; }

// Split-K reduction of one BMT x 128 tile inside its cluster: this CTA (rank
// z of S) owns tile rows [z*BMT/S, (z+1)*BMT/S); epilogue warp ew (of NW)
// takes every NW-th of them (<= 32 rows, so lane k can hold row k's
// metadata).  Partials are summed in split order 0..S-1 (the association of
// a sequential sum), then the epilogue is applied.  Rows go in groups of G
// with every load of the group issued before any store, so the L2 / DSMEM
// latencies overlap.
template <int EPI, int BMT, int NW>
__device__ __forceinline__ void cluster_epilogue(const GemmParams& p, uint32_t stage_u32,
                                                 int m_blk, int n_blk, int ew, int lane) {
  constexpr int G = 4;
  const int S = p.splits;
  const int z = static_cast<int>(cluster_rank());
  const int r0 = z * BMT / S, r1 = (z + 1) * BMT / S;
  uint32_t base[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) base[i] = i < S ? dsmem_addr(stage_u32, i) : 0u;
  const int last = min(r1, p.M - m_blk * BMT);
  const int nrows = last > r0 + ew ? (last - (r0 + ew) + NW - 1) / NW : 0;
  if constexpr (EPI == EPI_RESADD) {
    // h[m, n..n+3] += sum_z part_z: one row per warp step, one float4 per lane
    const int n = n_blk * 128 + lane * 4;
    if (n >= p.N) return;
    float* h = reinterpret_cast<float*>(p.out);
#pragma unroll 1
    for (int k0 = 0; k0 < nrows; k0 += G) {
      float4 x[G], acc[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (k0 + g < nrows) {
          const int rr = r0 + ew + NW * (k0 + g);
          x[g] = *reinterpret_cast<const float4*>(h + static_cast<size_t>(m_blk * BMT + rr) * p.ldo + n);
          const uint32_t off = static_cast<uint32_t>((rr * EPI_LDS + lane * 4) * 4);
          acc[g] = dsmem_ld4(base[0] + off);
#pragma unroll
          for (int i = 1; i < 8; ++i) {
            if (i < S) {
              const float4 v = dsmem_ld4(base[i] + off);
              acc[g].x += v.x;
              acc[g].y += v.y;
              acc[g].z += v.z;
              acc[g].w += v.w;
            }
          }
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (k0 + g < nrows) {
          const int rr = r0 + ew + NW * (k0 + g);
          x[g].x += acc[g].x;
          x[g].y += acc[g].y;
          x[g].z += acc[g].z;
          x[g].w += acc[g].w;
          *reinterpret_cast<float4*>(h + static_cast<size_t>(m_blk * BMT + rr) * p.ldo + n) = x[g];
        }
      }
    }
  } else if constexpr (EPI == EPI_ROPE) {
    // 64 rotation pairs (c1, c1 + D/2) per 128-column tile; lane takes pairs
    // lane and lane + 32.  x = sum_z part + bias; q/k rotated, v copied; K/V
    // into the slot's page.
    const RopeDst& d = p.rope;
    const int hd = d.d / 2;
    const size_t head_stride = static_cast<size_t>(2) * PAGE * d.d;
    int pos_l = 0;
    size_t kvo_l = 0;
    if (lane < nrows) {
      const int m = m_blk * BMT + r0 + ew + NW * lane;
      pos_l = d.row_pos[m];
      RLB_DEV_CHECK(pos_l / PAGE < d.bt_stride, "RoPE epilogue: position beyond the block table");
      const int page = d.block_table[static_cast<size_t>(d.row_slot[m]) * d.bt_stride + pos_l / PAGE];
      RLB_DEV_CHECK(page >= 0 && page < d.num_pages, "RoPE epilogue: page id");
      kvo_l = static_cast<size_t>(page) * head_stride * d.nkv + static_cast<size_t>(pos_l % PAGE) * d.d;
    }
    int jv[2], c1v[2], headv[2];
    float b1[2], b2[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      // pair lane + 32 t: physical column 64 t + lane and its partner (+32)
      c1v[t] = 64 * t + lane;
      const int col1 = n_blk * 128 + c1v[t];
      jv[t] = rope_j0(col1, d.d) + lane;
      headv[t] = col1 / d.d;
      b1[t] = __bfloat162float(p.bias[col1]);
      b2[t] = __bfloat162float(p.bias[col1 + 32]);
    }
#pragma unroll 1
    for (int k0 = 0; k0 < nrows; k0 += G) {
      float x1[G][2], x2[G][2];
      float2 cs[G][2];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int posg = __shfl_sync(0xffffffffu, pos_l, (k0 + g) & 31);
        if (k0 + g < nrows) {
          const int rr = r0 + ew + NW * (k0 + g);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const uint32_t o1 = static_cast<uint32_t>((rr * EPI_LDS + c1v[t]) * 4);
            const uint32_t o2 = o1 + 32u * 4u;                 // the partner column
            float a1 = dsmem_ld(base[0] + o1), a2 = dsmem_ld(base[0] + o2);
#pragma unroll
            for (int i = 1; i < 8; ++i) {
              if (i < S) {
                a1 += dsmem_ld(base[i] + o1);
                a2 += dsmem_ld(base[i] + o2);
              }
            }
            x1[g][t] = a1;
            x2[g][t] = a2;
            cs[g][t] = d.rope[static_cast<size_t>(posg) * hd + jv[t]];
          }
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const unsigned long long kvo =
            __shfl_sync(0xffffffffu, static_cast<unsigned long long>(kvo_l), (k0 + g) & 31);
        if (k0 + g >= nrows) continue;
        const int m = m_blk * BMT + r0 + ew + NW * (k0 + g);
        bf16* kv_page = d.kv + kvo;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int j = jv[t], head = headv[t];
          const float v1 = x1[g][t] + b1[t];
          const float v2 = x2[g][t] + b2[t];
          if (head < d.nq + d.nkv) {
            const float2 c = cs[g][t];
            const float y1 = __fmaf_rn(v1, c.x, -v2 * c.y);
            const float y2 = __fmaf_rn(v2, c.x, v1 * c.y);
            bf16* o = head < d.nq ? d.q + static_cast<size_t>(m) * d.ldq + head * d.d
                                  : kv_page + static_cast<size_t>(head - d.nq) * head_stride;
            o[j] = __float2bfloat16_rn(y1);
            o[j + hd] = __float2bfloat16_rn(y2);
          } else {
            bf16* o = kv_page + static_cast<size_t>(head - d.nq - d.nkv) * head_stride +
                      static_cast<size_t>(PAGE) * d.d;
            o[j] = __float2bfloat16_rn(v1);
            o[j + hd] = __float2bfloat16_rn(v2);
          }
        }
      }
    }
  }
}

// EPI_ROPE without split-K, straight from TMEM: the thread owns row m (its
// TMEM lane) and the tile's 128 columns (one head of D=128, two of D=64).
// Rotation partners c and c + D/2 are loaded as two 32-column chunks.
// Row metadata of the direct RoPE epilogue, loaded by the epilogue thread
// while the mainloop runs: position, its K/V slot, and an L1 prefetch of the
// (cos, sin) rows the thread's column pairs will read.
struct RopeRow {
  int pos = 0;
  bf16* kv_page = nullptr;
};
// Engine QKV layout (pull.cu relayout_segments): within a head, each 64-row
// block holds 32 rows of the first rotation half and their partners, i.e.
// physical column c of a head (block t = c / 64, b = c % 64) is head column
// t*32 + b for b < 32 and t*32 + (b - 32) + D/2 otherwise.  Chunk pair cp of a
// tile = physical columns [64 cp, 64 cp + 32) and their partners (+32).

__device__ __forceinline__ RopeRow rope_row_prefetch(const GemmParams& p, int m, bool live,
                                                     int col0, int cp0, int cp1) {
  RopeRow rr;
  if (!live) return rr;
  const RopeDst& d = p.rope;
  const int hd = d.d / 2;
  const size_t head_stride = static_cast<size_t>(2) * PAGE * d.d;
  rr.pos = d.row_pos[m];
  RLB_DEV_CHECK(rr.pos / PAGE < d.bt_stride, "RoPE epilogue: position beyond the block table");
  const int page = d.block_table[static_cast<size_t>(d.row_slot[m]) * d.bt_stride + rr.pos / PAGE];
  RLB_DEV_CHECK(page >= 0 && page < d.num_pages, "RoPE epilogue: page id");
  rr.kv_page = d.kv + static_cast<size_t>(page) * head_stride * d.nkv +
               static_cast<size_t>(rr.pos % PAGE) * d.d;
  for (int cp = cp0; cp < cp1; ++cp) {
    const int j0 = rope_j0(col0 + cp * 64, d.d);
    const char* c = reinterpret_cast<const char*>(d.rope + static_cast<size_t>(rr.pos) * hd + j0);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(c));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(c + 128));
  }
  return rr;
}

__device__ __forceinline__ void rope_direct(const GemmParams& p, uint32_t tbase, int m, bool live,
                                            int col0, int cp0, int cp1, const RopeRow& rr) {
  const RopeDst& d = p.rope;
  const int hd = d.d / 2;
  const size_t head_stride = static_cast<size_t>(2) * PAGE * d.d;
  const int pos = rr.pos;
  bf16* kv_page = rr.kv_page;
#pragma unroll 1
  for (int cp = cp0; cp < cp1; ++cp) {
    const int a = cp * 64;                                   // physical column of the chunk
    uint32_t r1[32], r2[32];
    tmem_ld32(tbase + a, r1);
    tmem_ld32(tbase + a + 32, r2);                           // the partners
    tmem_ld_wait();
    if (!live) continue;
    const int col1 = col0 + a;                               // physical output column
    const int head = col1 / d.d;
    const int j0 = rope_j0(col1, d.d);                       // head column (< hd)
    const uint4* bb1 = reinterpret_cast<const uint4*>(p.bias + col1);
    const uint4* bb2 = reinterpret_cast<const uint4*>(p.bias + col1 + 32);
    float v1[32], v2[32];
#pragma unroll
    for (int h4 = 0; h4 < 4; ++h4) {
      const uint4 u1 = bb1[h4], u2 = bb2[h4];
      const uint32_t w1[4] = {u1.x, u1.y, u1.z, u1.w}, w2[4] = {u2.x, u2.y, u2.z, u2.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v1[8 * h4 + 2 * i] = __uint_as_float(r1[8 * h4 + 2 * i]) + bf_lo(w1[i]);
        v1[8 * h4 + 2 * i + 1] = __uint_as_float(r1[8 * h4 + 2 * i + 1]) + bf_hi(w1[i]);
        v2[8 * h4 + 2 * i] = __uint_as_float(r2[8 * h4 + 2 * i]) + bf_lo(w2[i]);
        v2[8 * h4 + 2 * i + 1] = __uint_as_float(r2[8 * h4 + 2 * i + 1]) + bf_hi(w2[i]);
      }
    }
    uint32_t o1[16], o2[16];
    bf16* dst;
    if (head < d.nq + d.nkv) {
      const float4* cs4 = reinterpret_cast<const float4*>(d.rope + static_cast<size_t>(pos) * hd + j0);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float4 c = cs4[i];                   // (cos, sin) of j0+2i, j0+2i+1
        const float y1a = __fmaf_rn(v1[2 * i], c.x, -v2[2 * i] * c.y);
        const float y2a = __fmaf_rn(v2[2 * i], c.x, v1[2 * i] * c.y);
        const float y1b = __fmaf_rn(v1[2 * i + 1], c.z, -v2[2 * i + 1] * c.w);
        const float y2b = __fmaf_rn(v2[2 * i + 1], c.z, v1[2 * i + 1] * c.w);
        o1[i] = pack_bf2(y1a, y1b);
        o2[i] = pack_bf2(y2a, y2b);
      }
      dst = head < d.nq ? d.q + static_cast<size_t>(m) * d.ldq + head * d.d
                        : kv_page + static_cast<size_t>(head - d.nq) * head_stride;
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        o1[i] = pack_bf2(v1[2 * i], v1[2 * i + 1]);
        o2[i] = pack_bf2(v2[2 * i], v2[2 * i + 1]);
      }
      dst = kv_page + static_cast<size_t>(head - d.nq - d.nkv) * head_stride +
            static_cast<size_t>(PAGE) * d.d;
    }
    uint4* d1 = reinterpret_cast<uint4*>(dst + j0);
    uint4* d2 = reinterpret_cast<uint4*>(dst + j0 + hd);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      d1[i] = make_uint4(o1[4 * i], o1[4 * i + 1], o1[4 * i + 2], o1[4 * i + 3]);
      d2[i] = make_uint4(o2[4 * i], o2[4 * i + 1], o2[4 * i + 2], o2[4 * i + 3]);
    }
  }
}

template <int BN, int EPI, int NACC, int KPS = 1>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 GemmParams p) {
  using C = GemmCfg<BN, NACC, KPS>;
  static_assert(KPS == 1 || (NACC == 1 && C::STAGES >= 2),
                "two-K-block stages: one accumulator, at least two stages (the only tested form)");
  constexpr int BMT = C::BMT;
  constexpr int NEW = 4 * NACC;                 // epilogue warps with an accumulator
  // epilogue warps that run (direct RoPE with one accumulator splits columns)
  constexpr int NEW_ALL = (EPI == EPI_ROPE && NACC == 1 && BN == 128) ? 8 : NEW;
  constexpr bool kClusterEpi = cluster_epi(EPI) && BN == 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // row tiles vary fastest: the CTAs sharing a weight (B) tile are dispatched
  // together, so a weight tile is read from HBM once even when the whole
  // weight matrix does not fit in L2 (lm_head: 467 MB)
  const int m_blk = blockIdx.x;
  const int n_blk = blockIdx.y;
  const bool stamp = p.dbg != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
  auto gtime = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
  if (stamp && threadIdx.x == 0) p.dbg[0] = gtime();
  const int nk_total = p.K / BK;
  // split z covers K blocks [z*nk/S, (z+1)*nk/S): a fixed partition of the
  // weight's K range (uneven when S does not divide it)
  const int kb0 = static_cast<int>(blockIdx.z) * nk_total / p.splits;
  const int nk = (static_cast<int>(blockIdx.z) + 1) * nk_total / p.splits - kb0;
  // split-K cluster epilogue (S > 1) or direct from TMEM (S == 1)
  const bool via_cluster = kClusterEpi && p.splits > 1;
  // accumulators with at least one live row (a small-M tile skips the
  // loads, MMAs and TMEM reads of the empty one)
  const int live_acc = (NACC == 2 && p.M - m_blk * BMT > HM) ? 2 : 1;
  const uint32_t stage_tx = static_cast<uint32_t>(live_acc * C::A_BYTES + C::B_BYTES);

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
  if (stamp && threadIdx.x == 0) p.dbg[1] = gtime();
  pdl_trigger();
  // With programmatic dependent launch this CTA may start while the previous
  // kernel drains.  The weights (B) do not depend on it: the producer issues
  // the first stages' B tiles before waiting, then the A tiles after.  Every
  // other thread waits first (A, h and the outputs belong to the chain).
  const bool producer = warp == 0 && lane == 0;
  // stages of KPS K blocks (a partial last one still receives KPS blocks'
  // bytes: the extra block is unused, or zero-filled past K)
  const int ng = (nk + KPS - 1) / KPS;
  const int pre = ng < C::STAGES ? ng : C::STAGES;
  const uint32_t stage_txk = stage_tx * KPS;
  if (producer) {
    for (int g = 0; g < pre; ++g) {
      uint8_t* st = smem + g * C::STAGE_BYTES;
      mbar_expect_tx(smem_u32(&full[g]), stage_txk);
      if constexpr (KPS == 1)
        tma_load_2d(smem_u32(st + NACC * C::A_BYTES), &tmB, smem_u32(&full[g]), (kb0 + g) * BK,
                    n_blk * BN);
      else
        tma_load_3d(smem_u32(st + NACC * KPS * C::A_BYTES), &tmB, smem_u32(&full[g]), n_blk * BN,
                    kb0 + g * KPS);
    }
  }
  pdl_wait();
  if (stamp && threadIdx.x == 0) p.dbg[2] = gtime();

  if (warp == 0 && KPS > 1) {
    if (producer) {
      for (int g = 0; g < ng; ++g) {
        const int s = g % C::STAGES;
        const uint32_t ph = (g / C::STAGES) & 1;
        uint8_t* st = smem + s * C::STAGE_BYTES;
        if (g >= pre) {
          mbar_wait(smem_u32(&empty[s]), ph ^ 1);
          mbar_expect_tx(smem_u32(&full[s]), stage_txk);
          tma_load_3d(smem_u32(st + NACC * KPS * C::A_BYTES), &tmB, smem_u32(&full[s]), n_blk * BN,
                      kb0 + g * KPS);
        }
#pragma unroll
        for (int a = 0; a < NACC; ++a)
          if (a < live_acc)
            tma_load_3d(smem_u32(st + a * KPS * C::A_BYTES), &tmA, smem_u32(&full[s]),
                        m_blk * BMT + a * HM, kb0 + g * KPS);
      }
    }
  } else if (warp == 1 && KPS > 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(HM, BN);
      for (int g = 0; g < ng; ++g) {
        const int s = g % C::STAGES;
        const uint32_t ph = (g / C::STAGES) & 1;
        const uint32_t st = smem_u32(smem + s * C::STAGE_BYTES);
        mbar_wait(smem_u32(&full[s]), ph);
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < KPS; ++j) {
          if (g * KPS + j >= nk) break;
          const uint64_t bd = umma_desc_sw128(st + NACC * KPS * C::A_BYTES + j * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
#pragma unroll
            for (int a = 0; a < NACC; ++a)
              if (a < live_acc)
                umma_bf16(tmem + a * BN,
                          umma_desc_sw128(st + (a * KPS + j) * C::A_BYTES) + 2 * k, bd + 2 * k,
                          idesc, ((g * KPS + j) | k) != 0);
          }
        }
        umma_commit(smem_u32(&empty[s]));
      }
      umma_commit(smem_u32(tfull));
      if (stamp) p.dbg[3] = gtime();
    }
  } else if (warp == 0) {
    if (producer) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::STAGES;
        const uint32_t ph = (kb / C::STAGES) & 1;
        uint8_t* st = smem + s * C::STAGE_BYTES;
        const int kx = (kb0 + kb) * BK;
        if (kb >= pre) {
          mbar_wait(smem_u32(&empty[s]), ph ^ 1);
          mbar_expect_tx(smem_u32(&full[s]), stage_tx);
          tma_load_2d(smem_u32(st + NACC * C::A_BYTES), &tmB, smem_u32(&full[s]), kx, n_blk * BN);
        }
#pragma unroll
        for (int a = 0; a < NACC; ++a)
          if (a < live_acc)
            tma_load_2d(smem_u32(st + a * C::A_BYTES), &tmA, smem_u32(&full[s]), kx,
                        m_blk * BMT + a * HM);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(HM, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::STAGES;
        const uint32_t ph = (kb / C::STAGES) & 1;
        const uint32_t st = smem_u32(smem + s * C::STAGE_BYTES);
        mbar_wait(smem_u32(&full[s]), ph);
        tc_fence_after();
        const uint64_t bd = umma_desc_sw128(st + NACC * C::A_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          // +32 bytes per K=16 step inside the 128 B swizzle atom (encoded >> 4)
#pragma unroll
          for (int a = 0; a < NACC; ++a)
            if (a < live_acc)
              umma_bf16(tmem + a * BN, umma_desc_sw128(st + a * C::A_BYTES) + 2 * k, bd + 2 * k,
                        idesc, (kb | k) != 0);
        }
        umma_commit(smem_u32(&empty[s]));
      }
      umma_commit(smem_u32(tfull));
      if (stamp) p.dbg[3] = gtime();
    }
  } else if (warp >= 4 && warp < 4 + NEW_ALL) {
    // with one accumulator the RoPE epilogue uses all 8 epilogue warps: warps
    // 8-11 read the same TMEM lanes as 4-7 and take the second column pair
    const int half = NACC == 2 ? (warp - 4) >> 2 : 0;   // accumulator
    const int q = warp & 3;                    // TMEM lane quadrant
    const int m = m_blk * BMT + half * HM + q * 32 + lane;
    const bool live = m < p.M;
    // warp-uniform: no row of this warp exists -> no TMEM reads (tcgen05.ld is
    // warp-collective, so the skip is per warp)
    const bool warp_dead = m_blk * BMT + half * HM + q * 32 >= p.M;
    // RoPE chunk pairs (64 physical columns each) of this thread
    const int rcp0 = NEW_ALL > NEW ? (warp - 4) >> 2 : 0;
    const int rcp1 = NEW_ALL > NEW ? rcp0 + 1 : BN / 64;
    RopeRow rrow;
    if constexpr (EPI == EPI_ROPE) {
      if (!via_cluster) rrow = rope_row_prefetch(p, m, live, n_blk * BN, rcp0, rcp1);   // overlaps the mainloop
    }
    mbar_wait(smem_u32(tfull), 0);
    if (stamp && threadIdx.x == 128) p.dbg[4] = gtime();
    tc_fence_after();
    const uint32_t tbase = tmem + half * BN + (static_cast<uint32_t>(q * 32) << 16);
    if constexpr (EPI == EPI_SWIGLU) {
      // act = silu(gate) * up, staged as bf16 rows in the (now free) pipeline
      // smem, then written as full rows: a warp store covers 512 contiguous
      // bytes instead of 32 rows x 16 bytes.
      constexpr int OC = BN / 2;                       // output columns per row
      constexpr int PITCH = OC * 2 + 16;               // bytes; 16 B pad spreads banks
      uint8_t* stage = smem;
      const int row = half * HM + q * 32 + lane;       // row within the CTA tile
#pragma unroll 1
      for (int g = 0; g < (warp_dead ? 0 : BN / 128); ++g) {
#pragma unroll 1
        for (int jc = 0; jc < 64; jc += 32) {
          uint32_t rg[32], ru[32];
          tmem_ld32(tbase + g * 128 + jc, rg);
          tmem_ld32(tbase + g * 128 + 64 + jc, ru);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a0 = silu_f(__uint_as_float(rg[2 * i])) * __uint_as_float(ru[2 * i]);
            const float a1 = silu_f(__uint_as_float(rg[2 * i + 1])) * __uint_as_float(ru[2 * i + 1]);
            pk[i] = pack_bf2(a0, a1);
          }
          uint4* d = reinterpret_cast<uint4*>(stage + row * PITCH + (g * 64 + jc) * 2);
#pragma unroll
          for (int i = 0; i < 4; ++i) d[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      if (NACC == 2) asm volatile("bar.sync 1, 256;" ::: "memory");
      else asm volatile("bar.sync 1, 128;" ::: "memory");
      bf16* out = reinterpret_cast<bf16*>(p.out);
      constexpr int LPR = OC * 2 / 16;                 // lanes per row (16 B each)
      constexpr int RPW = 32 / LPR;                    // rows per warp instruction
      const int ew = warp - 4;
      const int sub = lane / LPR, cl = lane % LPR;
      const int col = n_blk * OC + cl * 8;
#pragma unroll 2
      for (int rr = ew * RPW + sub; rr < BMT; rr += NEW * RPW) {
        const int mm = m_blk * BMT + rr;
        if (mm >= p.M || col >= p.N / 2) continue;
        *reinterpret_cast<uint4*>(out + static_cast<size_t>(mm) * p.ldo + col) =
            *reinterpret_cast<const uint4*>(stage + rr * PITCH + cl * 16);
      }
    } else if constexpr (EPI == EPI_ARGMAX) {
      // greedy head: per (row, N-tile) max and its lowest column index; the
      // full-vocab logits never reach HBM.
      float best = -INFINITY;
      int bidx = 0x7fffffff;
#pragma unroll 1
      for (int c = 0; c < (warp_dead ? 0 : BN); c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c, r);
        tmem_ld_wait();
        const int n = n_blk * BN + c;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
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
    } else if constexpr (EPI == EPI_ROPE) {
      if (via_cluster) {
        // stage this split's fp32 tile for the cluster reduction (warps 4..)
        float* stage = reinterpret_cast<float*>(smem);
        const int row = half * HM + q * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < (warp_dead || warp >= 4 + NEW ? 0 : BN); c += 32) {
          uint32_t r[32];
          tmem_ld32(tbase + c, r);
          tmem_ld_wait();
          float4* s4 = reinterpret_cast<float4*>(stage + row * EPI_LDS + c);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            s4[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
        }
      } else if (!warp_dead) {
        rope_direct(p, tbase, m, live, n_blk * BN, rcp0, rcp1, rrow);
      }
    } else if constexpr ((EPI == EPI_PARTIAL || EPI == EPI_F32) && BN == 128) {
      // fp32 tile out through shared memory so every global store is a full
      // 512-byte row (a thread-per-row store would issue 32 scattered 16-byte
      // requests per instruction).  The pipeline stages are free: the MMA
      // that consumed them has completed.  EPI_PARTIAL = this K range's fp32
      // partial [z][M][N], reduced in split order by the consumer.
      float* stage = reinterpret_cast<float*>(smem);
      const int row = half * HM + q * 32 + lane;           // row within the CTA tile
#pragma unroll 1
      for (int c = 0; c < (warp_dead ? 0 : BN); c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c, r);
        tmem_ld_wait();
        float4* s4 = reinterpret_cast<float4*>(stage + row * EPI_LDS + c);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          s4[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                              __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
      }
      if (NACC == 2) asm volatile("bar.sync 1, 256;" ::: "memory");
      else asm volatile("bar.sync 1, 128;" ::: "memory");
      float* base = EPI == EPI_PARTIAL ? p.ws + static_cast<size_t>(blockIdx.z) * p.M * p.N
                                       : reinterpret_cast<float*>(p.out);
      const int ld = EPI == EPI_PARTIAL ? p.N : p.ldo;
      const int ew = warp - 4;
      const int n = n_blk * BN + lane * 4;
#pragma unroll 4
      for (int rr = ew; rr < BMT; rr += NEW) {
        const int mm = m_blk * BMT + rr;
        if (mm >= p.M || n >= p.N) continue;
        *reinterpret_cast<float4*>(base + static_cast<size_t>(mm) * ld + n) =
            *reinterpret_cast<const float4*>(stage + rr * EPI_LDS + lane * 4);
      }
    } else {
      // EPI_F32 / EPI_PARTIAL with BN=256, EPI_BF16(+bias), EPI_RESADD
      // (direct when not split, else staged for the cluster reduction).
      float* f32 = EPI == EPI_PARTIAL ? p.ws + static_cast<size_t>(blockIdx.z) * p.M * p.N
                                      : reinterpret_cast<float*>(p.out);
      const int ld = EPI == EPI_PARTIAL ? p.N : p.ldo;
#pragma unroll 1
      for (int c = 0; c < (warp_dead ? 0 : BN); c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c, r);
        tmem_ld_wait();
        if constexpr (kClusterEpi) {
          if (via_cluster) {
            float* stage = reinterpret_cast<float*>(smem);
            const int row = half * HM + q * 32 + lane;
            float4* s4 = reinterpret_cast<float4*>(stage + row * EPI_LDS + c);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              s4[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                  __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
            continue;
          }
        }
        const int n = n_blk * BN + c;
        if (!live || n >= p.N) continue;
        if constexpr (EPI == EPI_BF16) {
          bf16* out = reinterpret_cast<bf16*>(p.out);
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          if (p.bias != nullptr) {
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const uint4 b = reinterpret_cast<const uint4*>(p.bias + n)[h];
              const uint32_t bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                v[8 * h + 2 * i] += bf_lo(bb[i]);
                v[8 * h + 2 * i + 1] += bf_hi(bb[i]);
              }
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = pack_bf2(v[2 * i], v[2 * i + 1]);
          uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(m) * p.ldo + n);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        } else if constexpr (EPI == EPI_RESADD) {
          float4* h = reinterpret_cast<float4*>(f32 + static_cast<size_t>(m) * ld + n);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 x = h[i];
            x.x += __uint_as_float(r[4 * i]);
            x.y += __uint_as_float(r[4 * i + 1]);
            x.z += __uint_as_float(r[4 * i + 2]);
            x.w += __uint_as_float(r[4 * i + 3]);
            h[i] = x;
          }
        } else {  // EPI_F32, EPI_PARTIAL
          float4* o = reinterpret_cast<float4*>(f32 + static_cast<size_t>(m) * ld + n);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            o[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                               __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
        }
      }
    }
  }
  if constexpr (kClusterEpi) {
    if (via_cluster) {                       // uniform over the grid
      cluster_sync();                        // every split's partial tile is staged
      if (warp >= 4 && warp < 4 + NEW)
        cluster_epilogue<EPI, BMT, NEW>(p, smem_u32(smem), m_blk, n_blk, warp - 4, lane);
      cluster_sync();                        // remote reads done before any CTA exits
    }
  }
  if (stamp && threadIdx.x == 128) p.dbg[6] = gtime();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
    if (stamp && lane == 0) p.dbg[5] = gtime();
  }
}

// ---------------------------------------------------------------- CTA pairs --
// Persistent 2-SM GEMM: every (2,1,1) cluster loops over 256 x 256 pair tiles
// (CTA r: rows m*256 + r*128 + [0,128) and B rows n*256 + r*128 + [0,128)).
// A tile's accumulator (128 x 256 per SM) lives in one of two TMEM buffers,
// so the epilogue of tile i drains buffer i&1 while the MMAs of tile i+1 fill
// the other -- the TMEM epilogue leaves the critical path.  The leader's MMA
// thread waits for both CTAs' epilogue warps to release a buffer (16
// arrivals, the peer's through the cluster) before reusing it.
// EPI_PARTIAL (split-K, grid-stride over (m, n, split) tiles) gives one
// pipeline stage to per-warp staging of the fp32 partial (32 rows x 32
// columns at a time, written back as full 128-byte row segments).
// EPI_SUMRES runs a pair tile's splits back to back on one cluster and
// keeps their running sum (acc = p0; acc += p1 ... += p[S-1]) in the CTA's
// L2-resident scratch tile; the last split adds it into the fp32 residual h
// -- the bits resid_norm_kernel<S> produces from EPI_PARTIAL slabs, without
// the [S][M][N] slabs in HBM.
template <int EPI>
struct PairPCfg {
  static constexpr bool kStaged = EPI == EPI_PARTIAL || EPI == EPI_SUMRES;
  static constexpr int A_BYTES = HM * BK * 2;
  static constexpr int B_BYTES = 128 * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = kStaged ? 5 : 6;
  static constexpr int XPITCH = 36;                                // staged fp32 row (floats)
  static constexpr int XSTAGE = kStaged ? 8 * 32 * XPITCH * 4 : 0;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 2048 + XSTAGE;   // + barriers, argmax exchange
  static constexpr uint32_t TMEM_COLS = 512;
};

template <int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_pairp_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  GemmParams p) {
  using C = PairPCfg<EPI>;
  constexpr int BN = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;          // [2]
  uint64_t* tempty = bars + 2 * C::STAGES + 2;     // [2] (leader's copy is used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4);
  float2* xchg = reinterpret_cast<float2*>(bars + 2 * C::STAGES + 6);   // [128] argmax halves

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r = static_cast<int>(cluster_rank());
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int m_tiles = (p.M + 255) / 256, n_tiles = (p.N + BN - 1) / BN;
  // split-K: split z covers K blocks [z*nkt/S, (z+1)*nkt/S) -- the single-SM
  // kernel's partition, so every partial has the same bits
  const int S = (EPI == EPI_PARTIAL || EPI == EPI_SUMRES) ? p.splits : 1;
  const int ntiles = m_tiles * n_tiles * S;
  const int nkt = p.K / BK;
  auto krange = [&](int z, int& kb0, int& nk) {
    kb0 = z * nkt / S;
    nk = (z + 1) * nkt / S - kb0;
  };
  // the cluster's j-th work unit: (m tile, n tile, split).  Grid-stride over
  // (m, n, split) with the split slowest; EPI_SUMRES: grid-stride over pair
  // tiles, each tile's splits consecutively and the n tiles of an m tile on
  // neighbouring clusters (they stream the same A rows through L2 together)
  auto unit = [&](int j, int& mt, int& nt, int& z) {
    if constexpr (EPI == EPI_SUMRES) {
      const int tile = cid + (j / S) * ncl;
      if (tile >= m_tiles * n_tiles) return false;
      nt = tile % n_tiles;
      mt = tile / n_tiles;
      z = j % S;
    } else {
      const int t = cid + j * ncl;
      if (t >= ntiles) return false;
      mt = t % m_tiles;
      nt = (t / m_tiles) % n_tiles;
      z = t / (m_tiles * n_tiles);
    }
    return true;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), 16);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, mt, nt, z;
      for (int j = 0; unit(j, mt, nt, z); ++j) {
        int kb0, nk;
        krange(z, kb0, nk);
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % C::STAGES;
          const uint32_t ph = (g / C::STAGES) & 1;
          uint8_t* st = smem + s * C::STAGE_BYTES;
          const int kx = (kb0 + kb) * BK;
          mbar_wait(smem_u32(&empty[s]), ph ^ 1);
          if (r == 0) mbar_expect_tx(smem_u32(&full[s]), 2 * C::STAGE_BYTES);
          tma_load_2d_pair(smem_u32(st + C::A_BYTES), &tmB, smem_u32(&full[s]), kx,
                           nt * BN + r * 128);
          tma_load_2d_pair(smem_u32(st), &tmA, smem_u32(&full[s]), kx, mt * 256 + r * HM);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && r == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, BN);
      int g = 0, mt, nt, z;
      for (int i = 0; unit(i, mt, nt, z); ++i) {
        const int b = i & 1;
        mbar_wait_cluster(smem_u32(&tempty[b]), ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        int kb0, nk;
        krange(z, kb0, nk);
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % C::STAGES;
          const uint32_t ph = (g / C::STAGES) & 1;
          const uint32_t st = smem_u32(smem + s * C::STAGE_BYTES);
          mbar_wait(smem_u32(&full[s]), ph);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(st), bd = umma_desc_sw128(st + C::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_pair(tmem + b * BN, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          umma_commit_pair(smem_u32(&empty[s]), 0x3);
        }
        umma_commit_pair(smem_u32(&tfull[b]), 0x3);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;                    // TMEM lane quadrant (rows)
    const int ch = (warp - 4) >> 2;            // column half of the 256-column tile
    const uint32_t leader_tempty = dsmem_addr(smem_u32(&tempty[0]), 0);
    // hand TMEM buffer bb back to the leader's MMA thread (one arrival per warp)
    auto release = [&](int bb) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (r == 0) mbar_arrive(smem_u32(&tempty[bb]));
        else mbar_arrive_cluster(leader_tempty + bb * 8);
      }
    };
    int mt, nt, z;
    for (int i = 0; unit(i, mt, nt, z); ++i) {
      const int b = i & 1;
      const int m = mt * 256 + r * HM + q * 32 + lane;
      const bool live = m < p.M;
      const bool warp_dead = mt * 256 + r * HM + q * 32 >= p.M;
      RopeRow rrow;   // EPI_ROPE: row metadata loaded while the tile's MMAs run
      if constexpr (EPI == EPI_ROPE) rrow = rope_row_prefetch(p, m, live, nt * BN + ch * 128, 0, 2);
      mbar_wait(smem_u32(&tfull[b]), (i >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + b * BN + ch * 128 + (static_cast<uint32_t>(q * 32) << 16);
      if constexpr (EPI == EPI_ROPE) {
        // bias + RoPE + q / paged K, V stores of this warp's 128 columns (two
        // 64-column rotation blocks), the single-SM kernel's epilogue
        if (!warp_dead) rope_direct(p, tbase, m, live, nt * BN + ch * 128, 0, 2, rrow);
      } else if constexpr (EPI == EPI_SWIGLU) {
        bf16* out = reinterpret_cast<bf16*>(p.out);
#pragma unroll 1
        for (int jc = 0; jc < (warp_dead ? 0 : 64); jc += 32) {
          uint32_t rg[32], ru[32];
          tmem_ld32(tbase + jc, rg);
          tmem_ld32(tbase + 64 + jc, ru);
          tmem_ld_wait();
          const int col = nt * (BN / 2) + ch * 64 + jc;
          if (live && col < p.N / 2) {
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float a0 = silu_f(__uint_as_float(rg[2 * e])) * __uint_as_float(ru[2 * e]);
              const float a1 = silu_f(__uint_as_float(rg[2 * e + 1])) * __uint_as_float(ru[2 * e + 1]);
              pk[e] = pack_bf2(a0, a1);
            }
            uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(m) * p.ldo + col);
#pragma unroll
            for (int e = 0; e < 4; ++e) dst[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
          }
        }
      } else if constexpr (EPI == EPI_ARGMAX) {
        float best = -INFINITY;
        int bidx = 0x7fffffff;
#pragma unroll 1
        for (int c = 0; c < (warp_dead ? 0 : 128); c += 32) {
          uint32_t rv[32];
          tmem_ld32(tbase + c, rv);
          tmem_ld_wait();
          const int n = nt * BN + ch * 128 + c;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float v = __uint_as_float(rv[e]);
            if (n + e < p.N && v > best) {
              best = v;
              bidx = n + e;
            }
          }
        }
        // the two column halves of a row meet in shared memory: the lower
        // half wins ties (first maximum in column order, as one pass would)
        const int xi = q * 32 + lane;
        if (ch == 1) xchg[xi] = make_float2(best, __int_as_float(bidx));
        asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
        if (ch == 0 && live) {
          const float2 o = xchg[xi];
          if (o.x > best) {
            best = o.x;
            bidx = __float_as_int(o.y);
          }
          float2* part = reinterpret_cast<float2*>(p.out) + static_cast<size_t>(m) * p.ldo + nt;
          *part = make_float2(best, __int_as_float(bidx));
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");   // xchg reusable
      } else if constexpr (EPI == EPI_PARTIAL) {
        // this K range's fp32 partial [z][M][N]: each 32 x 32 block goes
        // through the warp's staging tile (row per lane in, 4 rows x 128 B
        // per store instruction out)
        float* xs = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + 2048) +
                    (warp - 4) * 32 * C::XPITCH;
        float* base = p.ws + static_cast<size_t>(z) * p.M * p.N;
        const int mrow0 = mt * 256 + r * HM + q * 32;
#pragma unroll 1
        for (int c = 0; c < (warp_dead ? 0 : 128); c += 32) {
          uint32_t rv[32];
          tmem_ld32(tbase + c, rv);
          tmem_ld_wait();
          float4* s4 = reinterpret_cast<float4*>(xs + lane * C::XPITCH);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            s4[e] = make_float4(__uint_as_float(rv[4 * e]), __uint_as_float(rv[4 * e + 1]),
                                __uint_as_float(rv[4 * e + 2]), __uint_as_float(rv[4 * e + 3]));
          __syncwarp();
          const int n = nt * BN + ch * 128 + c + (lane & 7) * 4;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int rr = e * 4 + (lane >> 3);
            const int mm = mrow0 + rr;
            if (mm < p.M && n < p.N)
              *reinterpret_cast<float4*>(base + static_cast<size_t>(mm) * p.N + n) =
                  *reinterpret_cast<const float4*>(xs + rr * C::XPITCH + (lane & 7) * 4);
          }
          __syncwarp();
        }
      } else if constexpr (EPI == EPI_SUMRES) {
       // the h rows the last split adds into: into L2 one unit ahead (the
       // last split's pass is otherwise a chain of HBM round trips)
       if (z == (S > 1 ? S - 2 : 0) && live && nt * BN + ch * 128 + 128 <= p.N)
         l2_prefetch_bulk(reinterpret_cast<const float*>(p.out) + static_cast<size_t>(m) * p.ldo +
                              nt * BN + ch * 128, 128 * sizeof(float));
       if (p.sum_tmem) {
        // Running sum in TMEM (splits of a few K blocks, where the L2 scratch
        // traffic below would outlast the MMAs): unit i's buffer holds p_z;
        // for z >= 1 the sum of the previous unit's buffer (s_{z-1}) and this
        // one is stored over p_z and the previous buffer goes back to the
        // MMA thread; the last split then adds its buffer into h.  Each
        // buffer use is released exactly once (by the next unit of its tile,
        // or by itself when it is the last split).
        const uint32_t tprev = tmem + (b ^ 1) * BN + ch * 128 + (static_cast<uint32_t>(q * 32) << 16);
        if (z > 0) {
#pragma unroll 1
          for (int c = 0; c < (warp_dead ? 0 : 128); c += 32) {
            uint32_t ra[32], rc[32];
            tmem_ld32(tprev + c, ra);
            tmem_ld32(tbase + c, rc);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e)
              ra[e] = __float_as_uint(__uint_as_float(ra[e]) + __uint_as_float(rc[e]));
            tmem_st32(tbase + c, ra);
          }
          tmem_st_wait();
          release(b ^ 1);
        }
        if (z == S - 1) {
          float* xs = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + 2048) +
                      (warp - 4) * 32 * C::XPITCH;
          float* hres = reinterpret_cast<float*>(p.out);
          const int mrow0 = mt * 256 + r * HM + q * 32;
#pragma unroll 1
          for (int c = 0; c < (warp_dead ? 0 : 128); c += 32) {
            uint32_t rv[32];
            tmem_ld32(tbase + c, rv);
            tmem_ld_wait();
            float4* s4 = reinterpret_cast<float4*>(xs + lane * C::XPITCH);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              s4[e] = make_float4(__uint_as_float(rv[4 * e]), __uint_as_float(rv[4 * e + 1]),
                                  __uint_as_float(rv[4 * e + 2]), __uint_as_float(rv[4 * e + 3]));
            __syncwarp();
            const int n = nt * BN + ch * 128 + c + (lane & 7) * 4;
            const float* xrow = xs + (lane >> 3) * C::XPITCH + (lane & 7) * 4;
            float* hrow = hres + static_cast<size_t>(mrow0 + (lane >> 3)) * p.ldo + n;
            float4 hv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const bool ok = mrow0 + e * 4 + (lane >> 3) < p.M && n < p.N;
              hv[e] = ok ? *reinterpret_cast<const float4*>(hrow + static_cast<size_t>(e) * 4 * p.ldo)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float4 a = *reinterpret_cast<const float4*>(xrow + e * 4 * C::XPITCH);
              if (mrow0 + e * 4 + (lane >> 3) < p.M && n < p.N)
                *reinterpret_cast<float4*>(hrow + static_cast<size_t>(e) * 4 * p.ldo) =
                    make_float4(hv[e].x + a.x, hv[e].y + a.y, hv[e].z + a.z, hv[e].w + a.w);
            }
            __syncwarp();
          }
          release(b);
        }
       } else {
        // 32 x 32 blocks through the warp's staging tile as EPI_PARTIAL.  The
        // running sum of the tile's splits lives in the CTA's scratch tile:
        // split 0 stores p0, split z adds p_z to it, the last split adds its
        // sum into h -- ((p0 + p1) + ...) + p[S-1], resid_norm's order.  A
        // scratch element is written and read by one thread; a block's loads
        // are issued before its stores.
        float* xs = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + 2048) +
                    (warp - 4) * 32 * C::XPITCH;
        float* scr = p.ws + static_cast<size_t>(blockIdx.x) * (128 * 256);
        float* hres = reinterpret_cast<float*>(p.out);
        const int mrow0 = mt * 256 + r * HM + q * 32;
        const bool fin = z == S - 1;
#pragma unroll 1
        for (int c = 0; c < (warp_dead ? 0 : 128); c += 32) {
          uint32_t rv[32];
          tmem_ld32(tbase + c, rv);
          tmem_ld_wait();
          float4* s4 = reinterpret_cast<float4*>(xs + lane * C::XPITCH);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            s4[e] = make_float4(__uint_as_float(rv[4 * e]), __uint_as_float(rv[4 * e + 1]),
                                __uint_as_float(rv[4 * e + 2]), __uint_as_float(rv[4 * e + 3]));
          __syncwarp();
          const int lc = ch * 128 + c + (lane & 7) * 4;     // column within the CTA tile
          const int n = nt * BN + lc;
          const float* xrow = xs + (lane >> 3) * C::XPITCH + (lane & 7) * 4;
          float* srow = scr + static_cast<size_t>(q * 32 + (lane >> 3)) * 256 + lc;
          float* hrow = hres + static_cast<size_t>(mrow0 + (lane >> 3)) * p.ldo + n;
          float4 a[8], hv[8];
          if (z > 0) {
#pragma unroll
            for (int e = 0; e < 8; ++e) a[e] = __ldcg(reinterpret_cast<const float4*>(srow + e * 4 * 256));
          }
          if (fin) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const bool ok = mrow0 + e * 4 + (lane >> 3) < p.M && n < p.N;
              hv[e] = ok ? *reinterpret_cast<const float4*>(hrow + static_cast<size_t>(e) * 4 * p.ldo)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float4 v = *reinterpret_cast<const float4*>(xrow + e * 4 * C::XPITCH);
            if (z > 0) {
              a[e].x += v.x;
              a[e].y += v.y;
              a[e].z += v.z;
              a[e].w += v.w;
            } else {
              a[e] = v;
            }
            if (!fin) {
              __stcg(reinterpret_cast<float4*>(srow + e * 4 * 256), a[e]);
            } else if (mrow0 + e * 4 + (lane >> 3) < p.M && n < p.N) {
              *reinterpret_cast<float4*>(hrow + static_cast<size_t>(e) * 4 * p.ldo) =
                  make_float4(hv[e].x + a[e].x, hv[e].y + a[e].y, hv[e].z + a[e].z, hv[e].w + a[e].w);
            }
          }
          __syncwarp();
        }
       }
      }
      if (EPI != EPI_SUMRES || !p.sum_tmem) release(b);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, C::TMEM_COLS);
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

int make_kv_map(CUtensorMap* map, const void* kv, int64_t rows, int head_dim) {
  RLB_CHECK(head_dim % BK == 0 && rows < (int64_t{1} << 31), RLB_ERR_ARG,
            "KV map: head_dim multiple of 64, < 2^31 rows");
  return make_kmajor_map3(map, kv, rows, head_dim, 16, head_dim / BK);
}

// 3D view of a K-major [rows, k] bf16 matrix: (64 elements, rows, k / 64
// K blocks), boxes of box_rows rows x kps K blocks (gemm_bf16_tc<..., KPS>)
int make_kmajor_map3(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int box_rows,
                     int kps) {
  PFN_encodeTiled_t enc = encode_fn();
  RLB_CHECK(enc != nullptr, RLB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  RLB_CHECK(k % BK == 0, RLB_ERR_ARG, "GEMM K must be a multiple of 64");
  RLB_CHECK((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, RLB_ERR_ARG, "TMA base not 16B aligned");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(BK), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(k / BK)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(k * 2), static_cast<cuuint64_t>(BK * 2)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows),
                       static_cast<cuuint32_t>(kps)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RLB_CHECK(r == CUDA_SUCCESS, RLB_ERR_CUDA, "cuTensorMapEncodeTiled (3D) failed: " + std::to_string(r));
  return RLB_OK;
}

template <int BN, int EPI, int NACC, int KPS = 1>
static int set_attr() {
  RLB_CUDA(cudaFuncSetAttribute(gemm_bf16_tc<BN, EPI, NACC, KPS>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                GemmCfg<BN, NACC, KPS>::SMEM));
  return RLB_OK;
}

template <int BN, int NACC>
static int set_attr_bn() {
  int rc;
  if ((rc = set_attr<BN, EPI_BF16, NACC>()) || (rc = set_attr<BN, EPI_RESADD, NACC>()) ||
      (rc = set_attr<BN, EPI_F32, NACC>()) || (rc = set_attr<BN, EPI_ARGMAX, NACC>()) ||
      (rc = set_attr<BN, EPI_SWIGLU, NACC>()) || (rc = set_attr<BN, EPI_PARTIAL, NACC>()))
    return rc;
  if constexpr (BN == 128) {
    if ((rc = set_attr<BN, EPI_ROPE, NACC>())) return rc;
  }
  return RLB_OK;
}

int gemm_prepare() {
  static bool done[64] = {false};
  int dev = 0;
  RLB_CUDA(cudaGetDevice(&dev));
  if (done[dev & 63]) return RLB_OK;
  int rc;
  if ((rc = set_attr_bn<128, 2>()) || (rc = set_attr_bn<256, 2>()) || (rc = set_attr_bn<128, 1>()) ||
      (rc = set_attr_bn<256, 1>()) ||
      (rc = set_attr<64, EPI_ROPE, 1>()) || (rc = set_attr<64, EPI_ROPE, 1, 2>()) ||
      (rc = set_attr<128, EPI_PARTIAL, 1, 2>()))
    return rc;
  RLB_CUDA(cudaFuncSetAttribute(gemm_pairp_tc<EPI_SWIGLU>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, PairPCfg<EPI_SWIGLU>::SMEM));
  RLB_CUDA(cudaFuncSetAttribute(gemm_pairp_tc<EPI_ARGMAX>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, PairPCfg<EPI_ARGMAX>::SMEM));
  RLB_CUDA(cudaFuncSetAttribute(gemm_pairp_tc<EPI_ROPE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, PairPCfg<EPI_ROPE>::SMEM));
  RLB_CUDA(cudaFuncSetAttribute(gemm_pairp_tc<EPI_PARTIAL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, PairPCfg<EPI_PARTIAL>::SMEM));
  RLB_CUDA(cudaFuncSetAttribute(gemm_pairp_tc<EPI_SUMRES>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, PairPCfg<EPI_SUMRES>::SMEM));
  done[dev & 63] = true;
  return RLB_OK;
}

template <int BN, int EPI, int NACC, int KPS = 1>
static int launch_one(const CUtensorMap& a, const CUtensorMap& b, const GemmParams& p,
                      cudaStream_t st) {
  using C = GemmCfg<BN, NACC, KPS>;
  RLB_CHECK((p.N + BN - 1) / BN <= 65535, RLB_ERR_ARG, "too many N tiles");
  dim3 grid((p.M + C::BMT - 1) / C::BMT, (p.N + BN - 1) / BN, p.splits);
  const bool split_cluster = cluster_epi(EPI) && BN == 128 && p.splits > 1;
  if (split_cluster) {   // split-K CTAs of a tile (DSMEM reduction)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = static_cast<unsigned>(p.splits);
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled(RLB_PDL_CLASS) ? 2 : 1;
    RLB_CUDA(cudaLaunchKernelEx(&cfg, gemm_bf16_tc<BN, EPI, NACC, KPS>, a, b, p));
    return RLB_OK;
  }
  RLB_CUDA(launch_k(gemm_bf16_tc<BN, EPI, NACC, KPS>, grid, dim3(GEMM_THREADS), C::SMEM, st, a, b,
                    p));
  return RLB_OK;
}

template <int BN, int NACC>
static int launch_bn(const CUtensorMap& a, const CUtensorMap& b, int epi, const GemmParams& p,
                     cudaStream_t st) {
  switch (epi) {
    case EPI_BF16: return launch_one<BN, EPI_BF16, NACC>(a, b, p, st);
    case EPI_RESADD: return launch_one<BN, EPI_RESADD, NACC>(a, b, p, st);
    case EPI_SWIGLU: return launch_one<BN, EPI_SWIGLU, NACC>(a, b, p, st);
    case EPI_F32: return launch_one<BN, EPI_F32, NACC>(a, b, p, st);
    case EPI_ARGMAX: return launch_one<BN, EPI_ARGMAX, NACC>(a, b, p, st);
    case EPI_PARTIAL: return launch_one<BN, EPI_PARTIAL, NACC>(a, b, p, st);
    case EPI_ROPE:
      if constexpr (BN == 128) return launch_one<BN, EPI_ROPE, NACC>(a, b, p, st);
      break;
  }
  set_error("bad epilogue");
  return RLB_ERR_ARG;
}

int gemm_launch(const CUtensorMap& a, const CUtensorMap& b, int block_n, int epi,
                const GemmParams& p, cudaStream_t st, int block_m, int a_multicast, int kps) {
  RLB_CHECK(kps == 1 || (a_multicast == 1 && ((block_n == 64 && epi == EPI_ROPE) ||
                                                (block_n == 128 && block_m == 128 &&
                                                 epi == EPI_PARTIAL))),
            RLB_ERR_ARG, "2 K blocks per stage: 64-column RoPE or 128 x 128 partial tiles");
  if (kps == 2 && epi == EPI_PARTIAL) {
    RLB_CHECK(p.ws != nullptr && p.K % BK == 0 && p.K / BK >= p.splits, RLB_ERR_ARG,
              "split-K partials need a workspace");
    return launch_one<128, EPI_PARTIAL, 1, 2>(a, b, p, st);
  }
  if (p.M <= 0) return RLB_OK;
  RLB_CHECK(a_multicast == 1, RLB_ERR_ARG, "A multicast is not built (measured slower)");
  RLB_CHECK(p.K % BK == 0 && p.N % 16 == 0, RLB_ERR_ARG, "GEMM shape not tileable");
  RLB_CHECK(p.splits >= 1 && p.K / BK >= p.splits, RLB_ERR_ARG,
            "split-K needs at least one K block per split");
  RLB_CHECK(p.splits == 1 || (epi == EPI_PARTIAL && p.ws != nullptr) ||
                (cluster_epi(epi) && block_n == 128 && p.splits <= 8),
            RLB_ERR_ARG,
            "split-K needs EPI_PARTIAL (workspace) or a cluster epilogue (BN=128, <= 8 splits)");
  RLB_CHECK(epi != EPI_ROPE || ((block_n == 128 || block_n == 64) && p.bias != nullptr &&
                                p.N % block_n == 0 && (p.rope.d == 64 || p.rope.d == 128)),
            RLB_ERR_ARG, "EPI_ROPE needs 64/128-column tiles, head_dim 64/128 and a bias");
  if (block_n == 64) {   // the narrow tile exists for single-split RoPE (decode QKV)
    RLB_CHECK(epi == EPI_ROPE && block_m == 128 && p.splits == 1, RLB_ERR_ARG,
              "64-column tiles: RoPE epilogue, 128-row tiles, no split");
    if (kps == 2) return launch_one<64, EPI_ROPE, 1, 2>(a, b, p, st);   // 3D-box maps
    return launch_one<64, EPI_ROPE, 1>(a, b, p, st);
  }
  RLB_CHECK(epi != EPI_SWIGLU || (block_n % 128 == 0 && p.N % 128 == 0), RLB_ERR_ARG,
            "SwiGLU GEMM needs 128-column gate/up tiles");
  RLB_CHECK(block_m == 128 || block_m == 256, RLB_ERR_ARG, "block_m must be 128 or 256");
  const bool two = block_m == 256;
  switch (block_n) {
    case 128: return two ? launch_bn<128, 2>(a, b, epi, p, st) : launch_bn<128, 1>(a, b, epi, p, st);
    case 256: return two ? launch_bn<256, 2>(a, b, epi, p, st) : launch_bn<256, 1>(a, b, epi, p, st);
  }
  set_error("block_n must be 128 or 256");
  return RLB_ERR_ARG;
}

// Persistent 2-SM pair tiles (256 x 256 per cluster, double-buffered TMEM).
int pairp_units(int epi, int M, int N, int splits) {
  const int tiles = ((M + 255) / 256) * ((N + 255) / 256);
  return epi == EPI_PARTIAL ? tiles * splits : tiles;
}

size_t pairp_sumres_scratch(int splits) {
  int dev = 0, n_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    n_sm = 148;
  return splits > 1 ? static_cast<size_t>(n_sm / 2) * 2 * 128 * 256 : 0;
}

int gemm_launch_pairp(const CUtensorMap& a, const CUtensorMap& b128, int epi, const GemmParams& p,
                      cudaStream_t st) {
  if (p.M <= 0) return RLB_OK;
  const bool split_epi = epi == EPI_PARTIAL || epi == EPI_SUMRES;
  RLB_CHECK(p.K % BK == 0 && (p.splits == 1 || split_epi), RLB_ERR_ARG,
            "persistent pair GEMM: K multiple of 64, split-K only with fp32 partials");
  RLB_CHECK(epi == EPI_SWIGLU || epi == EPI_ARGMAX ||
                (epi == EPI_ROPE && p.splits == 1 && p.bias != nullptr && p.N % 256 == 0 &&
                 (p.rope.d == 64 || p.rope.d == 128)) ||
                (split_epi && p.ws != nullptr && p.splits >= 1 && p.K / BK >= p.splits) ,
            RLB_ERR_ARG, "persistent pair GEMM epilogues: SwiGLU, argmax, RoPE, fp32 partials");
  RLB_CHECK(epi != EPI_SUMRES || (p.out != nullptr && p.N % 4 == 0 && p.ldo % 4 == 0),
            RLB_ERR_ARG, "split-sum pair GEMM: fp32 residual rows, 16-byte aligned");
  RLB_CHECK(epi != EPI_SWIGLU || p.N % 256 == 0, RLB_ERR_ARG, "SwiGLU pair tiles are 256 wide");
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    RLB_CUDA(cudaGetDevice(&dev));
    RLB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  }
  const int clusters = std::min(pairp_units(epi, p.M, p.N, p.splits), n_sm / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters, 1, 1);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = split_epi ? PairPCfg<EPI_PARTIAL>::SMEM : PairPCfg<EPI_SWIGLU>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(RLB_PDL_CLASS) ? 2 : 1;
  if (epi == EPI_SWIGLU) RLB_CUDA(cudaLaunchKernelEx(&cfg, gemm_pairp_tc<EPI_SWIGLU>, a, b128, p));
  else if (epi == EPI_PARTIAL) RLB_CUDA(cudaLaunchKernelEx(&cfg, gemm_pairp_tc<EPI_PARTIAL>, a, b128, p));
  else if (epi == EPI_SUMRES) RLB_CUDA(cudaLaunchKernelEx(&cfg, gemm_pairp_tc<EPI_SUMRES>, a, b128, p));
  else if (epi == EPI_ROPE) RLB_CUDA(cudaLaunchKernelEx(&cfg, gemm_pairp_tc<EPI_ROPE>, a, b128, p));
  else RLB_CUDA(cudaLaunchKernelEx(&cfg, gemm_pairp_tc<EPI_ARGMAX>, a, b128, p));
  return RLB_OK;
}

}  // namespace rlb

// Microbenchmark: `iters` back-to-back launches of one GEMM configuration on
// scratch buffers, timed with CUDA events (tile / split tuning).
extern "C" int rlb_bench_gemm(int device, int32_t M, int32_t N, int32_t K, int32_t epilogue,
                              int32_t block_n, int32_t splits, int32_t block_m, int32_t iters,
                              double* avg_ms) {
  using namespace rlb;
  RLB_CUDA(cudaSetDevice(device));
  int rc = gemm_prepare();
  if (rc) return rc;
  bf16 *A = nullptr, *B = nullptr;
  float* C = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  struct Scratch {   // released on every return path
    bf16** a;
    bf16** b;
    float** c;
    cudaEvent_t* e0;
    cudaEvent_t* e1;
    ~Scratch() {
      cudaFree(*a);
      cudaFree(*b);
      cudaFree(*c);
      if (*e0) cudaEventDestroy(*e0);
      if (*e1) cudaEventDestroy(*e1);
    }
  } scratch{&A, &B, &C, &e0, &e1};
  const int S = splits < 1 ? 1 : splits;
  RLB_CUDA(cudaMalloc(&A, sizeof(bf16) * static_cast<size_t>(M) * K));
  RLB_CUDA(cudaMalloc(&B, sizeof(bf16) * static_cast<size_t>(N) * K));
  RLB_CUDA(cudaMalloc(&C, sizeof(float) * static_cast<size_t>(S) * M * N));
  RLB_CUDA(cudaMemset(A, 0, sizeof(bf16) * static_cast<size_t>(M) * K));
  RLB_CUDA(cudaMemset(B, 0, sizeof(bf16) * static_cast<size_t>(N) * K));
  CUtensorMap ma, mb;
  if ((rc = make_kmajor_map(&ma, A, M, K, HM)) || (rc = make_kmajor_map(&mb, B, N, K, block_n)))
    return rc;
  GemmParams p{M, N, K, nullptr, C, epilogue == EPI_SWIGLU ? N / 2 : N, S, C};
  if (epilogue == EPI_ARGMAX) p.ldo = (N + block_n - 1) / block_n;
  RLB_CHECK(epilogue != EPI_ROPE, RLB_ERR_ARG, "EPI_ROPE needs an instance (rlb_profile_kernel)");
  const int epi = S > 1 && !cluster_epi(epilogue) ? static_cast<int>(EPI_PARTIAL) : epilogue;
  RLB_CUDA(cudaEventCreate(&e0));
  RLB_CUDA(cudaEventCreate(&e1));
  const bool pair = std::getenv("RLB_GEMM_PAIR") != nullptr;   // persistent 2-SM tiles
  CUtensorMap mb128;
  if (pair && (rc = make_kmajor_map(&mb128, B, N, K, 128))) return rc;
  auto go = [&]() {
    return pair ? gemm_launch_pairp(ma, mb128, epi, p, 0)
                : gemm_launch(ma, mb, block_n, epi, p, 0, block_m);
  };
  if ((rc = go())) return rc;
  RLB_CUDA(cudaEventRecord(e0, 0));
  for (int i = 0; i < iters && !rc; ++i) rc = go();
  RLB_CUDA(cudaEventRecord(e1, 0));
  RLB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  RLB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *avg_ms = ms / iters;
  if (std::getenv("RLB_GEMM_DBG")) {   // latency breakdown of CTA 0 of one more launch
    unsigned long long* d = nullptr;
    unsigned long long h[8] = {0};
    RLB_CUDA(cudaMalloc(&d, sizeof(h)));
    RLB_CUDA(cudaMemset(d, 0, sizeof(h)));
    p.dbg = d;
    rc = go();
    RLB_CUDA(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "gemm dbg (ns from CTA start): setup %lld wait %lld mma_done %lld "
                 "epi_start %lld epi_end %lld dealloc %lld\n",
                 (long long)(h[1] - h[0]), (long long)(h[2] - h[0]), (long long)(h[3] - h[0]),
                 (long long)(h[4] - h[0]), (long long)(h[6] - h[0]), (long long)(h[5] - h[0]));
    cudaFree(d);
  }
  return rc;
}

extern "C" int rlb_gemm(int device, int32_t M, int32_t N, int32_t K, const void* A, const void* B,
                        const void* bias, void* Cout, int32_t epilogue, int32_t block_n,
                        int32_t splits, int32_t block_m) {
  using namespace rlb;
  RLB_CUDA(cudaSetDevice(device));
  int rc = gemm_prepare();
  if (rc) return rc;
  CUtensorMap ma, mb;
  rc = make_kmajor_map(&ma, A, M, K, HM);
  if (rc) return rc;
  rc = make_kmajor_map(&mb, B, N, K, block_n);
  if (rc) return rc;
  GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.bias = static_cast<const bf16*>(bias);
  p.out = Cout;
  p.ldo = epilogue == EPI_SWIGLU ? N / 2 : N;
  p.splits = splits < 1 ? 1 : splits;
  // (test entry) RLB_GEMM_PAIR: the persistent 2-SM tiles instead of the
  // single-SM kernel -- the same bits (tests/test_gpu_kernels.py)
  if (std::getenv("RLB_GEMM_PAIR") && p.splits == 1) {
    CUtensorMap mb128;
    rc = make_kmajor_map(&mb128, B, N, K, 128);
    if (!rc) rc = gemm_launch_pairp(ma, mb128, epilogue, p, 0);
  } else if (p.splits == 1 || (epilogue == EPI_RESADD && block_n == 128)) {
    rc = gemm_launch(ma, mb, block_n, epilogue, p, 0, block_m);   // RESADD: cluster split-K
  } else {
    RLB_CUDA(cudaMalloc(&p.ws, sizeof(float) * static_cast<size_t>(p.splits) * M * N));
    if (std::getenv("RLB_GEMM_PAIR")) {   // persistent 2-SM tiles, split-K partials
      CUtensorMap mb128;
      rc = make_kmajor_map(&mb128, B, N, K, 128);
      if (!rc) rc = gemm_launch_pairp(ma, mb128, EPI_PARTIAL, p, 0);
    } else {
      rc = gemm_launch(ma, mb, block_n, EPI_PARTIAL, p, 0, block_m);
    }
    if (!rc) {
      switch (epilogue) {
        case EPI_BF16: splitk_reduce_kernel<EPI_BF16><<<M, 256>>>(p); break;
        case EPI_RESADD: splitk_reduce_kernel<EPI_RESADD><<<M, 256>>>(p); break;
        case EPI_F32: splitk_reduce_kernel<EPI_F32><<<M, 256>>>(p); break;
        default: set_error("split-K supports epilogues 0, 1, 3"); rc = RLB_ERR_ARG;
      }
    }
    cudaDeviceSynchronize();
    cudaFree(p.ws);
  }
  if (rc) return rc;
  RLB_CUDA(cudaDeviceSynchronize());
  return RLB_OK;
}
