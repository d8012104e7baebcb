// K7: pull-based weight transfer with the HF -> engine re-layout fused into
// the copy.
//
// Reference: the pull is a modelled byte count shared over agent egress /
// instance ingress (pkg/src/spotrl/transfer.py:87-170) and, in live mode, a
// framed byte stream whose payload is the concatenated weights
// (pkg/src/spotrl/protocol.py:92-157).  Here the bytes are real: a receiver
// reads the trainer's bf16 tensors (local, or a peer GPU's memory mapped via
// CUDA IPC so the loads travel over NVLink) and writes its engine arena.
// Every re-layout piece is a contiguous byte range (fused QKV rows, 64-row
// gate/up interleave blocks), so the whole pull is one chunked copy kernel:
// 16-byte vector loads, 4 in flight per thread, L1 no-allocate.
#include "internal.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace rlb {

static int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }

int32_t hf_count(const rlb_model_cfg& m) { return 1 + 12 * m.layers + 1 + (m.tied ? 0 : 1); }

// Mirrors paper_2510_19225_b200/shapes.py engine_layout(): arena offsets of
// each engine tensor in carve order.
struct ArenaCursor {
  int64_t off = 0;
  int64_t put(int64_t elems) {
    const int64_t at = off;
    off = align256(off + 2 * elems);
    return at;
  }
};

int64_t arena_bytes(const rlb_model_cfg& m) {
  ArenaCursor c;
  const int64_t H = m.hidden, QD = static_cast<int64_t>(m.n_q_heads) * m.head_dim,
                KD = static_cast<int64_t>(m.n_kv_heads) * m.head_dim, F = m.ffn;
  c.put(static_cast<int64_t>(m.vocab) * H);
  for (int i = 0; i < m.layers; ++i) {
    c.put(H);
    c.put((QD + 2 * KD) * H);
    c.put(QD + 2 * KD);
    c.put(H * QD);
    c.put(H);
    c.put(2 * F * H);
    c.put(H * F);
  }
  c.put(H);
  if (!m.tied) c.put(static_cast<int64_t>(m.vocab) * H);
  return c.off;
}

void relayout_segments(const rlb_model_cfg& m, std::vector<Segment>* out) {
  out->clear();
  const int64_t H = m.hidden, QD = static_cast<int64_t>(m.n_q_heads) * m.head_dim,
                KD = static_cast<int64_t>(m.n_kv_heads) * m.head_dim, F = m.ffn;
  constexpr int64_t GU = 64;
  ArenaCursor c;
  int32_t hf = 0;
  auto seg = [&](int32_t h, int64_t so, int64_t d, int64_t b) { out->push_back({h, so, d, b}); };
  int64_t e = c.put(static_cast<int64_t>(m.vocab) * H);
  seg(hf++, 0, e, 2 * m.vocab * H);
  for (int i = 0; i < m.layers; ++i) {
    const int64_t ln1 = c.put(H), wqkv = c.put((QD + 2 * KD) * H), bqkv = c.put(QD + 2 * KD),
                  wo = c.put(H * QD), ln2 = c.put(H), wgu = c.put(2 * F * H), wd = c.put(H * F);
    const int32_t base = hf;  // ln1 q qb k kb v vb o ln2 gate up down
    seg(base + 0, 0, ln1, 2 * H);
    // q / k / v heads in 32-row pieces: each 64-row block = 32 rows of the
    // first rotation half + their partners (row + D/2), so a 64-column GEMM
    // tile holds whole RoPE pairs (identity for D = 64)
    const int64_t D = m.head_dim, hd = D / 2, P = 32;
    int64_t row0 = 0;
    const int heads[3] = {m.n_q_heads, m.n_kv_heads, m.n_kv_heads};
    for (int pj = 0; pj < 3; ++pj) {
      const int32_t wi = base + 1 + 2 * pj, bi = base + 2 + 2 * pj;
      for (int64_t hh = 0; hh < heads[pj]; ++hh)
        for (int64_t t = 0; t < hd / P; ++t)
          for (int half = 0; half < 2; ++half) {
            const int64_t r_src = hh * D + half * hd + t * P;
            const int64_t r_dst = row0 + hh * D + (2 * t + half) * P;
            seg(wi, 2 * r_src * H, wqkv + 2 * r_dst * H, 2 * P * H);
            seg(bi, 2 * r_src, bqkv + 2 * r_dst, 2 * P);
          }
      row0 += heads[pj] * D;
    }
    seg(base + 7, 0, wo, 2 * H * QD);
    seg(base + 8, 0, ln2, 2 * H);
    const int64_t blk = 2 * GU * H;
    for (int64_t b = 0; b < F / GU; ++b) {
      seg(base + 9, b * blk, wgu + (2 * b) * blk, blk);
      seg(base + 10, b * blk, wgu + (2 * b + 1) * blk, blk);
    }
    seg(base + 11, 0, wd, 2 * H * F);
    hf += 12;
  }
  seg(hf++, 0, c.put(H), 2 * H);
  if (!m.tied) seg(hf++, 0, c.put(static_cast<int64_t>(m.vocab) * H), 2 * m.vocab * H);
}

struct CopyChunk {
  const uint8_t* src;
  uint8_t* dst;
  int64_t bytes;
};

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

constexpr int COPY_THREADS = 512;
constexpr int COPY_UNROLL = 4;
constexpr int64_t CHUNK_BYTES = 1 << 20;

__global__ void __launch_bounds__(COPY_THREADS) chunk_copy_kernel(const CopyChunk* __restrict__ ch,
                                                                 int n) {
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const CopyChunk k = ch[c];
    const int64_t nv = k.bytes >> 4;
    const uint4* s = reinterpret_cast<const uint4*>(k.src);
    uint4* d = reinterpret_cast<uint4*>(k.dst);
    int64_t i = threadIdx.x;
    for (; i + (COPY_UNROLL - 1) * COPY_THREADS < nv; i += COPY_UNROLL * COPY_THREADS) {
      uint4 v[COPY_UNROLL];
#pragma unroll
      for (int u = 0; u < COPY_UNROLL; ++u) v[u] = ld_stream(s + i + u * COPY_THREADS);
#pragma unroll
      for (int u = 0; u < COPY_UNROLL; ++u) d[i + u * COPY_THREADS] = v[u];
    }
    for (; i < nv; i += COPY_THREADS) d[i] = ld_stream(s + i);
    // byte tail (never hit for bf16 tensors of the supported shapes)
    for (int64_t b = (nv << 4) + threadIdx.x; b < k.bytes; b += COPY_THREADS) k.dst[b] = k.src[b];
  }
}

static int run_chunks(const std::vector<CopyChunk>& chunks, cudaStream_t st) {
  if (chunks.empty()) return RLB_OK;
  CopyChunk* d = nullptr;
  const size_t bytes = chunks.size() * sizeof(CopyChunk);
  int sms = 148, dev = 0;
  RLB_CUDA(cudaGetDevice(&dev));
  RLB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int cap = sms * 4;
  if (const char* c = std::getenv("RLB_COPY_CTAS")) cap = std::max(1, std::atoi(c));
  const int grid = static_cast<int>(std::min<size_t>(chunks.size(), static_cast<size_t>(cap)));
  RLB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), bytes, st));
  // the chunk list is freed stream-ordered on every path once it is allocated
  cudaError_t e = cudaMemcpyAsync(d, chunks.data(), bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    chunk_copy_kernel<<<grid, COPY_THREADS, 0, st>>>(d, static_cast<int>(chunks.size()));
    e = cudaGetLastError();
  }
  const cudaError_t ef = cudaFreeAsync(d, st);
  RLB_CUDA(e);
  RLB_CUDA(ef);
  return RLB_OK;
}

static void split_into(std::vector<CopyChunk>* v, const uint8_t* s, uint8_t* d, int64_t bytes) {
  for (int64_t o = 0; o < bytes; o += CHUNK_BYTES)
    v->push_back({s + o, d + o, std::min<int64_t>(CHUNK_BYTES, bytes - o)});
}

int relayout_copy(const rlb_model_cfg& m, const void* const* hf_ptrs, int32_t n, void* dst,
                  cudaStream_t st) {
  RLB_CHECK(n == hf_count(m), RLB_ERR_ARG,
            "expected " + std::to_string(hf_count(m)) + " HF tensors, got " + std::to_string(n));
  std::vector<Segment> segs;
  relayout_segments(m, &segs);
  std::vector<CopyChunk> chunks;
  chunks.reserve(segs.size() + 16384);
  for (const Segment& s : segs) {
    const uint8_t* src = static_cast<const uint8_t*>(hf_ptrs[s.hf]) + s.src_off;
    uint8_t* d = static_cast<uint8_t*>(dst) + s.dst_off;
    RLB_CHECK(((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(d)) & 15) == 0,
              RLB_ERR_ARG, "weight tensors must be 16-byte aligned");
    split_into(&chunks, src, d, s.bytes);
  }
  return run_chunks(chunks, st);
}

// The part of the fused re-layout that lands in arena bytes [lo, hi): used by
// the scatter phase of the 1->N fan-out (each receiver pulls one slice).
int relayout_copy_range(const rlb_model_cfg& m, const void* const* hf_ptrs, int32_t n, void* dst,
                        int64_t lo, int64_t hi, cudaStream_t st) {
  RLB_CHECK(n == hf_count(m), RLB_ERR_ARG, "wrong HF tensor count");
  RLB_CHECK(lo % 16 == 0 && hi % 16 == 0 && lo <= hi, RLB_ERR_ARG, "range must be 16B aligned");
  std::vector<Segment> segs;
  relayout_segments(m, &segs);
  std::vector<CopyChunk> chunks;
  for (const Segment& s : segs) {
    const int64_t a = std::max(lo, s.dst_off), b = std::min(hi, s.dst_off + s.bytes);
    if (a >= b) continue;
    const uint8_t* src = static_cast<const uint8_t*>(hf_ptrs[s.hf]) + s.src_off + (a - s.dst_off);
    uint8_t* d = static_cast<uint8_t*>(dst) + a;
    RLB_CHECK(((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(d)) & 15) == 0,
              RLB_ERR_ARG, "weight tensors must be 16-byte aligned");
    split_into(&chunks, src, d, b - a);
  }
  return run_chunks(chunks, st);
}

int copy_bytes(void* dst, const void* src, int64_t nbytes, cudaStream_t st) {
  RLB_CHECK(((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0,
            RLB_ERR_ARG, "copy buffers must be 16-byte aligned");
  std::vector<CopyChunk> chunks;
  split_into(&chunks, static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), nbytes);
  return run_chunks(chunks, st);
}

}  // namespace rlb

extern "C" {

int64_t rlb_arena_bytes(const rlb_model_cfg* m) { return m ? rlb::arena_bytes(*m) : -1; }

int32_t rlb_hf_tensor_count(const rlb_model_cfg* m) { return m ? rlb::hf_count(*m) : -1; }

int64_t rlb_relayout_table(const rlb_model_cfg* m, int64_t* out, int64_t cap) {
  if (!m) return RLB_ERR_ARG;
  std::vector<rlb::Segment> segs;
  rlb::relayout_segments(*m, &segs);
  for (int64_t i = 0; i < static_cast<int64_t>(segs.size()) && i < cap; ++i) {
    out[4 * i] = segs[i].hf;
    out[4 * i + 1] = segs[i].src_off;
    out[4 * i + 2] = segs[i].dst_off;
    out[4 * i + 3] = segs[i].bytes;
  }
  return static_cast<int64_t>(segs.size());
}

int rlb_relayout_copy(int device, const rlb_model_cfg* m, const void* const* hf_ptrs,
                      int32_t n_tensors, void* dst_arena, void* stream) {
  RLB_CHECK(m && hf_ptrs && dst_arena, RLB_ERR_ARG, "null argument");
  RLB_CUDA(cudaSetDevice(device));
  return rlb::relayout_copy(*m, hf_ptrs, n_tensors, dst_arena, static_cast<cudaStream_t>(stream));
}

// ---- NCCL broadcast fan-out (libnccl resolved at runtime; no link dependency)
namespace {
struct NcclApi {
  ncclResult_t (*unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                        cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*err)(ncclResult_t) = nullptr;
  bool ok = false;
};
NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.unique_id = reinterpret_cast<decltype(api.unique_id)>(dlsym(h, "ncclGetUniqueId"));
      api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.bcast = reinterpret_cast<decltype(api.bcast)>(dlsym(h, "ncclBroadcast"));
      api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
      api.err = reinterpret_cast<decltype(api.err)>(dlsym(h, "ncclGetErrorString"));
      api.ok = api.unique_id && api.init_rank && api.bcast && api.destroy && api.err;
    }
  }
  return &api;
}
}  // namespace

#define RLB_NCCL(call)                                                              \
  do {                                                                              \
    ncclResult_t _r = (call);                                                       \
    if (_r != ncclSuccess) {                                                        \
      rlb::set_error(std::string("NCCL: ") + nccl_api()->err(_r));                  \
      return RLB_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

int rlb_nccl_unique_id(uint8_t out[128]) {
  NcclApi* a = nccl_api();
  RLB_CHECK(a->ok, RLB_ERR_CUDA, "libnccl.so.2 not available");
  ncclUniqueId id;
  RLB_NCCL(a->unique_id(&id));
  memcpy(out, &id, sizeof(id) < 128 ? sizeof(id) : 128);
  return RLB_OK;
}

int rlb_nccl_init(int device, int nranks, int rank, const uint8_t id[128], void** comm) {
  NcclApi* a = nccl_api();
  RLB_CHECK(a->ok, RLB_ERR_CUDA, "libnccl.so.2 not available");
  RLB_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  RLB_NCCL(a->init_rank(&c, nranks, uid, rank));
  *comm = c;
  return RLB_OK;
}

int rlb_nccl_broadcast(void* comm, void* buf, int64_t nbytes, int root, void* stream) {
  NcclApi* a = nccl_api();
  RLB_CHECK(a->ok && comm, RLB_ERR_ARG, "no NCCL communicator");
  RLB_NCCL(a->bcast(buf, buf, static_cast<size_t>(nbytes), ncclUint8, root,
                    static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)));
  return RLB_OK;
}

int rlb_nccl_destroy(void* comm) {
  NcclApi* a = nccl_api();
  if (a->ok && comm) RLB_NCCL(a->destroy(static_cast<ncclComm_t>(comm)));
  return RLB_OK;
}

int rlb_enable_peer(int device, int peer) {
  RLB_CUDA(cudaSetDevice(device));
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return RLB_OK;
  }
  RLB_CUDA(e);
  return RLB_OK;
}

int rlb_relayout_copy_range(int device, const rlb_model_cfg* m, const void* const* hf_ptrs,
                            int32_t n_tensors, void* dst_arena, int64_t lo, int64_t hi,
                            void* stream) {
  RLB_CHECK(m && hf_ptrs && dst_arena, RLB_ERR_ARG, "null argument");
  RLB_CUDA(cudaSetDevice(device));
  return rlb::relayout_copy_range(*m, hf_ptrs, n_tensors, dst_arena, lo, hi,
                                  static_cast<cudaStream_t>(stream));
}

int rlb_copy_segments(int device, int32_t n, const void* const* src, void* const* dst,
                      const int64_t* nbytes, void* stream) {
  RLB_CHECK(n >= 0 && (n == 0 || (src && dst && nbytes)), RLB_ERR_ARG, "bad segment list");
  RLB_CUDA(cudaSetDevice(device));
  std::vector<rlb::CopyChunk> chunks;
  for (int32_t i = 0; i < n; ++i) {
    RLB_CHECK(((reinterpret_cast<uintptr_t>(src[i]) | reinterpret_cast<uintptr_t>(dst[i])) & 15) == 0,
              RLB_ERR_ARG, "segments must be 16-byte aligned");
    rlb::split_into(&chunks, static_cast<const uint8_t*>(src[i]), static_cast<uint8_t*>(dst[i]),
                    nbytes[i]);
  }
  return rlb::run_chunks(chunks, static_cast<cudaStream_t>(stream));
}

int rlb_copy_bytes(int device, void* dst, const void* src, int64_t nbytes, void* stream) {
  RLB_CHECK(dst && src && nbytes >= 0, RLB_ERR_ARG, "bad copy arguments");
  RLB_CUDA(cudaSetDevice(device));
  return rlb::copy_bytes(dst, src, nbytes, static_cast<cudaStream_t>(stream));
}

int rlb_ipc_handle(const void* dev_ptr, uint8_t out_handle[64], int64_t* out_offset) {
  // The handle names the whole allocation; report where dev_ptr sits in it
  // (allocations from a caching allocator are sub-ranges of a segment).
  typedef CUresult (*PFN_range)(CUdeviceptr*, size_t*, CUdeviceptr);
  static PFN_range range_fn = nullptr;
  if (range_fn == nullptr) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      range_fn = reinterpret_cast<PFN_range>(fp);
  }
  RLB_CHECK(range_fn != nullptr, RLB_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  RLB_CHECK(range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) == CUDA_SUCCESS,
            RLB_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  RLB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(out_handle, &h, 64);
  if (out_offset) *out_offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return RLB_OK;
}

int rlb_ipc_open(int device, const uint8_t handle[64], void** dev_ptr) {
  RLB_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  RLB_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return RLB_OK;
}

int rlb_ipc_close(int device, void* dev_ptr) {
  RLB_CUDA(cudaSetDevice(device));
  RLB_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return RLB_OK;
}

}  // extern "C"
