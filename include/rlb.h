/* librlb -- B200-native rollout data path of RLBoost (arXiv 2510.19225).
 *
 * C ABI: plain pointers and sizes, no torch types.  One opaque handle per
 * rollout instance (one GPU); a handle is not thread-safe (the reference's
 * single-writer rule, pkg/src/spotrl/manager.py:1-8); distinct
 * handles are independent.  Every function returns RLB_OK (0) or a negative
 * code; rlb_last_error() gives the thread-local message.  Host buffers are
 * owned by the caller; device memory is owned by the handle.
 *
 * Reference interfaces each entry point replaces (the reference is Python and
 * has no FFI; these are the call sites a binding plugs in under):
 *   rlb_instance_create/destroy -- the simulated rollout instance GenUnit
 *       (pkg/src/spotrl/sim/engine.py:63-83) + its rate model
 *       instance_throughput (pkg/src/spotrl/sim/models.py:39-48)
 *   rlb_submit / rlb_submit_varlen -- protocol `generate{request_id,
 *       prompt_tokens, prefix_tokens}` (pkg/src/spotrl/protocol.py:75-81) and the
 *       simulator's admit + prefill of prompt_len+len(generated)
 *       (pkg/src/spotrl/sim/engine.py:699-743)
 *   rlb_step -- the decode advance _sync_unit (pkg/src/spotrl/sim/engine.py:745-784)
 *       feeding RolloutManager.on_tokens/complete (pkg/src/spotrl/manager.py:295-334)
 *   rlb_cancel -- protocol `cancel{request_id}` (pkg/src/spotrl/protocol.py:84-85),
 *       the simulator's _detach_from_unit (pkg/src/spotrl/sim/engine.py:822-836)
 *   rlb_export_partials -- migrate_out keeping `generated`
 *       (pkg/src/spotrl/manager.py:336-357; RolloutRequest.generated,
 *       pkg/src/spotrl/domain.py:49)
 *   rlb_status -- protocol `status{m_pending, m_exec, weight_version}`
 *       (pkg/src/spotrl/protocol.py:26-31)
 *   rlb_load_weights / rlb_relayout_copy -- protocol `pull_weights{version,
 *       agent_endpoint}` (pkg/src/spotrl/protocol.py:88-89) and the pull session
 *       receive_weights (pkg/src/spotrl/protocol.py:143-157); TransferPool
 *       request_pull/finish (pkg/src/spotrl/transfer.py:87-140)
 */
#ifndef RLB_H_
#define RLB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RLB_OK 0
#define RLB_ERR_ARG (-1)      /* bad argument (ValueError) */
#define RLB_ERR_CUDA (-2)     /* CUDA runtime/driver failure */
#define RLB_ERR_STATE (-3)    /* unknown / duplicate request key, wrong state */
#define RLB_ERR_CAPACITY (-4) /* out of slots / KV pages / output capacity */

typedef struct rlb_instance rlb_instance;

typedef struct {
  int32_t vocab, hidden, layers, n_q_heads, n_kv_heads, head_dim, ffn, tied;
  float rope_theta, rms_eps;
} rlb_model_cfg;

typedef struct {
  int32_t max_slots;          /* concurrent sequences (decode batch) */
  int32_t max_seq_len;        /* prompt + generated tokens per sequence */
  int32_t num_pages;          /* KV pages of 64 tokens (one is reserved for the padding rows of
                                 bucketed decode batches); 0 = max_slots*ceil(max_seq_len/64)+1 */
  int32_t max_prefill_rows;   /* token rows per prefill chunk */
  int32_t graph_steps;        /* decode steps per captured CUDA graph; 0 = eager */
  /* Numerics plan: the split-K factors of the O and down projections fix the
   * order in which a row's dot products are summed, so they are part of the
   * bits an instance produces.  0 = the measured default for the shape.
   * Instances that migrate requests between them must share the plan
   * (rlb_numerics_plan). */
  int32_t split_o;
  int32_t split_down;
  int32_t reserved;
} rlb_engine_cfg;

/* Output of rlb_step: per request that produced tokens this call, its key,
 * the number of new tokens, whether it completed (reached target_len), and
 * the tokens themselves concatenated in entry order.  Arrays are caller-owned
 * (pinned host memory recommended). */
typedef struct {
  int32_t cap_entries;
  int64_t cap_tokens;
  uint64_t* keys;
  int32_t* counts;
  int32_t* done;
  int32_t* tokens;
  int32_t n_entries;  /* out */
  int64_t n_tokens;   /* out */
  int32_t steps_run;  /* out: decode steps executed */
  int32_t prefill_rows; /* out: prefill token rows executed */
} rlb_token_batch;

typedef struct {
  int64_t bytes;
  double seconds; /* copy-stream time of the pull (CUDA events) */
} rlb_pull_stats;

/* ---- instance lifecycle ------------------------------------------------ */
int rlb_instance_create(int device, const rlb_model_cfg* model, const rlb_engine_cfg* engine,
                        rlb_instance** out);
int rlb_instance_destroy(rlb_instance* h);
const char* rlb_last_error(void);

/* Everything that fixes the bits a row's arithmetic produces, as int32s:
 * [0] plan format version (2), [1] QKV split-K, [2] O split-K, [3] down
 * split-K, [4] attention positions per CTA window, [5] attention warps per
 * item (page p -> warp p mod warps), [6] positions per KV page, [7] greedy
 * tie rule (0 = lowest index).  Two instances whose plans are equal produce
 * identical ids for the same request whatever their batch, slot count or
 * tile shapes (those never change a row's bits); a resume across unequal
 * plans is not bit-exact.  Returns the number of ints (8), writes at most
 * cap. */
int32_t rlb_numerics_plan(const rlb_instance* h, int32_t* out, int32_t cap);

/* (test hook) The paged KV pool: device base pointer and bytes.  Bitwise
 * A/B checks of kernels that must not change a row's bits compare it. */
int rlb_kv_pool(rlb_instance* h, void** base, int64_t* bytes);

/* ---- weights (K7) ------------------------------------------------------ */
/* Engine-arena size in bytes for a model shape. */
int64_t rlb_arena_bytes(const rlb_model_cfg* model);
/* Number of HF tensors (canonical order, see paper_2510_19225_b200/shapes.py). */
int32_t rlb_hf_tensor_count(const rlb_model_cfg* model);
/* The fused re-layout as (hf_index, src_off, dst_off, nbytes) int64 quads;
 * returns the segment count, writes at most cap quads. */
int64_t rlb_relayout_table(const rlb_model_cfg* model, int64_t* out, int64_t cap);
/* Pull a full HF-layout weight set into the instance's engine arena with the
 * re-layout fused into the copy.  hf_ptrs are device pointers (local, or a
 * peer's memory mapped with rlb_ipc_open -- the copy then runs over NVLink).
 * ready_event (a cudaEvent_t, any device, or NULL): the copy waits on the
 * device until the producer of the source tensors recorded it (e.g. after the
 * trainer's optimizer step), so it never reads weights still being written.
 * Refused (RLB_ERR_STATE) while requests are on the instance: in-flight
 * sequences must not mix weight versions (use the shadow arena + swap).
 * Synchronous; the new version serves from the next rlb_step. */
int rlb_load_weights(rlb_instance* h, const void* const* hf_ptrs, int32_t n_tensors,
                     uint64_t version, void* ready_event, rlb_pull_stats* stats);
/* Engine arena device pointer + bytes (for bytewise checks / chained hops). */
int rlb_weights_arena(rlb_instance* h, void** arena, int64_t* bytes);
/* Declare the arena filled with `version` by an external copy (the fan-out
 * writes it with rlb_relayout_copy_range / rlb_copy_bytes).  Refused while
 * requests are on the instance, like rlb_load_weights. */
int rlb_mark_weights(rlb_instance* h, uint64_t version);

/* ---- double-buffered weights ------------------------
 * Replaces the pull lifecycle mark_pulling -> pull -> mark_active
 * (pkg/src/spotrl/sim/engine.py:597-656, manager.py:147-154): version v+1 is
 * pulled into a second (shadow) arena on the instance's copy stream while v
 * keeps serving, and swapped in at the step boundary (manager.begin_step,
 * manager.py:416-426) with no pull stall.
 *   rlb_shadow_arena   shadow arena pointer + bytes (allocated on first use;
 *                      the target of external fan-out / IPC / NCCL pulls)
 *   rlb_load_shadow    fused re-layout copy of HF tensors into the shadow,
 *                      enqueued on the copy stream after `ready_event` (the
 *                      producer's, or NULL); returns immediately
 *   rlb_mark_shadow    the shadow was filled externally by work enqueued on
 *                      `stream` (NULL = legacy default stream) with `version`
 *   rlb_shadow_status  state 0 empty / 1 copy in flight / 2 filled; seconds =
 *                      device time of an rlb_load_shadow copy once filled
 *   rlb_swap_weights   step boundary (no requests on the instance, else
 *                      RLB_ERR_STATE): the shadow becomes the active set (the
 *                      compute stream waits for its copy on the device), the
 *                      old set becomes the empty shadow; out = active version */
int rlb_shadow_arena(rlb_instance* h, void** arena, int64_t* bytes);
int rlb_load_shadow(rlb_instance* h, const void* const* hf_ptrs, int32_t n_tensors,
                    uint64_t version, void* ready_event);
int rlb_mark_shadow(rlb_instance* h, uint64_t version, void* stream);
int rlb_shadow_status(rlb_instance* h, uint64_t* version, int32_t* state, double* seconds);
int rlb_swap_weights(rlb_instance* h, uint64_t* version);
/* Stand-alone fused re-layout copy on `device` (stream 0 if stream==NULL). */
int rlb_relayout_copy(int device, const rlb_model_cfg* model, const void* const* hf_ptrs,
                      int32_t n_tensors, void* dst_arena, void* stream);
/* The slice of the fused re-layout that writes arena bytes [lo, hi) (16-byte
 * aligned): the scatter phase of the 1->N fan-out. */
int rlb_relayout_copy_range(int device, const rlb_model_cfg* model, const void* const* hf_ptrs,
                            int32_t n_tensors, void* dst_arena, int64_t lo, int64_t hi,
                            void* stream);
/* A list of byte-range copies (src[i] -> dst[i], nbytes[i]) as one chunked
 * copy kernel: the re-layout of one received piece of a broadcast blob. */
int rlb_copy_segments(int device, int32_t n, const void* const* src, void* const* dst,
                      const int64_t* nbytes, void* stream);
/* Plain chunked device copy (peer or local): the all-gather phase of the
 * fan-out copies engine-layout slices between rollout GPUs. */
int rlb_copy_bytes(int device, void* dst, const void* src, int64_t nbytes, void* stream);

/* NCCL broadcast fan-out of a staged engine-layout weight set (1->N pulls at
 * once): unique id (out: 128 bytes), per-rank communicator on `device`, in-place
 * byte broadcast from `root` on `stream`.  libnccl.so.2 is resolved at runtime. */
int rlb_nccl_unique_id(uint8_t out[128]);
int rlb_nccl_init(int device, int nranks, int rank, const uint8_t id[128], void** comm);
int rlb_nccl_broadcast(void* comm, void* buf, int64_t nbytes, int root, void* stream);
int rlb_nccl_destroy(void* comm);
/* Let `device` read `peer`'s memory directly (single-process multi-GPU pulls). */
int rlb_enable_peer(int device, int peer);

/* ---- CUDA IPC (pull sessions between processes) ------------------------ */
/* Handle of the allocation containing dev_ptr, plus dev_ptr's byte offset in it. */
int rlb_ipc_handle(const void* dev_ptr, uint8_t out_handle[64], int64_t* out_offset);
int rlb_ipc_open(int device, const uint8_t handle[64], void** dev_ptr);
int rlb_ipc_close(int device, void* dev_ptr);

/* ---- requests ---------------------------------------------------------- */
/* generate{request_id, prompt_tokens, prefix_tokens}: target_len is the total
 * generated length (prefix included), RolloutRequest.target_len. */
int rlb_submit(rlb_instance* h, uint64_t key, const int32_t* prompt, int32_t n_prompt,
               const int32_t* prefix, int32_t n_prefix, int32_t target_len);
/* Batched resume: sequence i is tokens[cu_lens[i]:cu_lens[i+1]] of which the
 * first n_prompt[i] are prompt and the rest generated prefix. */
int rlb_submit_varlen(rlb_instance* h, int32_t n, const uint64_t* keys, const int32_t* tokens,
                      const int64_t* cu_lens, const int32_t* n_prompt, const int32_t* target_len);
/* Admit + prefill pending requests, then run up to n_steps decode steps
 * (stopping early when nothing is executing). */
int rlb_step(rlb_instance* h, int32_t n_steps, rlb_token_batch* out);
/* Remove a request (pending or executing); returns its generated tokens. */
int rlb_cancel(rlb_instance* h, uint64_t key, int32_t* out_tokens, int32_t cap,
               int32_t* out_len);
/* K5 compaction: gather prompt+generated of each key (device-side gather into
 * one contiguous varlen buffer + exclusive-scan offsets), copy to host.
 * out_cu_lens has n+1 entries; out_n_prompt n entries. */
int rlb_export_partials(rlb_instance* h, int32_t n, const uint64_t* keys, int32_t* out_tokens,
                        int64_t cap, int64_t* out_cu_lens, int32_t* out_n_prompt);
int rlb_status(rlb_instance* h, int32_t* m_pending, int32_t* m_exec, uint64_t* weight_version);
/* Cumulative device-side accounting of an instance (CUDA events on its stream). */
typedef struct {
  double prefill_ms;       /* device time of admission + varlen prefill */
  double decode_ms;        /* device time of decode steps */
  int64_t prefill_rows;
  int64_t decode_steps;
  int64_t decode_rows;     /* sum over decode steps of executing sequences */
  int64_t kernel_launches; /* librlb kernels launched (graph nodes counted) */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
} rlb_stats;
int rlb_get_stats(rlb_instance* h, rlb_stats* out, int32_t reset);
/* Measured decode profile (replaces the modelled
 * instance_throughput + profile_acc capture of _refresh_rate,
 * pkg/src/spotrl/sim/engine.py:786-802, and _finalize_profile, :928-939):
 * per batch size b (rows of a decode step), the decode steps run, their
 * device seconds (CUDA events around every constant-batch burst) and the mean
 * context length.  decode throughput = b * steps / seconds tokens/s.  Arrays
 * of `cap` entries (NULL arrays: count only); ascending batch size. */
int rlb_decode_profile(rlb_instance* h, int32_t cap, int32_t* batch, int64_t* steps,
                       double* seconds, double* ctx_mean, int32_t* n_out, int32_t reset);
/* Re-launch one kernel of the last decode step `iters` times on the instance
 * stream (rows, KV and weights as that step left them) and time it with CUDA
 * events.  which: 0 attention (layer 0), 1 gate_up GEMM, 2 down GEMM (+ fused
 * residual add), 3 QKV GEMM (+ fused RoPE / KV append), 4 O GEMM (+ residual
 * add), 5 lm_head GEMM (+ argmax partials), 6 RMSNorm row kernel.  Timing
 * only: it overwrites scratch and the last layer's KV entries of the current
 * positions, so the rollout being profiled must be discarded.  Returns the
 * average launch time and the algorithmic bytes (attention, norm) or FLOPs
 * (GEMMs) of one launch. */
int rlb_profile_kernel(rlb_instance* h, int32_t which, int32_t iters, double* avg_ms,
                       double* work_per_launch);
/* Teacher-forced scoring: fp32 logits of every row of `tokens` (one sequence,
 * scratch slot), written to host out_logits[n][vocab]. */
int rlb_score(rlb_instance* h, const int32_t* tokens, int32_t n, float* out_logits);

/* ---- kernel-level entry points (parity tests) -------------------------- */
/* C = A[M,K] . B[N,K]^T with epilogue: 0 bf16 out (+bias if bias!=NULL),
 * 1 fp32 residual add (C fp32 in/out), 2 SwiGLU over 64-row interleaved
 * gate/up blocks (bf16 out [M, N/2]), 3 fp32 out.  block_n 128 or 256;
 * block_m 256 (two 128-row accumulators per CTA) or 128 (one).  splits > 1
 * runs split-K: epilogue 1 with block_n 128 reduces the splits inside a
 * thread-block cluster (the engine's path); epilogues 0 and 3 write fp32
 * partials and reduce them in order in a second kernel.  All device
 * pointers. */
int rlb_gemm(int device, int32_t M, int32_t N, int32_t K, const void* A, const void* B,
             const void* bias, void* C, int32_t epilogue, int32_t block_n, int32_t splits,
             int32_t block_m);
/* Average time of `iters` back-to-back launches of one GEMM configuration on
 * scratch buffers (tile / split-K tuning; epilogue 4 = argmax partials). */
int rlb_bench_gemm(int device, int32_t M, int32_t N, int32_t K, int32_t epilogue, int32_t block_n,
                   int32_t splits, int32_t block_m, int32_t iters, double* avg_ms);

#ifdef __cplusplus
}
#endif
#endif /* RLB_H_ */
