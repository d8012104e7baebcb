"""RolloutInstance: one B200 rollout instance behind the rlb_* C ABI.

This is the object the reference's rollout-instance surfaces plug into:

  reference                                           here
  -------------------------------------------------   ------------------------------
  protocol `generate{request_id, prompt_tokens,        generate(request_id, prompt_tokens,
    prefix_tokens}` (pkg/src/spotrl/protocol.py:75-81)   prefix_tokens, target_len)
  protocol `cancel{request_id}` (protocol.py:84-85)    cancel(request_id) -> generated ids
  protocol `status{m_pending, m_exec, weight_version}` status() -> same dict
    (protocol.py:26-31)
  protocol `pull_weights{version, agent_endpoint}`     pull_weights(version, source)
    (protocol.py:88-89)
  GenUnit decode advance _sync_unit                    step(n_steps) -> [(request_id,
    (pkg/src/spotrl/sim/engine.py:745-784)               new_token_ids, done)]
  migrate_out keeping `generated`                      export_partials(request_ids)
    (pkg/src/spotrl/manager.py:336-357)

Unlike the reference, token ids are real (greedy decode of a Qwen2-shape
decoder on the GPU) and the prefix in `generate` is honoured: the instance
rebuilds the KV cache of prompt + prefix with one varlen prefill and the
continuation is bit-identical to an uninterrupted run.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, i32, ptr
from .shapes import ModelShape, hf_manifest


@dataclass
class PullResult:
    version: int
    bytes: int
    seconds: float

    @property
    def gbps(self) -> float:
        return self.bytes / self.seconds / 1e9 if self.seconds > 0 else float("inf")


class RolloutInstance:
    def __init__(self, shape: ModelShape, device: int = 0, *, max_slots: int = 512,
                 max_seq_len: int = 1536, max_prefill_rows: int = 18944, graph_steps: int = 8,
                 num_pages: int = 0, split_o: int = 0, split_down: int = 0):
        """max_prefill_rows: token rows per prefill chunk; 18,944 = 74 x 256
        puts the same number of 256-row pair tiles on each of the 74 SM
        pairs in every prefill GEMM.  split_o / split_down: split-K factors of
        the O / down projections (0 = the measured default).  They are part of the numerics plan:
        instances exchanging requests must agree on it (`plan`)."""
        self.shape = shape
        self.device = device
        self.max_slots = max_slots
        self.max_seq_len = max_seq_len
        if os.environ.get("RLB_GRAPH_STEPS"):
            graph_steps = int(os.environ["RLB_GRAPH_STEPS"])
        self._cfg = _lib.ModelCfg.from_shape(shape)
        ecfg = _lib.EngineCfg(max_slots, max_seq_len, num_pages, max_prefill_rows, graph_steps,
                              split_o, split_down, 0)
        h = ctypes.c_void_p()
        check(_lib.lib().rlb_instance_create(device, ctypes.byref(self._cfg), ctypes.byref(ecfg),
                                             ctypes.byref(h)))
        self._h = h
        self._key_of: dict[str, int] = {}
        self._rid_of: dict[int, str] = {}
        self._next_key = 1
        cap = max_slots
        self._keys = np.zeros(cap, np.uint64)
        self._counts = np.zeros(cap, np.int32)
        self._done = np.zeros(cap, np.int32)
        self._tok_cap = max_slots * 520
        self._tokens = np.zeros(self._tok_cap, np.int32)
        self.last_steps = 0
        self.last_prefill_rows = 0
        self._events: list = []

    # -- lifecycle ---------------------------------------------------------

    def close(self) -> None:
        if self._h:
            _lib.lib().rlb_instance_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    # -- weights (pull) ----------------------------------------------------

    def _source_ptrs(self, src) -> list[int]:
        """HF tensor device pointers (`hf_manifest` order) of a weight source:
        a name -> tensor dict, an object with `.ptrs` (TrainerWeights,
        MappedSource, TcpPulledSource) or a pointer list."""
        if isinstance(src, dict):
            return [int(src[name].data_ptr()) for name, _ in hf_manifest(self.shape)]
        if hasattr(src, "ptrs"):
            return [int(p) for p in src.ptrs]
        return [int(p) for p in src]

    def _ready_event(self, src):
        """For a torch tensor dict: an event recorded on the producing stream
        (torch's current stream of the tensors' device), so the copy kernels
        wait on the device for whatever is still writing the weights (e.g. the
        trainer's optimizer step).  Other sources order themselves."""
        if not isinstance(src, dict):
            return None
        import torch
        t = next(iter(src.values()))
        if not t.is_cuda:
            return None
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(t.device))
        self._events.append(ev)            # kept alive until the copy is enqueued / done
        del self._events[:-2]
        return ev

    def load_weights(self, hf_weights, version: int) -> PullResult:
        """Pull an HF-layout weight set (dict name -> CUDA tensor, or a list of
        device pointers in `hf_manifest` order) with the fused re-layout.
        Only at a step boundary (no requests on the instance)."""
        ptrs = self._source_ptrs(hf_weights)
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        stats = _lib.PullStats()
        ev = self._ready_event(hf_weights)
        check(_lib.lib().rlb_load_weights(self._h, arr, len(ptrs), version,
                                          ev.cuda_event if ev is not None else None,
                                          ctypes.byref(stats)))
        return PullResult(version, stats.bytes, stats.seconds)

    pull_weights = load_weights

    def mark_weights(self, version: int) -> None:
        """The arena was filled externally (fan-out pull) with `version`."""
        check(_lib.lib().rlb_mark_weights(self._h, version))

    def kv_pool(self) -> tuple[int, int]:
        """(test hook) device pointer + bytes of the paged KV pool."""
        p, n = ctypes.c_void_p(), ctypes.c_int64()
        check(_lib.lib().rlb_kv_pool(self._h, ctypes.byref(p), ctypes.byref(n)))
        return int(p.value or 0), int(n.value)

    def arena(self) -> tuple[int, int]:
        p, n = ctypes.c_void_p(), ctypes.c_int64()
        check(_lib.lib().rlb_weights_arena(self._h, ctypes.byref(p), ctypes.byref(n)))
        return int(p.value or 0), int(n.value)

    # -- double-buffered weights -------------------------

    def shadow_arena(self) -> tuple[int, int]:
        """Device pointer + bytes of the second weight arena (allocated on
        first use): the target of a pull that must not disturb serving."""
        p, n = ctypes.c_void_p(), ctypes.c_int64()
        check(_lib.lib().rlb_shadow_arena(self._h, ctypes.byref(p), ctypes.byref(n)))
        return int(p.value or 0), int(n.value)

    def pull_shadow(self, hf_weights, version: int) -> None:
        """Start pulling `version` into the shadow arena (fused re-layout on the
        copy stream); returns at once while the active weights keep serving."""
        ptrs = self._source_ptrs(hf_weights)
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        ev = self._ready_event(hf_weights)
        check(_lib.lib().rlb_load_shadow(self._h, arr, len(ptrs), version,
                                         ev.cuda_event if ev is not None else None))

    @property
    def pull_bytes(self) -> int:
        """Bytes one pull moves (the HF tensors of the weight set)."""
        return sum(2 * int(np.prod(shape)) for _, shape in hf_manifest(self.shape))

    def mark_shadow(self, version: int, stream: int | None = None) -> None:
        """The shadow arena was filled externally by work on `stream`."""
        check(_lib.lib().rlb_mark_shadow(self._h, version, stream))

    SHADOW_STATES = ("empty", "pulling", "ready")

    def shadow_status(self) -> tuple[int, str, float]:
        """(version, 'empty'|'pulling'|'ready', device seconds of the copy)."""
        v, st, sec = ctypes.c_uint64(), ctypes.c_int32(), ctypes.c_double()
        check(_lib.lib().rlb_shadow_status(self._h, ctypes.byref(v), ctypes.byref(st),
                                           ctypes.byref(sec)))
        return int(v.value), self.SHADOW_STATES[st.value], float(sec.value)

    def swap_weights(self) -> int:
        """Step boundary: the shadow set becomes active (no host wait; the next
        decode kernels wait for its copy on the device).  Raises
        RlbStateError if requests are still on the instance."""
        v = ctypes.c_uint64()
        check(_lib.lib().rlb_swap_weights(self._h, ctypes.byref(v)))
        return int(v.value)

    # -- requests ----------------------------------------------------------

    def _key(self, request_id: str, create: bool) -> int:
        key = self._key_of.get(request_id)
        if key is None:
            if not create:
                raise KeyError(f"unknown request {request_id!r}")
            key = self._next_key
            self._next_key += 1
            self._key_of[request_id] = key
            self._rid_of[key] = request_id
        return key

    def _forget(self, request_id: str) -> None:
        key = self._key_of.pop(request_id, None)
        if key is not None:
            self._rid_of.pop(key, None)

    def generate(self, request_id: str, prompt_tokens, prefix_tokens=(), *, target_len: int) -> None:
        """protocol `generate`: serve prompt + prefix, stop at target_len generated ids."""
        if request_id in self._key_of:
            raise ValueError(f"duplicate request {request_id!r}")
        p, x = i32(prompt_tokens), i32(prefix_tokens)
        key = self._key(request_id, create=True)
        try:
            check(_lib.lib().rlb_submit(self._h, key, ptr(p), len(p), ptr(x) if len(x) else None,
                                        len(x), target_len))
        except Exception:
            self._forget(request_id)
            raise

    submit = generate

    def generate_varlen(self, request_ids, tokens, cu_lens, n_prompt, target_len) -> None:
        """Batched resume: sequence i = tokens[cu_lens[i]:cu_lens[i+1]], first n_prompt[i] prompt."""
        n = len(request_ids)
        keys = np.array([self._key(r, create=True) for r in request_ids], np.uint64)
        t, cu = i32(tokens), np.ascontiguousarray(np.asarray(cu_lens, np.int64))
        npr, tl = i32(n_prompt), i32(target_len)
        check(_lib.lib().rlb_submit_varlen(self._h, n, ptr(keys), ptr(t), ptr(cu), ptr(npr), ptr(tl)))

    def step(self, n_steps: int = 16) -> list[tuple[str, np.ndarray, bool]]:
        """Admit + prefill pending requests, decode up to n_steps; returns the
        new ids per request and whether it reached target_len (the request is
        then retired from the instance)."""
        b = _lib.TokenBatch(len(self._keys), self._tok_cap,
                            self._keys.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                            self._counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                            self._done.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                            self._tokens.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 0, 0, 0, 0)
        self._ensure_token_cap(n_steps)
        b.cap_tokens = self._tok_cap
        b.tokens = self._tokens.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        check(_lib.lib().rlb_step(self._h, n_steps, ctypes.byref(b)))
        self.last_steps, self.last_prefill_rows = b.steps_run, b.prefill_rows
        out = []
        off = 0
        for i in range(b.n_entries):
            key, cnt, done = int(self._keys[i]), int(self._counts[i]), bool(self._done[i])
            rid = self._rid_of[key]
            out.append((rid, self._tokens[off:off + cnt].copy(), done))
            off += cnt
            if done:
                self._forget(rid)
        return out

    def _ensure_token_cap(self, n_steps: int) -> None:
        need = self.max_slots * (n_steps + 2)
        if need > self._tok_cap:
            self._tok_cap = need
            self._tokens = np.zeros(need, np.int32)

    def cancel(self, request_id: str) -> list[int]:
        """protocol `cancel`: drop the request, return its generated ids."""
        key = self._key(request_id, create=False)
        buf = np.zeros(self.max_seq_len, np.int32)
        n = ctypes.c_int32()
        check(_lib.lib().rlb_cancel(self._h, key, ptr(buf), len(buf), ctypes.byref(n)))
        self._forget(request_id)
        return buf[:n.value].tolist()

    def export_partials(self, request_ids) -> list[tuple[list[int], list[int]]]:
        """K5 compaction: (prompt ids, generated ids) of each request, gathered
        on the device into one contiguous varlen buffer."""
        n = len(request_ids)
        if n == 0:
            return []
        keys = np.array([self._key(r, create=False) for r in request_ids], np.uint64)
        cap = n * self.max_seq_len
        toks = np.zeros(cap, np.int32)
        cu = np.zeros(n + 1, np.int64)
        npr = np.zeros(n, np.int32)
        check(_lib.lib().rlb_export_partials(self._h, n, ptr(keys), ptr(toks), cap, ptr(cu), ptr(npr)))
        out = []
        for i in range(n):
            seq = toks[cu[i]:cu[i + 1]]
            out.append((seq[:npr[i]].tolist(), seq[npr[i]:].tolist()))
        return out

    PLAN_FIELDS = ("format", "split_qkv", "split_o", "split_down", "attn_window", "attn_warps",
                   "page", "tie_rule")

    @property
    def plan(self) -> str:
        """The numerics plan (`rlb_numerics_plan`): what fixes the bits of a
        row's arithmetic.  A resume is bit-exact only between equal plans."""
        buf = (ctypes.c_int32 * 8)()
        n = _lib.lib().rlb_numerics_plan(self._h, buf, 8)
        return ".".join(f"{k}{buf[i]}"
                        for i, k in zip(range(n), ("v", "q", "o", "d", "w", "a", "p", "t")))

    def status(self) -> dict:
        """protocol `status` payload (+ the numerics plan, an extra field the
        protocol permits, `protocol.py:23-24`)."""
        mp, me, wv = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_uint64()
        check(_lib.lib().rlb_status(self._h, ctypes.byref(mp), ctypes.byref(me), ctypes.byref(wv)))
        return {"m_pending": mp.value, "m_exec": me.value, "weight_version": int(wv.value),
                "plan": self.plan}

    def score(self, tokens) -> np.ndarray:
        """Teacher-forced fp32 logits [len(tokens), vocab] of one sequence."""
        t = i32(tokens)
        out = np.zeros((len(t), self.shape.vocab), np.float32)
        check(_lib.lib().rlb_score(self._h, ptr(t), len(t), ptr(out)))
        return out

    KERNELS = {"attention": 0, "gate_up": 1, "down": 2, "qkv": 3, "o_proj": 4, "lm_head": 5,
               "resid_norm": 6}

    def stats(self, reset: bool = False) -> dict:
        """Cumulative device-time accounting (CUDA events on the instance stream)."""
        s = _lib.Stats()
        check(_lib.lib().rlb_get_stats(self._h, ctypes.byref(s), int(reset)))
        return s.as_dict()

    def decode_profile(self, reset: bool = False) -> list[tuple[int, int, float, float]]:
        """Measured decode profile: (batch size, decode steps, device seconds,
        mean context) per batch size seen so far (`rlb_decode_profile`)."""
        n = ctypes.c_int32()
        lib = _lib.lib()
        check(lib.rlb_decode_profile(self._h, 0, None, None, None, None, ctypes.byref(n), 0))
        k = max(n.value, 1)
        b, st = np.zeros(k, np.int32), np.zeros(k, np.int64)
        sec, ctx = np.zeros(k, np.float64), np.zeros(k, np.float64)
        check(lib.rlb_decode_profile(self._h, k, ptr(b), ptr(st), ptr(sec), ptr(ctx),
                                     ctypes.byref(n), int(reset)))
        return [(int(b[i]), int(st[i]), float(sec[i]), float(ctx[i])) for i in range(n.value)]

    def profile_kernel(self, name: str, iters: int = 20) -> tuple[float, float]:
        """(avg launch ms, algorithmic bytes or FLOPs per launch) of one kernel of
        the last decode step, re-launched `iters` times and timed with CUDA events."""
        ms, work = ctypes.c_double(), ctypes.c_double()
        check(_lib.lib().rlb_profile_kernel(self._h, self.KERNELS[name], iters, ctypes.byref(ms),
                                            ctypes.byref(work)))
        return ms.value, work.value

    # -- convenience -------------------------------------------------------

    def run_to_completion(self, n_steps: int = 64) -> dict[str, list[int]]:
        """Step until nothing is pending or executing; returns all ids generated."""
        got: dict[str, list[int]] = {}
        while True:
            st = self.status()
            if st["m_pending"] == 0 and st["m_exec"] == 0:
                return got
            for rid, toks, _ in self.step(n_steps):
                got.setdefault(rid, []).extend(toks.tolist())


def gemm(device: int, A, B, bias=None, out=None, epilogue: int = 0, block_n: int = 128,
         splits: int = 1, block_m: int = 256):
    """Kernel-level entry point rlb_gemm on torch CUDA tensors (parity tests)."""
    import torch
    M, K = A.shape
    N = B.shape[0]
    if out is None:
        if epilogue == 0:
            out = torch.empty(M, N, dtype=torch.bfloat16, device=A.device)
        elif epilogue == 2:
            out = torch.empty(M, N // 2, dtype=torch.bfloat16, device=A.device)
        else:
            out = torch.zeros(M, N, dtype=torch.float32, device=A.device)
    check(_lib.lib().rlb_gemm(device, M, N, K, A.data_ptr(), B.data_ptr(),
                              bias.data_ptr() if bias is not None else None, out.data_ptr(),
                              epilogue, block_n, splits, block_m))
    return out
