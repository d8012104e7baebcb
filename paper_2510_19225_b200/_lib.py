"""ctypes binding of librlb.so (include/rlb.h).

The product path has no CPU fallback: if the library is missing or fails to
load, importing a module that needs it raises immediately.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

# RLB_LIB selects another build of the same ABI (A/B bit-identity checks of a
# kernel change against the previous build); the default is the in-tree build.
LIB_PATH = os.environ.get("RLB_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "librlb.so")

RLB_OK, RLB_ERR_ARG, RLB_ERR_CUDA, RLB_ERR_STATE, RLB_ERR_CAPACITY = 0, -1, -2, -3, -4


class RlbError(RuntimeError):
    """A librlb call failed (CUDA error or internal fault)."""


class RlbStateError(RlbError):
    """Unknown / duplicate request key or call in the wrong state."""


class RlbCapacityError(RlbError):
    """Out of slots, KV pages or output capacity."""


class ModelCfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("vocab", "hidden", "layers", "n_q_heads", "n_kv_heads", "head_dim", "ffn", "tied")] + \
               [("rope_theta", ctypes.c_float), ("rms_eps", ctypes.c_float)]

    @classmethod
    def from_shape(cls, s) -> "ModelCfg":
        return cls(s.vocab, s.hidden, s.layers, s.n_q_heads, s.n_kv_heads, s.head_dim, s.ffn,
                   int(s.tied), s.rope_theta, s.rms_eps)


class EngineCfg(ctypes.Structure):
    _fields_ = [("max_slots", ctypes.c_int32), ("max_seq_len", ctypes.c_int32),
                ("num_pages", ctypes.c_int32), ("max_prefill_rows", ctypes.c_int32),
                ("graph_steps", ctypes.c_int32), ("split_o", ctypes.c_int32),
                ("split_down", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class TokenBatch(ctypes.Structure):
    _fields_ = [("cap_entries", ctypes.c_int32), ("cap_tokens", ctypes.c_int64),
                ("keys", ctypes.POINTER(ctypes.c_uint64)), ("counts", ctypes.POINTER(ctypes.c_int32)),
                ("done", ctypes.POINTER(ctypes.c_int32)), ("tokens", ctypes.POINTER(ctypes.c_int32)),
                ("n_entries", ctypes.c_int32), ("n_tokens", ctypes.c_int64),
                ("steps_run", ctypes.c_int32), ("prefill_rows", ctypes.c_int32)]


class PullStats(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_int64), ("seconds", ctypes.c_double)]


class Stats(ctypes.Structure):
    _fields_ = [("prefill_ms", ctypes.c_double), ("decode_ms", ctypes.c_double),
                ("prefill_rows", ctypes.c_int64), ("decode_steps", ctypes.c_int64),
                ("decode_rows", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_P = ctypes.c_void_p
_SIGS = {
    "rlb_get_stats": (ctypes.c_int, [_P, ctypes.POINTER(Stats), ctypes.c_int32]),
    "rlb_profile_kernel": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double)]),
    "rlb_instance_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ModelCfg),
                                           ctypes.POINTER(EngineCfg), ctypes.POINTER(_P)]),
    "rlb_instance_destroy": (ctypes.c_int, [_P]),
    "rlb_numerics_plan": (ctypes.c_int32, [_P, _P, ctypes.c_int32]),
    "rlb_kv_pool": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_int64)]),
    "rlb_last_error": (ctypes.c_char_p, []),
    "rlb_arena_bytes": (ctypes.c_int64, [ctypes.POINTER(ModelCfg)]),
    "rlb_hf_tensor_count": (ctypes.c_int32, [ctypes.POINTER(ModelCfg)]),
    "rlb_relayout_table": (ctypes.c_int64, [ctypes.POINTER(ModelCfg), _P, ctypes.c_int64]),
    "rlb_load_weights": (ctypes.c_int, [_P, _P, ctypes.c_int32, ctypes.c_uint64, _P,
                                        ctypes.POINTER(PullStats)]),
    "rlb_weights_arena": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_int64)]),
    "rlb_mark_weights": (ctypes.c_int, [_P, ctypes.c_uint64]),
    "rlb_relayout_copy": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ModelCfg), _P,
                                         ctypes.c_int32, _P, _P]),
    "rlb_copy_bytes": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_int64, _P]),
    "rlb_copy_segments": (ctypes.c_int, [ctypes.c_int, ctypes.c_int32, _P, _P, _P, _P]),
    "rlb_relayout_copy_range": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ModelCfg), _P,
                                               ctypes.c_int32, _P, ctypes.c_int64, ctypes.c_int64, _P]),
    "rlb_enable_peer": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "rlb_nccl_unique_id": (ctypes.c_int, [_P]),
    "rlb_nccl_init": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P,
                                     ctypes.POINTER(_P)]),
    "rlb_nccl_broadcast": (ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_int, _P]),
    "rlb_nccl_destroy": (ctypes.c_int, [_P]),
    "rlb_ipc_handle": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_int64)]),
    "rlb_ipc_open": (ctypes.c_int, [ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "rlb_ipc_close": (ctypes.c_int, [ctypes.c_int, _P]),
    "rlb_submit": (ctypes.c_int, [_P, ctypes.c_uint64, _P, ctypes.c_int32, _P, ctypes.c_int32,
                                  ctypes.c_int32]),
    "rlb_submit_varlen": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, _P, _P, _P]),
    "rlb_step": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.POINTER(TokenBatch)]),
    "rlb_cancel": (ctypes.c_int, [_P, ctypes.c_uint64, _P, ctypes.c_int32,
                                  ctypes.POINTER(ctypes.c_int32)]),
    "rlb_export_partials": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, ctypes.c_int64, _P, _P]),
    "rlb_status": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                  ctypes.POINTER(ctypes.c_uint64)]),
    "rlb_score": (ctypes.c_int, [_P, _P, ctypes.c_int32, _P]),
    "rlb_shadow_arena": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_void_p),
                                        ctypes.POINTER(ctypes.c_int64)]),
    "rlb_load_shadow": (ctypes.c_int, [_P, _P, ctypes.c_int32, ctypes.c_uint64, _P]),
    "rlb_mark_shadow": (ctypes.c_int, [_P, ctypes.c_uint64, _P]),
    "rlb_shadow_status": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(ctypes.c_double)]),
    "rlb_swap_weights": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64)]),
    "rlb_decode_profile": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, _P, _P,
                                          ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]),
    "rlb_bench_gemm": (ctypes.c_int, [ctypes.c_int] + [ctypes.c_int32] * 8 +
                       [ctypes.POINTER(ctypes.c_double)]),
    "rlb_gemm": (ctypes.c_int, [ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P,
                                _P, _P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int32]),
}
EXPORTED = tuple(_SIGS)

_lib: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    """Load librlb.so once; raises OSError (loudly) when it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is not built (run `make` or __graft_entry__.build())")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == RLB_OK:
        return
    msg = lib().rlb_last_error().decode(errors="replace")
    if rc == RLB_ERR_ARG:
        raise ValueError(msg)
    if rc == RLB_ERR_STATE:
        raise RlbStateError(msg)
    if rc == RLB_ERR_CAPACITY:
        raise RlbCapacityError(msg)
    raise RlbError(f"librlb error {rc}: {msg}")


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data
