"""Pull-based weight transfer over NVLink (K7) -- trainer side, receiver side
and the 1->N fan-out.

Reference: an instance pulls the full weights from its paired agent as an
isolated byte-stream session (`pkg/src/spotrl/transfer.py:87-170`,
`pkg/src/spotrl/protocol.py:92-157`, SPEC.md "pull"), and a 1->N broadcast is
future work (`PAPER.md:548`).  B200 data plane:

  * `TrainerWeights` keeps the trainer's HF-layout bf16 tensors in one device
    allocation and publishes it as a `cuda-ipc://` endpoint (one IPC handle +
    per-tensor offsets) -- the `agent_endpoint` of `pull_weights`;
  * `MappedSource` maps that endpoint in a rollout process; the fused
    re-layout copy kernel then reads the trainer GPU's memory over NVLink;
  * `fanout_pull` serves N receivers of one trainer without dividing its
    egress N ways: the arena is cut into N x R slices; in round k receiver j
    pulls slice (k, j) from the trainer (scatter, re-layout fused) while
    copying the round k-1 slices of its peers from their engine arenas
    (all-gather, plain copy), so every receiver's ingress stays busy and the
    trainer sends each byte once.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check
from .protocol import cuda_ipc_endpoint, parse_cuda_ipc_endpoint
from .shapes import ModelShape, hf_manifest, relayout_segments


def _ipc_handle(ptr: int) -> tuple[bytes, int]:
    buf = (ctypes.c_uint8 * 64)()
    off = ctypes.c_int64()
    check(_lib.lib().rlb_ipc_handle(ptr, buf, ctypes.byref(off)))
    return bytes(buf), off.value


def blob_layout(shape: ModelShape) -> tuple[list[int], int]:
    """Byte offset of every HF tensor in the trainer's contiguous weight blob
    (256-byte aligned, `hf_manifest` order) and the blob size."""
    offs, total = [], 0
    for _, s in hf_manifest(shape):
        offs.append(total)
        n = 2
        for d in s:
            n *= d
        total += (n + 255) // 256 * 256
    return offs, total


def relayout_by_source(shape: ModelShape, lo: int, hi: int) -> list[tuple[int, int, int]]:
    """(blob_offset, arena_offset, nbytes) re-layout copies whose source bytes
    lie in blob range [lo, hi): the piece of the fused re-layout that can run
    once that range of the blob has arrived."""
    offs, _ = blob_layout(shape)
    out = []
    for hf, so, do, nb in relayout_segments(shape):
        a, b = offs[hf] + so, offs[hf] + so + nb
        x, y = max(a, lo), min(b, hi)
        if x < y:
            out.append((x, do + (x - a), y - x))
    return out


def copy_segments(device: int, segs: list[tuple[int, int, int]], src_base: int, dst_base: int,
                  stream) -> None:
    n = len(segs)
    if n == 0:
        return
    src = (ctypes.c_void_p * n)(*[src_base + s for s, _, _ in segs])
    dst = (ctypes.c_void_p * n)(*[dst_base + d for _, d, _ in segs])
    nb = (ctypes.c_int64 * n)(*[b for _, _, b in segs])
    check(_lib.lib().rlb_copy_segments(device, n, src, dst, nb, stream))


class NcclFanout:
    """1->N pull when several instances pull the same version at once
    (north_star: "NCCL broadcast when several instances pull at once").

    The trainer stages the version once in engine layout (the fused re-layout
    runs at staging time, the reference's agent staging step,
    `pkg/src/spotrl/transfer.py:64-85`), then one NCCL broadcast (ring / NVLS
    over NVSwitch) writes it straight into every receiver's engine arena: no
    receiver-side copy, each receiver's NVLink ingress is the only bound."""

    def __init__(self, device: int, nranks: int, rank: int, exchange_id):
        self.device = device
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            check(_lib.lib().rlb_nccl_unique_id(uid))
        uid_bytes = exchange_id(bytes(uid))
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(uid_bytes)
        comm = ctypes.c_void_p()
        check(_lib.lib().rlb_nccl_init(device, nranks, rank, uid, ctypes.byref(comm)))
        self.comm = comm
        self.staged: torch.Tensor | None = None

    def stage(self, trainer: "TrainerWeights") -> float:
        """Trainer side: re-layout the HF weights into an engine-layout buffer."""
        import time
        cfg = _lib.ModelCfg.from_shape(trainer.shape)
        nbytes = _lib.lib().rlb_arena_bytes(ctypes.byref(cfg))
        if self.staged is None or self.staged.numel() != nbytes:
            self.staged = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        ptrs = trainer.ptrs
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        torch.cuda.synchronize(self.device)
        t0 = time.perf_counter()
        check(_lib.lib().rlb_relayout_copy(self.device, ctypes.byref(cfg), arr, len(ptrs),
                                           self.staged.data_ptr(), None))
        torch.cuda.synchronize(self.device)
        return time.perf_counter() - t0

    def broadcast(self, instance=None, version: int = 0, root: int = 0) -> None:
        """Root: send the staged buffer; receivers: land it in `instance`'s arena."""
        if instance is None:
            ptr, nbytes = self.staged.data_ptr(), self.staged.numel()
        else:
            ptr, nbytes = instance.arena()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(_lib.lib().rlb_nccl_broadcast(self.comm, ptr, nbytes, root, stream))
        torch.cuda.current_stream(self.device).synchronize()
        if instance is not None:
            instance.mark_weights(version)

    def close(self) -> None:
        if self.comm:
            _lib.lib().rlb_nccl_destroy(self.comm)
            self.comm = None


class TrainerWeights:
    """HF-layout bf16 weights of one trainer GPU, contiguous, IPC-exportable."""

    def __init__(self, shape: ModelShape, device: int, tensors: dict[str, torch.Tensor]):
        self.shape = shape
        self.device = device
        manifest = hf_manifest(shape)
        offs, total = blob_layout(shape)
        self.blob = torch.empty(total, dtype=torch.uint8, device=f"cuda:{device}")
        self.views: dict[str, torch.Tensor] = {}
        self.nbytes: list[int] = []
        for (name, s), off in zip(manifest, offs):
            t = tensors[name]
            n = t.numel() * 2
            view = self.blob[off:off + n].view(torch.bfloat16).view(s)
            view.copy_(t)
            self.views[name] = view
            self.nbytes.append(n)
        self.offsets = offs
        torch.cuda.synchronize(device)

    @property
    def ptrs(self) -> list[int]:
        base = self.blob.data_ptr()
        return [base + o for o in self.offsets]

    def endpoint(self) -> str:
        handle, base_off = _ipc_handle(self.blob.data_ptr())
        return cuda_ipc_endpoint(self.device, [(handle, base_off + o) for o in self.offsets],
                                 self.nbytes)


class MappedSource:
    """A trainer's weights mapped into this process (peer memory via CUDA IPC)."""

    def __init__(self, endpoint: str, device: int):
        self.device = device
        _, tensors = parse_cuda_ipc_endpoint(endpoint)
        self._bases: dict[bytes, int] = {}
        ptrs = []
        for handle, off, _ in tensors:
            base = self._bases.get(handle)
            if base is None:
                p = ctypes.c_void_p()
                hb = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
                check(_lib.lib().rlb_ipc_open(device, hb, ctypes.byref(p)))
                base = self._bases[handle] = int(p.value)
            ptrs.append(base + off)
        self.ptrs = ptrs

    def close(self) -> None:
        for base in self._bases.values():
            _lib.lib().rlb_ipc_close(self.device, base)
        self._bases.clear()


def map_arena(endpoint_handle: tuple[bytes, int], device: int) -> tuple[int, object]:
    """Map a peer instance's engine arena: returns (device pointer, closer)."""
    handle, off = endpoint_handle
    p = ctypes.c_void_p()
    hb = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    check(_lib.lib().rlb_ipc_open(device, hb, ctypes.byref(p)))
    base = int(p.value)
    return base + off, lambda: _lib.lib().rlb_ipc_close(device, base)


def arena_handle(instance) -> tuple[bytes, int]:
    ptr, _ = instance.arena()
    return _ipc_handle(ptr)


@dataclass
class FanoutPlan:
    n_receivers: int
    rounds: int
    arena_bytes: int

    def slice(self, k: int, j: int) -> tuple[int, int]:
        """Arena byte range of round k, receiver j (16-byte aligned)."""
        n = self.n_receivers * self.rounds
        idx = k * self.n_receivers + j
        lo = (self.arena_bytes * idx // n) // 16 * 16
        hi = self.arena_bytes if idx == n - 1 else (self.arena_bytes * (idx + 1) // n) // 16 * 16
        return lo, hi


class FanoutReceiver:
    """One receiver of the scatter + all-gather fan-out (`me` of n receivers).

    Ordering between GPUs uses CUDA IPC events, not host round trips: the
    receiver enqueues its R scatter slices on stream s1, recording event k
    after slice k; after one host barrier (every receiver has enqueued its
    records) it enqueues, on stream s2, for each round k and peer j a wait on
    j's event k followed by the plain copy of slice (k, j) from j's arena.
    The GPUs then run scatter k+1 and gather k concurrently with no further
    host involvement."""

    def __init__(self, instance, me: int, n: int, rounds: int, exchange, barrier):
        self.inst = instance
        self.me, self.n = me, n
        self.rounds = rounds if n > 1 else 1
        self.barrier = barrier
        dev = instance.device
        self.s1 = torch.cuda.Stream(device=dev)
        self.s2 = torch.cuda.Stream(device=dev)
        self.events = [torch.cuda.Event(enable_timing=False, interprocess=True)
                       for _ in range(self.rounds)]
        for ev in self.events:          # materialise the events before exporting
            ev.record(self.s1)
        torch.cuda.synchronize(dev)
        mine = {"arena": arena_handle(instance), "events": [ev.ipc_handle() for ev in self.events]}
        every = exchange(mine)           # list over receivers
        self.peer_arenas: list[int | None] = []
        self.peer_events: list[list | None] = []
        self._closers = []
        for j, info in enumerate(every):
            if j == me:
                self.peer_arenas.append(None)
                self.peer_events.append(None)
                continue
            ptr, close = map_arena(info["arena"], dev)
            self.peer_arenas.append(ptr)
            self._closers.append(close)
            self.peer_events.append([torch.cuda.Event.from_ipc_handle(dev, h) for h in info["events"]])
        _, nbytes = instance.arena()
        self.plan = FanoutPlan(n, self.rounds, nbytes)
        self.cfg = _lib.ModelCfg.from_shape(instance.shape)

    def pull(self, source_ptrs: list[int], version: int) -> float:
        """Returns seconds from the start barrier to this receiver's last byte."""
        import time
        lib = _lib.lib()
        dev = self.inst.device
        arena, _ = self.inst.arena()
        arr = (ctypes.c_void_p * len(source_ptrs))(*source_ptrs)
        self.barrier()
        t0 = time.perf_counter()
        for k in range(self.rounds):
            lo, hi = self.plan.slice(k, self.me)
            check(lib.rlb_relayout_copy_range(dev, ctypes.byref(self.cfg), arr, len(source_ptrs),
                                              arena, lo, hi, self.s1.cuda_stream))
            self.events[k].record(self.s1)
        self.barrier()                   # every receiver's records are enqueued
        for k in range(self.rounds):
            for j in range(self.n):
                if j == self.me:
                    continue
                self.s2.wait_event(self.peer_events[j][k])
                lo, hi = self.plan.slice(k, j)
                check(lib.rlb_copy_bytes(dev, arena + lo, self.peer_arenas[j] + lo, hi - lo,
                                         self.s2.cuda_stream))
        self.s1.synchronize()
        self.s2.synchronize()
        dt = time.perf_counter() - t0
        self.barrier()                   # peers finished reading my arena
        self.inst.mark_weights(version)
        return dt

    def close(self) -> None:
        for c in self._closers:
            c()
        self._closers.clear()
