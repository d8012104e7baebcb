"""Live mode: the rollout manager and B200 instances in separate processes,
speaking the reference wire protocol.

Control plane (`pkg/src/spotrl/protocol.py:1-89`): each instance connects to
the manager over TCP and sends line-delimited JSON messages -- `register`,
`status`, `token`, `complete` -- and receives `generate`, `cancel` and
`pull_weights`.  Connection close without deregistration is a preemption
(`protocol.py:6`, `SPEC.md:350`): the manager keeps every token it received,
re-holds the displaced requests at the front, and they resume elsewhere with
`generate(prompt_tokens, prefix_tokens)`.

`ManagerServer` runs the manager's single serialized command stream
(`manager.py:1-8`): connection reader threads only enqueue decoded messages;
one loop applies them, dispatches (Alg. 2 JSQ) and admits.  `serve_instance`
is the instance process: it registers, executes messages with
`InstanceAdapter`, steps its RolloutInstance and streams tokens back.

Weight pulls name an `agent_endpoint`: `cuda-ipc://` (same node: the fused
re-layout reads the trainer GPU over NVLink, `pull.MappedSource`) or
`tcp://host:port` (another node: `AgentServer` streams the trainer's HF blob
as `W` shard frames + a `D` done frame, `protocol.py:92-157`; the receiver
lands each shard in a pinned buffer, copies it to the GPU and runs the same
fused re-layout, `tcp_pull`).
"""
from __future__ import annotations

import json
import queue
import socket
import threading
import time
from typing import Callable

from spotrl.domain import InstanceStatus

from .protocol import (DONE_KIND, SHARD_KIND, InstanceAdapter, ProtocolError, decode_line,
                       encode_message, msg_cancel, msg_generate, msg_pull_weights, read_frames,
                       read_pull_request, write_done, write_pull_request, write_shard)
from .responses import ResponseBuffer, dispatch

TCP_SCHEME = "tcp://"


class _Conn:
    """One TCP connection: a reader thread feeding decoded messages (or the
    close) into a shared queue, and a locked line writer."""

    def __init__(self, sock: socket.socket, cid: int, events: "queue.Queue"):
        self.sock = sock
        self.cid = cid
        self.rfile = sock.makefile("rb")
        self._wlock = threading.Lock()
        self.closed = False
        self.events = events

    def start(self) -> "_Conn":
        threading.Thread(target=self._read, daemon=True).start()
        return self

    def _read(self) -> None:
        try:
            for line in self.rfile:
                if line.strip():
                    self.events.put(("msg", self.cid, decode_line(line)))
        except (OSError, ValueError):
            pass
        self.events.put(("closed", self.cid, None))

    def send(self, *messages: dict) -> None:
        data = b"".join(encode_message(m) for m in messages)
        with self._wlock:
            self.sock.sendall(data)

    def close(self) -> None:
        if not self.closed:
            self.closed = True
            try:
                self.sock.shutdown(socket.SHUT_RDWR)
            except OSError:
                pass
            self.sock.close()


class ManagerServer:
    """The manager side of live mode around an unmodified reference
    `RolloutManager`.  `endpoint_for(instance_id)` names the agent endpoint
    each registering instance pulls `version` from; requests are created with
    `submit` (prompt ids go to the `ResponseBuffer`)."""

    def __init__(self, manager, version: int, endpoint_for: Callable[[str], str], *,
                 host: str = "127.0.0.1", port: int = 0, max_inflight: int | None = None,
                 responses: ResponseBuffer | None = None):
        self.manager = manager
        self.responses = responses if responses is not None else ResponseBuffer(manager)
        self.version = version
        self.endpoint_for = endpoint_for
        self.max_inflight = max_inflight
        self.events: queue.Queue = queue.Queue()
        self.conns: dict[int, _Conn] = {}
        self.iid_of: dict[int, str] = {}
        self.conn_of: dict[str, _Conn] = {}
        self._pull_t0: dict[str, float] = {}
        self.plan: str | None = None          # numerics plan shared by every instance
        self._t0 = time.perf_counter()
        self._lsock = socket.create_server((host, port))
        self.address = self._lsock.getsockname()
        self._stop = False
        threading.Thread(target=self._accept, daemon=True).start()

    def now(self) -> float:
        return time.perf_counter() - self._t0

    def submit(self, request_id: str, prompt_tokens: list[int], target_len: int,
               group_id: str = "g"):
        return self.responses.create_request(request_id, prompt_tokens, target_len, group_id,
                                             self.now())

    def _accept(self) -> None:
        cid = 0
        while not self._stop:
            try:
                sock, _ = self._lsock.accept()
            except OSError:
                return
            sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            cid += 1
            conn = self.conns[cid] = _Conn(sock, cid, self.events)
            conn.start()               # registered before its first message can arrive

    # -- the serialized command stream ------------------------------------------

    def _apply(self, kind: str, cid: int, msg: dict | None) -> None:
        m, now = self.manager, self.now()
        if kind == "closed":
            iid = self.iid_of.pop(cid, None)
            self.conns.pop(cid, None)
            if iid is not None and m.records[iid].status is not InstanceStatus.PREEMPTED:
                self.conn_of.pop(iid, None)
                displaced = m.on_preempt(iid, now)
                for rid in sorted(displaced, key=m.request_seq.__getitem__, reverse=True):
                    m.hold(rid, front=True)
            return
        t = msg["type"]
        if t == "register":
            iid = msg["instance_id"]
            res = m.register_instance(iid, msg["gpu_count"], now)
            conn = self.conns[cid]
            if res.value != "accepted":
                conn.close()
                return
            self.iid_of[cid] = iid
            self.conn_of[iid] = conn
            m.mark_pulling(iid, now)
            endpoint = self.endpoint_for(iid)
            m.log.emit(now, "pull_request", instance_id=iid, version=self.version, started=True)
            self._pull_t0[iid] = now
            conn.send(msg_pull_weights(self.version, endpoint))
        elif t == "status":
            iid = self.iid_of[cid]
            plan = msg.get("plan")
            if plan is not None:
                if self.plan is None:
                    self.plan = plan
                elif plan != self.plan:
                    # a resume across plans would not be bit-exact: refuse the
                    # instance (its close event is handled like a preemption)
                    m.log.emit(now, "plan_mismatch", instance_id=iid, plan=plan,
                               expected=self.plan)
                    self.conns[cid].close()
                    return
            rec = m.records[iid]
            if rec.status is InstanceStatus.PULLING_WEIGHTS and \
                    msg["weight_version"] >= self.version:
                m.mark_active(iid, msg["weight_version"], now)
                m.log.emit(now, "pull_done", instance_id=iid, version=msg["weight_version"],
                           seconds=now - self._pull_t0.pop(iid, now))
        elif t == "token":
            self.responses.on_tokens(msg["request_id"], self.iid_of[cid], [msg["token_id"]], now)
        elif t == "complete":
            m.complete(msg["request_id"], self.iid_of[cid], now)
        else:
            raise ProtocolError(f"{t} is not an instance->manager message")

    def _dispatch_and_admit(self) -> None:
        m, now = self.manager, self.now()
        dispatch(m, now)
        for iid, conn in list(self.conn_of.items()):
            out = []
            for rid in list(m.pending_queues.get(iid, ())):
                if self.max_inflight is not None and \
                        len(m.executing_sets[iid]) >= self.max_inflight:
                    break
                req = m.requests[rid]
                m.admit(rid, iid, now)
                msg = msg_generate(rid, self.responses.prompt(rid), list(req.generated))
                msg["target_len"] = req.target_len
                out.append(msg)
            if out:
                try:
                    conn.send(*out)
                except OSError:
                    pass          # the close event re-holds them

    def run_until_done(self, timeout: float = 600.0) -> None:
        """Apply events until every request of the step is complete."""
        t_end = time.monotonic() + timeout
        while not self.manager.all_generated():
            if time.monotonic() > t_end:
                raise TimeoutError("live rollout did not finish")
            try:
                ev = self.events.get(timeout=0.05)
            except queue.Empty:
                self._dispatch_and_admit()
                continue
            self._apply(*ev)
            while True:                       # drain what is already queued
                try:
                    self._apply(*self.events.get_nowait())
                except queue.Empty:
                    break
            self._dispatch_and_admit()

    def cancel(self, request_id: str) -> None:
        iid = self.manager.owner[request_id]
        self.conn_of[iid].send(msg_cancel(request_id))

    def close(self) -> None:
        self._stop = True
        self._lsock.close()
        for c in list(self.conns.values()):
            c.close()


def serve_instance(address, instance, instance_id: str, *, open_endpoint, gpu_count: int = 1,
                   n_steps: int = 16, stop: threading.Event | None = None,
                   die_after_tokens: int | None = None) -> None:
    """The instance process: register, pull, then serve until the manager
    closes the connection (or `stop` is set).  `die_after_tokens` drops the
    connection abruptly (a spot preemption) at the first flush that would
    take the streamed token count past it; that flush is lost."""
    sock = socket.create_connection(address)
    sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    inbox: queue.Queue = queue.Queue()
    conn = _Conn(sock, 0, inbox).start()
    adapter = InstanceAdapter(instance, instance_id, gpu_count, open_endpoint=open_endpoint)
    conn.send(adapter.register())
    sent = 0
    busy = False
    try:
        while stop is None or not stop.is_set():
            try:
                ev = inbox.get(timeout=0 if busy else 0.05)
            except queue.Empty:
                ev = None
            while ev is not None:
                kind, _, msg = ev
                if kind == "closed":
                    return
                replies = adapter.handle(msg)
                if replies:
                    conn.send(*replies)
                try:
                    ev = inbox.get_nowait()
                except queue.Empty:
                    ev = None
            st = instance.status()
            busy = st["m_pending"] + st["m_exec"] > 0
            if not busy:
                continue
            out = adapter.pump(n_steps)
            if die_after_tokens is not None:
                n_tok = sum(1 for o in out if o["type"] == "token")
                if sent + n_tok > die_after_tokens:
                    return                 # vanish mid-flight: this flush never arrives
                sent += n_tok
            if out:
                conn.send(*out)
    finally:
        conn.close()


# -- cross-node pull over W/D frames ------------------------------------------

class AgentServer:
    """A transfer agent outside the NVLink domain: serves pull sessions for
    staged versions as `W` shard frames + a `D` done frame (the trainer's HF
    blob, `pull.blob_layout` order)."""

    def __init__(self, host: str = "127.0.0.1", port: int = 0, shard_bytes: int = 64 << 20):
        self.staged: dict[int, memoryview] = {}
        self.shard_bytes = shard_bytes
        self._lsock = socket.create_server((host, port))
        self.address = self._lsock.getsockname()
        self.sessions = 0
        threading.Thread(target=self._accept, daemon=True).start()

    @property
    def endpoint(self) -> str:
        return f"{TCP_SCHEME}{self.address[0]}:{self.address[1]}"

    def stage(self, version: int, blob) -> None:
        """blob: bytes-like (e.g. a pinned host copy of TrainerWeights.blob)."""
        self.staged[version] = memoryview(blob).cast("B")

    def _accept(self) -> None:
        while True:
            try:
                sock, _ = self._lsock.accept()
            except OSError:
                return
            threading.Thread(target=self._session, args=(sock,), daemon=True).start()

    def _session(self, sock: socket.socket) -> None:
        with sock, sock.makefile("rwb") as f:
            version = read_pull_request(f)
            blob = self.staged.get(version)
            if blob is None:
                return                       # not staged: the puller sees EOF
            for lo in range(0, len(blob), self.shard_bytes):
                write_shard(f, blob[lo:lo + self.shard_bytes])
            write_done(f, version, len(blob))
            f.flush()
            self.sessions += 1

    def close(self) -> None:
        self._lsock.close()


class TcpPulledSource:
    """Weights pulled over TCP into this GPU: the HF blob lands shard by shard
    in a pinned host buffer and is copied to a device staging blob on a side
    stream as it arrives; `ptrs` are the HF tensor pointers the fused
    re-layout copy reads (`RolloutInstance.pull_weights(source)`)."""

    def __init__(self, endpoint: str, version: int, shape, device: int):
        import torch
        from .pull import blob_layout
        if not endpoint.startswith(TCP_SCHEME):
            raise ProtocolError(f"not a tcp endpoint: {endpoint!r}")
        host, port = endpoint[len(TCP_SCHEME):].rsplit(":", 1)
        offs, total = blob_layout(shape)
        self.host_blob = torch.empty(total, dtype=torch.uint8, pin_memory=True)
        self.dev_blob = torch.empty(total, dtype=torch.uint8, device=f"cuda:{device}")
        stream = torch.cuda.Stream(device=device)
        t0 = time.perf_counter()
        got = 0
        done = None
        with socket.create_connection((host, int(port))) as sock, sock.makefile("rwb") as f:
            write_pull_request(f, version)
            f.flush()
            hb = memoryview(self.host_blob.numpy()).cast("B")
            for kind, payload in read_frames(f):
                if kind == SHARD_KIND:
                    n = len(payload)
                    if got + n > total:
                        raise ProtocolError("more weight bytes than the model holds")
                    hb[got:got + n] = payload
                    with torch.cuda.stream(stream):
                        self.dev_blob[got:got + n].copy_(self.host_blob[got:got + n],
                                                         non_blocking=True)
                    got += n
                elif kind == DONE_KIND:
                    done = json.loads(payload)
        if done is None:
            raise ProtocolError("pull session ended before the done frame")
        if done["bytes"] != got or got != total or done["version"] != version:
            raise ProtocolError(f"pull session mismatch: {done} vs {got}/{total} bytes, "
                                f"version {version}")
        stream.synchronize()
        self.seconds = time.perf_counter() - t0
        self.bytes = got
        base = self.dev_blob.data_ptr()
        self.ptrs = [base + o for o in offs]


def open_endpoint_for(shape, device: int, version_of: Callable[[], int] | None = None):
    """`InstanceAdapter.open_endpoint` resolver for both endpoint schemes."""
    def resolve(endpoint: str, version: int):
        if endpoint.startswith(TCP_SCHEME):
            return TcpPulledSource(endpoint, version, shape, device)
        from .pull import MappedSource
        return MappedSource(endpoint, device)
    return resolve
