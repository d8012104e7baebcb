"""Rollout-instance wire protocol and pull-session framing.

Same messages, fields, framing and errors as the reference
(`pkg/src/spotrl/protocol.py:1-157`): JSON lines with a `type`
(instance->manager register/status/token/complete; manager->instance
generate/cancel/pull_weights) and pull sessions of `>cI`-framed `W` shards
closed by a `D` frame carrying {"type":"done","version","bytes"}.

For the B200 path the `agent_endpoint` of `pull_weights` names where the
trainer's weights live.  `cuda_ipc_endpoint()` encodes a CUDA-IPC manifest
(one handle + byte offset per HF tensor, in `hf_manifest` order) so a rollout
process can map the trainer GPU's buffers and pull them over NVLink with the
fused re-layout copy; `InstanceAdapter` maps the messages onto a
`RolloutInstance`.
"""
from __future__ import annotations

import base64
import json
import struct
from typing import IO, Iterator


class ProtocolError(ValueError):
    pass


INSTANCE_TO_MANAGER = {
    "register": ("instance_id", "gpu_count"),
    "status": ("m_pending", "m_exec", "weight_version"),
    "token": ("request_id", "token_id"),
    "complete": ("request_id",),
}
MANAGER_TO_INSTANCE = {
    "generate": ("request_id", "prompt_tokens", "prefix_tokens"),
    "cancel": ("request_id",),
    "pull_weights": ("version", "agent_endpoint"),
}
MESSAGE_FIELDS = {**INSTANCE_TO_MANAGER, **MANAGER_TO_INSTANCE}


def validate_message(message: dict) -> None:
    kind = message.get("type")
    fields = MESSAGE_FIELDS.get(kind)
    if fields is None:
        raise ProtocolError(f"unknown message type: {kind!r}")
    missing = [f for f in fields if f not in message]
    if missing:
        raise ProtocolError(f"{kind}: missing fields {missing}")


def encode_message(message: dict) -> bytes:
    validate_message(message)
    return json.dumps(message, sort_keys=True, separators=(",", ":")).encode() + b"\n"


def decode_line(line: bytes | str) -> dict:
    text = line.decode() if isinstance(line, (bytes, bytearray)) else line
    try:
        message = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ProtocolError(f"malformed message: {exc}") from exc
    if not isinstance(message, dict):
        raise ProtocolError(f"expected JSON object, got {type(message).__name__}")
    validate_message(message)
    return message


def iter_messages(stream: IO[bytes]) -> Iterator[dict]:
    for line in stream:
        if line.strip():
            yield decode_line(line)


def msg_generate(request_id: str, prompt_tokens: list[int], prefix_tokens: list[int]) -> dict:
    return {"type": "generate", "request_id": request_id, "prompt_tokens": prompt_tokens,
            "prefix_tokens": prefix_tokens}


def msg_cancel(request_id: str) -> dict:
    return {"type": "cancel", "request_id": request_id}


def msg_pull_weights(version: int, agent_endpoint: str) -> dict:
    return {"type": "pull_weights", "version": version, "agent_endpoint": agent_endpoint}


# -- pull-session framing -----------------------------------------------------

_HEADER = struct.Struct(">cI")
SHARD_KIND = b"W"
DONE_KIND = b"D"


def write_pull_request(stream: IO[bytes], version: int) -> None:
    stream.write(json.dumps({"type": "pull", "version": version}).encode() + b"\n")


def read_pull_request(stream: IO[bytes]) -> int:
    message = json.loads(stream.readline())
    if message.get("type") != "pull" or "version" not in message:
        raise ProtocolError(f"bad pull request: {message!r}")
    return message["version"]


def write_shard(stream: IO[bytes], payload: bytes) -> None:
    stream.write(_HEADER.pack(SHARD_KIND, len(payload)))
    stream.write(payload)


def write_done(stream: IO[bytes], version: int, total_bytes: int) -> None:
    body = json.dumps({"type": "done", "version": version, "bytes": total_bytes},
                      sort_keys=True).encode()
    stream.write(_HEADER.pack(DONE_KIND, len(body)))
    stream.write(body)


def read_frames(stream: IO[bytes]) -> Iterator[tuple[bytes, bytes]]:
    """(kind, payload) frames up to and including the done frame, or EOF."""
    while True:
        head = stream.read(_HEADER.size)
        if not head:
            return
        if len(head) < _HEADER.size:
            raise ProtocolError("truncated frame header")
        kind, length = _HEADER.unpack(head)
        payload = stream.read(length)
        if len(payload) < length:
            raise ProtocolError("truncated frame payload")
        yield kind, payload
        if kind == DONE_KIND:
            return
        if kind != SHARD_KIND:
            raise ProtocolError(f"unknown frame kind: {kind!r}")


def receive_weights(stream: IO[bytes]) -> tuple[int, bytes]:
    """A full pull session -> (version, concatenated weight bytes)."""
    parts: list[bytes] = []
    done = None
    for kind, payload in read_frames(stream):
        if kind == SHARD_KIND:
            parts.append(payload)
        else:
            done = json.loads(payload)
    if done is None:
        raise ProtocolError("stream ended before done frame")
    blob = b"".join(parts)
    if done["bytes"] != len(blob):
        raise ProtocolError(f"byte count mismatch: {done['bytes']} != {len(blob)}")
    return done["version"], blob


# -- CUDA-IPC agent endpoints (B200 data plane) -----------------------------

IPC_SCHEME = "cuda-ipc://"


def cuda_ipc_endpoint(device: int, handles: list[tuple[bytes, int]], nbytes: list[int]) -> str:
    """Encode the trainer's weight manifest: per HF tensor (ipc handle, offset)."""
    body = {"device": device,
            "tensors": [[base64.b64encode(h).decode(), off, nb]
                        for (h, off), nb in zip(handles, nbytes)]}
    return IPC_SCHEME + base64.urlsafe_b64encode(json.dumps(body).encode()).decode()


def parse_cuda_ipc_endpoint(endpoint: str) -> tuple[int, list[tuple[bytes, int, int]]]:
    if not endpoint.startswith(IPC_SCHEME):
        raise ProtocolError(f"not a CUDA-IPC endpoint: {endpoint[:32]!r}")
    try:
        body = json.loads(base64.urlsafe_b64decode(endpoint[len(IPC_SCHEME):]))
        return body["device"], [(base64.b64decode(h), off, nb) for h, off, nb in body["tensors"]]
    except (ValueError, KeyError) as exc:
        raise ProtocolError(f"bad CUDA-IPC endpoint: {exc}") from exc


class InstanceAdapter:
    """Serves the manager->instance messages with a RolloutInstance and turns
    its output into instance->manager messages (live mode).
    `generate` needs the request's target length; the manager side sends it
    as an extra field (`target_len`), which the protocol permits (senders may
    add fields, reference `protocol.py:23-24`)."""

    def __init__(self, instance, instance_id: str, gpu_count: int = 1, open_endpoint=None):
        self.instance = instance
        self.instance_id = instance_id
        self.gpu_count = gpu_count
        self._open_endpoint = open_endpoint

    def register(self) -> dict:
        return {"type": "register", "instance_id": self.instance_id, "gpu_count": self.gpu_count}

    def handle(self, message: dict) -> list[dict]:
        validate_message(message)
        kind = message["type"]
        if kind == "generate":
            if "target_len" not in message:
                raise ProtocolError("generate: the B200 instance needs target_len")
            self.instance.generate(message["request_id"], message["prompt_tokens"],
                                   message["prefix_tokens"], target_len=message["target_len"])
            return []
        if kind == "cancel":
            self.instance.cancel(message["request_id"])
            return []
        if kind == "pull_weights":
            if self._open_endpoint is None:
                raise ProtocolError("no weight source resolver configured")
            src = self._open_endpoint(message["agent_endpoint"], message["version"])
            self.instance.pull_weights(src, message["version"])
            if hasattr(src, "close"):
                src.close()
            return [self.status()]
        raise ProtocolError(f"{kind} is not a manager->instance message")

    def status(self) -> dict:
        return {"type": "status", **self.instance.status()}

    def pump(self, n_steps: int = 16) -> list[dict]:
        out: list[dict] = []
        for rid, ids, done in self.instance.step(n_steps):
            out.extend({"type": "token", "request_id": rid, "token_id": int(t)} for t in ids)
            if done:
                out.append({"type": "complete", "request_id": rid})
        return out
