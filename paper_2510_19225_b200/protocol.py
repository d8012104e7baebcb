"""B200 additions to the reference wire protocol.

The messages, validators, builders and pull-session framing are the
reference's own (`pkg/src/spotrl/protocol.py:1-157`), imported unmodified and
re-exported here for the live-mode modules.  This module adds:

  * `cuda_ipc_endpoint` / `parse_cuda_ipc_endpoint`: the `agent_endpoint` of
    `pull_weights` for a same-node agent names a CUDA-IPC manifest (one
    handle + byte offset per HF tensor, in `hf_manifest` order) so a rollout
    process can map the trainer GPU's buffers and pull them over NVLink with
    the fused re-layout copy;
  * `InstanceAdapter`: serves the manager->instance messages with a
    `RolloutInstance` and turns its output into instance->manager messages.
"""
from __future__ import annotations

import base64
import json

from spotrl.protocol import (DONE_KIND, INSTANCE_TO_MANAGER, MANAGER_TO_INSTANCE,  # noqa: F401
                             MESSAGE_FIELDS, SHARD_KIND, ProtocolError, decode_line,
                             encode_message, iter_messages, msg_cancel, msg_generate,
                             msg_pull_weights, read_frames, read_pull_request, receive_weights,
                             validate_message, write_done, write_pull_request, write_shard)


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
