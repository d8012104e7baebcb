"""CPU stand-in for RolloutInstance used by host-logic tests (no GPU).

Deterministic greedy "decoder": the next id is a hash of the whole context,
so a resumed request continues exactly like an uninterrupted one -- the same
property the real instance guarantees with batch-invariant kernels.  It keeps
the RolloutInstance surface (generate / step / cancel / export_partials /
status / pull_weights / close) and its admission and flush semantics."""
from __future__ import annotations

import hashlib

import numpy as np


class FakePull:
    def __init__(self, version, nbytes, seconds):
        self.version, self.bytes, self.seconds = version, nbytes, seconds

    @property
    def gbps(self):
        return self.bytes / self.seconds / 1e9


class FakeInstance:
    def __init__(self, vocab: int = 1000, max_slots: int = 8, plan: str | None = None):
        self.vocab = vocab
        self.max_slots = max_slots
        self.plan = plan            # numerics plan (RolloutInstance.plan); None = not reported
        self.pending: list[str] = []
        self.active: dict[str, dict] = {}
        self.version = 0
        self.closed = False
        self.last_steps = 0

    def next_token(self, ctx: list[int]) -> int:
        h = hashlib.blake2b(np.asarray(ctx, np.int64).tobytes(), digest_size=8).digest()
        return int.from_bytes(h, "little") % self.vocab

    def pull_weights(self, source, version):
        self.version = version
        return FakePull(version, 1 << 20, 1e-3)

    load_weights = pull_weights

    # double-buffered weights (RolloutInstance.pull_shadow / swap_weights)
    shadow_version, shadow_state = 0, "empty"

    def pull_shadow(self, source, version):
        self.shadow_version, self.shadow_state = version, "ready"

    def shadow_status(self):
        return self.shadow_version, self.shadow_state, 1e-3

    def swap_weights(self):
        if self.active:
            from paper_2510_19225_b200._lib import RlbStateError
            raise RlbStateError("weights swap only at a step boundary")
        if self.shadow_state == "empty":
            from paper_2510_19225_b200._lib import RlbStateError
            raise RlbStateError("shadow arena holds no weights")
        self.version, self.shadow_version = self.shadow_version, self.version
        self.shadow_state = "empty"
        return self.version

    def generate(self, request_id, prompt_tokens, prefix_tokens=(), *, target_len):
        if request_id in self.active or request_id in self.pending:
            raise ValueError(f"duplicate request {request_id!r}")
        self.active[request_id] = {"prompt": list(prompt_tokens), "gen": list(prefix_tokens),
                                   "target": target_len, "reported": len(prefix_tokens),
                                   "admitted": False}
        self.pending.append(request_id)

    def step(self, n_steps: int = 16):
        while self.pending and sum(r["admitted"] for r in self.active.values()) < self.max_slots:
            rid = self.pending.pop(0)
            r = self.active[rid]
            r["admitted"] = True
            if len(r["gen"]) < r["target"]:
                r["gen"].append(self.next_token(r["prompt"] + r["gen"]))   # prefill token
        live = [r for r in self.active.values() if r["admitted"]]
        steps = 0
        for _ in range(n_steps):
            moved = False
            for r in live:
                if len(r["gen"]) < r["target"]:
                    r["gen"].append(self.next_token(r["prompt"] + r["gen"]))
                    moved = True
            if not moved:
                break
            steps += 1
        self.last_steps = steps
        out = []
        for rid in sorted(self.active):
            r = self.active[rid]
            new = r["gen"][r["reported"]:]
            done = r["admitted"] and len(r["gen"]) >= r["target"]
            if new or done:
                out.append((rid, np.array(new, np.int32), done))
                r["reported"] = len(r["gen"])
        for rid, _, done in out:
            if done:
                del self.active[rid]
        return out

    def cancel(self, request_id):
        r = self.active.pop(request_id)
        if request_id in self.pending:
            self.pending.remove(request_id)
        return list(r["gen"])

    def export_partials(self, request_ids):
        return [(list(self.active[r]["prompt"]), list(self.active[r]["gen"])) for r in request_ids]

    def status(self):
        st = {"m_pending": len(self.pending), "m_exec": len(self.active) - len(self.pending),
              "weight_version": self.version}
        if self.plan is not None:
            st["plan"] = self.plan
        return st

    def close(self):
        self.closed = True


def reference_continuation(inst: FakeInstance, prompt, target):
    gen: list[int] = []
    while len(gen) < target:
        gen.append(inst.next_token(list(prompt) + gen))
    return gen
