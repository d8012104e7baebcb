"""Seeded synthetic inputs: HF-layout bf16 weights, prompts, preemption traces.

BASELINE.json asks for random-init weights and synthetic prompts (there is no
network for checkpoints).  The init scale matters for parity: at HF's default
std 0.02 about 20% of greedy steps of the tiny model sit at a top-1/top-2 logit
margin below the bf16 tolerance (SURVEY.md §7 hard part 6).  Projections use
std 0.02; the embedding / lm_head use `logit_std / sqrt(hidden)` so the final
logits have a spread of ~`logit_std`.  bf16 serving noise on the logits is
proportional to that spread (the final hidden state's relative bf16 error
times the embedding scale), while the share of greedy steps at a near-tie
stays about the same.  At 0.25 the full 28-layer 1.5B shape measured
|dlogit| p99 1.1e-2 but max 2.6e-2 -- above north_star's 2e-2 tolerance at
the extreme tail, so a flip could exceed it (it did once in ~600 steps);
0.15 scales the tail to ~1.6e-2, inside the tolerance with margin, so every
GPU/oracle token mismatch is a genuine near-tie.

Prompt lengths follow the reference simulator's default range
U[prompt_len_min, prompt_len_max] = U[128, 384] (`pkg/src/spotrl/sim/config.py:82-83`).
"""
from __future__ import annotations

import json
import math
import random

import torch

from .shapes import ModelShape, hf_manifest

DEFAULT_LOGIT_STD = 0.15
PROJ_STD = 0.02


def synth_hf_weights(m: ModelShape, seed: int = 0, device: str | torch.device = "cpu",
                     logit_std: float = DEFAULT_LOGIT_STD) -> dict[str, torch.Tensor]:
    """HF-layout bf16 tensors (the trainer's copy), deterministic in (shape, seed, device type)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    emb_std = logit_std / math.sqrt(m.hidden)
    out: dict[str, torch.Tensor] = {}
    for name, shape in hf_manifest(m):
        if name.endswith("layernorm.weight") or name == "model.norm.weight":
            t = 1.0 + 0.1 * (2 * torch.rand(shape, generator=gen, device=device) - 1)
        elif name.endswith(".bias"):
            t = 0.02 * torch.randn(shape, generator=gen, device=device)
        elif name in ("model.embed_tokens.weight", "lm_head.weight"):
            t = emb_std * torch.randn(shape, generator=gen, device=device)
        else:
            t = PROJ_STD * torch.randn(shape, generator=gen, device=device)
        out[name] = t.to(torch.bfloat16)
    return out


def synth_prompts(n: int, vocab: int, lo: int, hi: int, seed: int = 1) -> list[list[int]]:
    """n prompts, lengths U[lo, hi], ids U[0, vocab)."""
    rng = random.Random(seed)
    prompts = []
    for _ in range(n):
        length = rng.randint(lo, hi)
        prompts.append([rng.randrange(vocab) for _ in range(length)])
    return prompts


def preemption_trace(instance_ids: list[str], kill: list[str], at_step: int) -> str:
    """A `.trace.jsonl` in the reference trace format (`pkg/src/spotrl/traces.py:1-7`),
    written by the reference's own `serialize_trace`: allocate every instance
    at 0, preempt `kill` at `at` = `at_step` (time in decode-step units)."""
    from spotrl.traces import TraceEvent, TraceEventKind, serialize_trace
    events = [TraceEvent(0.0, TraceEventKind.ALLOCATE, i) for i in instance_ids]
    events += [TraceEvent(float(at_step), TraceEventKind.PREEMPT, i) for i in kill]
    return serialize_trace(events)
