#!/usr/bin/env python
"""Generate the committed golden fixtures under tests/golden/ (run in the
builder container; /root/reference and transformers must be importable).

0. qwen15_hf.npz -- the same cross-check at the benchmarked depth: the full
   28-layer Qwen2.5-1.5B shape, greedy tokens + top-32 logits per position.
1. tiny_hf.npz -- the arithmetic oracle's independent cross-check: the tiny
   config-1 decoder with the seeded synthetic weights, run through
   transformers' Qwen2ForCausalLM (fp32, eager attention): greedy tokens and
   last-position logits for 4 prompts.  Pins oracle/qwen2_fp32.py.
2. ref_sim_{migrate,recompute}.jsonl.gz -- event logs of the UNMODIFIED
   reference simulator (pkg/src/spotrl/sim/engine.py) on the first config +
   trace of the reference's fuzzed preemption corpus
   (pkg/tests/test_acceptance.py:191-227), 8 steps,
   plus the counts the reference oracles (pkg/tests/oracles.py) derive from
   them.  Pins oracle/audit.py.
"""
from __future__ import annotations

import dataclasses
import gzip
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
GOLD = os.path.join(ROOT, "tests", "golden")
REF = "/root/reference/pkg"


def tiny_hf():
    from transformers import Qwen2Config, Qwen2ForCausalLM
    from paper_2510_19225_b200.shapes import TINY as m
    from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts
    w = synth_hf_weights(m, seed=0)
    cfg = Qwen2Config(vocab_size=m.vocab, hidden_size=m.hidden, intermediate_size=m.ffn,
                      num_hidden_layers=m.layers, num_attention_heads=m.n_q_heads,
                      num_key_value_heads=m.n_kv_heads, head_dim=m.head_dim,
                      rope_theta=m.rope_theta, rms_norm_eps=m.rms_eps,
                      tie_word_embeddings=m.tied, max_position_embeddings=4096,
                      attn_implementation="eager", torch_dtype=torch.float32)
    hf = Qwen2ForCausalLM(cfg).eval()
    hf.load_state_dict({k: v.float() for k, v in w.items()}, strict=True)
    prompts = synth_prompts(4, m.vocab, 16, 64, seed=1)
    new = 24
    toks, last = [], []
    with torch.no_grad():
        for p in prompts:
            out = hf.generate(torch.tensor([p]), max_new_tokens=new, do_sample=False,
                              min_new_tokens=new)
            g = out[0, len(p):].tolist()
            toks.append(g)
            logits = hf(torch.tensor([p + g[:-1]])).logits[0]
            last.append(logits[len(p) - 1:].numpy()[:: 6])  # every 6th position
    wsum = np.array([float(w[k].float().sum()) for k in sorted(w)], np.float64)
    np.savez_compressed(os.path.join(GOLD, "tiny_hf.npz"),
                        prompt_lens=np.array([len(p) for p in prompts]),
                        prompts=np.concatenate([np.array(p) for p in prompts]),
                        tokens=np.array(toks), logits=np.stack(last).astype(np.float32),
                        weight_sums=wsum)
    print("tiny_hf.npz", np.array(toks)[:, :8])


def qwen15_hf():
    """The full 28-layer Qwen2.5-1.5B shape through transformers (fp32, eager
    attention) on the seeded synthetic weights (CPU generator): greedy tokens
    and the top-32 logits at every generated position for 2 prompts.  Pins
    oracle/qwen2_fp32.py at the depth the bench runs."""
    from transformers import Qwen2Config, Qwen2ForCausalLM
    from paper_2510_19225_b200.shapes import QWEN25_1_5B as m
    from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts
    torch.set_num_threads(os.cpu_count() or 1)
    w = synth_hf_weights(m, seed=0)
    cfg = Qwen2Config(vocab_size=m.vocab, hidden_size=m.hidden, intermediate_size=m.ffn,
                      num_hidden_layers=m.layers, num_attention_heads=m.n_q_heads,
                      num_key_value_heads=m.n_kv_heads, head_dim=m.head_dim,
                      rope_theta=m.rope_theta, rms_norm_eps=m.rms_eps,
                      tie_word_embeddings=m.tied, max_position_embeddings=4096,
                      attn_implementation="eager", torch_dtype=torch.float32)
    hf = Qwen2ForCausalLM(cfg).eval()
    sd = {k: v.float() for k, v in w.items()}
    if m.tied:
        sd["lm_head.weight"] = sd["model.embed_tokens.weight"]
    hf.load_state_dict(sd, strict=True)
    prompts = synth_prompts(2, m.vocab, 40, 60, seed=3)
    new = 12
    toks, topv, topi = [], [], []
    with torch.no_grad():
        for p in prompts:
            out = hf.generate(torch.tensor([p]), max_new_tokens=new, do_sample=False,
                              min_new_tokens=new)
            g = out[0, len(p):].tolist()
            toks.append(g)
            logits = hf(torch.tensor([p + g[:-1]])).logits[0][len(p) - 1:]
            v, i = logits.topk(32, dim=-1)
            topv.append(v.numpy())
            topi.append(i.numpy())
    wsum = np.array([float(w[k].float().sum()) for k in sorted(w)], np.float64)
    np.savez_compressed(os.path.join(GOLD, "qwen15_hf.npz"),
                        prompt_lens=np.array([len(p) for p in prompts]),
                        prompts=np.concatenate([np.array(p) for p in prompts]),
                        tokens=np.array(toks), top_values=np.stack(topv).astype(np.float32),
                        top_indices=np.stack(topi).astype(np.int64), weight_sums=wsum)
    print("qwen15_hf.npz", np.array(toks))


def ref_sim():
    sys.path[:0] = [f"{REF}/src", f"{REF}/tests"]
    from spotrl.sim.config import SimConfig
    from spotrl.sim.engine import run_experiment
    from spotrl.traces import SynthesisParams, synthesize
    import oracles
    import random
    from test_acceptance import fuzz_config, fuzz_trace   # the reference's fuzz corpus, run 0
    rng = random.Random(1234)
    base, trace = fuzz_config(rng), fuzz_trace(rng)
    for policy in ("migrate", "recompute"):
        cfg = dataclasses.replace(base, migration=policy, steps=8)
        res = run_experiment(cfg, trace)
        recs = res.log.records
        facts = {
            "requests": oracles.assert_token_conservation(recs),
            "gated_token_events": oracles.assert_version_gating(recs),
            "preemptions": len(res.log.of_type("preempt")),
            "migrate_out": len(res.log.of_type("migrate_out")),
            "kept_tokens": sum(r["kept_tokens"] for r in res.log.of_type("migrate_out")),
        }
        oracles.assert_stats_closure(recs)
        path = os.path.join(GOLD, f"ref_sim_{policy}.jsonl.gz")
        with gzip.open(path, "wt") as f:
            f.write(json.dumps({"facts": facts}) + "\n")
            f.write(res.log.to_jsonl())
        print(path, facts, len(recs))


if __name__ == "__main__":
    os.makedirs(GOLD, exist_ok=True)
    which = sys.argv[1:] or ["tiny_hf", "qwen15_hf", "ref_sim"]
    for name in which:
        globals()[name]()
