"""The CPU fp32 oracle, pinned against transformers' Qwen2ForCausalLM golden
vectors (tests/golden/tiny_hf.npz, made by scripts/make_golden.py)."""
import os

import numpy as np
import pytest
import torch

from oracle.qwen2_fp32 import ParityReport, Qwen2Fp32, argmax_lowest, teacher_forced_compare
from paper_2510_19225_b200.shapes import TINY
from paper_2510_19225_b200.synth import synth_hf_weights

GOLD = os.path.join(os.path.dirname(__file__), "golden", "tiny_hf.npz")


@pytest.fixture(scope="module")
def golden():
    g = np.load(GOLD)
    lens = g["prompt_lens"]
    flat = g["prompts"].tolist()
    prompts, off = [], 0
    for n in lens:
        prompts.append(flat[off:off + n])
        off += n
    return g, prompts


@pytest.fixture(scope="module")
def tiny_oracle():
    w = synth_hf_weights(TINY, seed=0)
    return w, Qwen2Fp32(TINY, w)


def test_synthetic_weights_are_pinned(golden, tiny_oracle):
    g, _ = golden
    w, _ = tiny_oracle
    sums = np.array([float(w[k].float().sum()) for k in sorted(w)])
    np.testing.assert_allclose(sums, g["weight_sums"], rtol=0, atol=1e-6)


def test_greedy_tokens_match_transformers(golden, tiny_oracle):
    g, prompts = golden
    _, oracle = tiny_oracle
    for p, ref in zip(prompts, g["tokens"]):
        assert oracle.generate(p, len(ref)) == ref.tolist()


def test_logits_match_transformers(golden, tiny_oracle):
    g, prompts = golden
    _, oracle = tiny_oracle
    for i, (p, ref) in enumerate(zip(prompts, g["tokens"])):
        logits = oracle.teacher_forced_logits(p, ref.tolist()).numpy()[::6]
        np.testing.assert_allclose(logits, g["logits"][i], atol=1e-4, rtol=0)


def test_prefix_resume_equals_uninterrupted(tiny_oracle):
    _, oracle = tiny_oracle
    p = list(range(5, 45))
    full = oracle.generate(p, 20)
    assert oracle.generate(p, 20, prefix=full[:7]) == full
    assert oracle.generate(p, 20, prefix=full) == full


def test_argmax_lowest_index_tie_break():
    assert argmax_lowest(torch.tensor([0.5, 2.0, 1.0, 2.0])) == 1


def test_teacher_forced_rule():
    class Fixed:
        def teacher_forced_logits(self, prompt, gen):
            return torch.tensor([[1.0, 0.99, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 3.0]])

    rep = teacher_forced_compare(Fixed(), [[1]], [[1, 0, 2]], 2e-2)   # near-tie flip: exempt
    assert rep.ok and rep.exempt == 1 and rep.steps == 3
    rep = teacher_forced_compare(Fixed(), [[1]], [[0, 1, 2]], 2e-2)   # margin 1.0: failure
    assert not rep.ok and rep.failures[0][:4] == (0, 1, 1, 0)
    assert isinstance(rep, ParityReport)


def test_full_depth_oracle_pinned_to_transformers():
    """The oracle at the benchmarked depth (28-layer Qwen2.5-1.5B shape, the
    seeded synthetic weights) against transformers' Qwen2ForCausalLM
    (tests/golden/qwen15_hf.npz): same greedy tokens, top-32 logits within
    1e-3 at every generated position."""
    from paper_2510_19225_b200.shapes import QWEN25_1_5B
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "qwen15_hf.npz"))
    w = synth_hf_weights(QWEN25_1_5B, seed=0)
    sums = np.array([float(w[k].float().sum()) for k in sorted(w)])
    np.testing.assert_allclose(sums, g["weight_sums"], rtol=0, atol=1e-3)
    oracle = Qwen2Fp32(QWEN25_1_5B, w)
    flat, off = g["prompts"].tolist(), 0
    for k, n in enumerate(g["prompt_lens"]):
        p = flat[off:off + n]
        off += n
        want = g["tokens"][k].tolist()
        logits = oracle.teacher_forced_logits(p, want).numpy()
        assert [argmax_lowest(torch.from_numpy(r)) for r in logits] == want
        got = np.take_along_axis(logits, g["top_indices"][k], axis=1)
        np.testing.assert_allclose(got, g["top_values"][k], rtol=0, atol=1e-3)
