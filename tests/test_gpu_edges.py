"""Edge cases of the B200 rollout instance against the CPU fp32 oracle.

* long contexts: > 2048 positions split attention into windows that are
  combined in a second kernel, and a prompt longer than the prefill chunk
  spans several varlen prefill chunks -- parity with the oracle and
  bit-exact migration across both;
* length extremes: 1-token prompts, target_len 1, prompt + target exactly
  max_seq_len, and the capacity / argument errors at and past the limits;
* more requests than slots or KV pages: requests queue, and each one's
  tokens are identical to a run where nothing waits (admission order and
  batch composition never change a token).
"""
import pytest
import torch

from paper_2510_19225_b200.shapes import TINY
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts
from oracle.qwen2_fp32 import Qwen2Fp32, teacher_forced_compare

pytestmark = pytest.mark.gpu
TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def tiny():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = synth_hf_weights(TINY, seed=0, device="cuda")
    return w, Qwen2Fp32(TINY, w)


def _inst(w, **kw):
    from paper_2510_19225_b200.instance import RolloutInstance
    inst = RolloutInstance(TINY, 0, **kw)
    inst.load_weights(w, version=1)
    return inst


def _gen(inst, prompts, target, prefix=None, n_steps=16):
    for i, p in enumerate(prompts):
        inst.generate(f"r{i}", p, prefix[i] if prefix else (), target_len=target)
    got = inst.run_to_completion(n_steps)
    return [(list(prefix[i]) if prefix else []) + got.get(f"r{i}", []) for i in range(len(prompts))]


def test_long_context_windows_and_chunks(tiny):
    """Prompts of 2500-4200 tokens (2-3 attention windows of 2048 positions),
    prefill chunks of 1024 rows: teacher-forced parity with the oracle."""
    w, oracle = tiny
    prompts = synth_prompts(3, TINY.vocab, 2500, 4200, seed=21)
    inst = _inst(w, max_slots=4, max_seq_len=4608, max_prefill_rows=1024)
    gen = _gen(inst, prompts, 96)
    assert all(len(g) == 96 for g in gen)
    rep = teacher_forced_compare(oracle, prompts, gen, TOL_BF16)
    print(f"long context: {rep.steps} steps, exemption rate {rep.exemption_rate:.4f}")
    assert rep.ok, rep.failures[:5]


def test_long_context_migration_bit_exact(tiny):
    """Resume at ~2100-4300 positions (multi-window attention, multi-chunk
    prefill of prompt + prefix) continues bit-identically."""
    w, _ = tiny
    prompts = synth_prompts(4, TINY.vocab, 2000, 4100, seed=22)
    ref = _gen(_inst(w, max_slots=4, max_seq_len=4608), prompts, 200)
    src = _inst(w, max_slots=4, max_seq_len=4608, max_prefill_rows=2048)
    for i, p in enumerate(prompts):
        src.generate(f"r{i}", p, target_len=200)
    for _ in range(4):
        src.step(23)
    exported = src.export_partials([f"r{i}" for i in range(len(prompts))])
    assert all(0 < len(g) < 200 for _, g in exported)
    dst = _inst(w, max_slots=2, max_seq_len=4608, max_prefill_rows=640)
    assert _gen(dst, prompts, 200, prefix=[g for _, g in exported]) == ref


def test_length_extremes(tiny):
    """1-token prompts, target 1, and prompt + target == max_seq_len."""
    w, oracle = tiny
    inst = _inst(w, max_slots=8, max_seq_len=256)
    one = [[7], [4000], [0]]
    gen = _gen(inst, one, 40)
    rep = teacher_forced_compare(oracle, one, gen, TOL_BF16)
    assert rep.ok and all(len(g) == 40 for g in gen)
    assert [len(g) for g in _gen(inst, synth_prompts(3, TINY.vocab, 5, 30, seed=3), 1)] == [1, 1, 1]
    full = synth_prompts(2, TINY.vocab, 200, 200, seed=4)
    gen = _gen(inst, full, 56)                       # 200 + 56 == max_seq_len
    rep = teacher_forced_compare(oracle, full, gen, TOL_BF16)
    assert rep.ok and all(len(g) == 56 for g in gen)


def test_limits_raise(tiny):
    from paper_2510_19225_b200._lib import RlbCapacityError, RlbStateError
    w, _ = tiny
    inst = _inst(w, max_slots=4, max_seq_len=256)
    with pytest.raises(RlbCapacityError):
        inst.generate("big", list(range(200)), target_len=57)        # 257 > max_seq_len
    with pytest.raises(ValueError):
        inst.generate("empty", [], target_len=4)
    with pytest.raises(ValueError):
        inst.generate("oov", [TINY.vocab], target_len=4)
    with pytest.raises(ValueError):
        inst.generate("pre", [1, 2], [3, 4, 5], target_len=2)          # prefix > target
    inst.generate("a", [1, 2, 3], target_len=8)
    with pytest.raises(ValueError):
        inst.generate("a", [1, 2, 3], target_len=8)                    # duplicate id
    with pytest.raises(KeyError):
        inst.cancel("nope")
    assert inst.cancel("a") == []                                       # pending, nothing yet
    assert inst.status()["m_pending"] == 0
    inst.generate("b", [5, 6], target_len=8)
    inst.step(3)
    got = inst.cancel("b")
    assert 1 <= len(got) <= 4
    with pytest.raises(RlbStateError):
        inst.swap_weights()                                             # no shadow weights


def test_queueing_on_slots_and_pages_is_invisible(tiny):
    """40 requests on 6 slots, and on a KV pool of 9 usable pages (+1 the
    scratch slot of bucketed decode batches reserves): every request's tokens
    equal those of a run with room for all of them at once."""
    w, _ = tiny
    prompts = synth_prompts(40, TINY.vocab, 8, 120, seed=31)
    ref = _gen(_inst(w, max_slots=40, max_seq_len=256), prompts, 70)
    assert _gen(_inst(w, max_slots=6, max_seq_len=256), prompts, 70, n_steps=9) == ref
    # each request needs ceil((prompt + 70) / 64) <= 3 pages: at most 3 run at once
    assert _gen(_inst(w, max_slots=16, max_seq_len=256, num_pages=10), prompts, 70) == ref
