"""End-to-end parity of the B200 rollout instance against the CPU fp32 oracle.

* greedy rollouts, teacher-forced comparison (north_star rule, tolerance 2e-2
  on logits for bf16 serving, exemption rate reported);
* teacher-forced GPU logits vs oracle logits;
* migrate/resume: export partials mid-rollout, resume on a fresh instance via
  generate(prompt, prefix) -> bit-identical to the uninterrupted run;
* weight pull: the engine arena equals the reference re-layout bytewise.
"""
import numpy as np
import pytest
import torch

from paper_2510_19225_b200.shapes import TINY, small_shape, engine_layout, relayout_segments, hf_manifest
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts
from oracle.qwen2_fp32 import Qwen2Fp32, teacher_forced_compare

pytestmark = pytest.mark.gpu
TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return 0


def _instance(shape, w, **kw):
    from paper_2510_19225_b200.instance import RolloutInstance
    inst = RolloutInstance(shape, 0, **kw)
    inst.load_weights(w, version=1)
    return inst


def _rollout(inst, prompts, target, n_steps=16, prefix=None):
    for i, p in enumerate(prompts):
        inst.generate(f"r{i}", p, prefix[i] if prefix else (), target_len=target)
    got = inst.run_to_completion(n_steps)
    return [(list(prefix[i]) if prefix else []) + got.get(f"r{i}", []) for i in range(len(prompts))]


@pytest.fixture(scope="module")
def tiny(cuda):
    w = synth_hf_weights(TINY, seed=0, device="cuda")
    oracle = Qwen2Fp32(TINY, w)
    return w, oracle


def test_tiny_rollout_teacher_forced(tiny):
    """Config 1: 64 prompts (lengths U[16,64]) x 128 greedy tokens."""
    w, oracle = tiny
    prompts = synth_prompts(64, TINY.vocab, 16, 64, seed=1)
    inst = _instance(TINY, w, max_slots=64, max_seq_len=256)
    gen = _rollout(inst, prompts, 128)
    assert all(len(g) == 128 for g in gen)
    rep = teacher_forced_compare(oracle, prompts, gen, TOL_BF16)
    print(f"tiny: {rep.steps} steps, exemption rate {rep.exemption_rate:.4f}")
    assert rep.ok, rep.failures[:5]
    assert rep.exemption_rate < 0.05


def test_tiny_score_logits(tiny):
    w, oracle = tiny
    prompt = synth_prompts(1, TINY.vocab, 200, 200, seed=3)[0]
    inst = _instance(TINY, w, max_slots=8, max_seq_len=512)
    got = inst.score(prompt)
    ref, _ = oracle.forward(prompt)
    err = float(np.abs(got - ref.numpy()).max())
    print("tiny score max |dlogit|", err)
    assert err < 1e-2


def test_tiny_migration_bit_exact(tiny):
    """Kill mid-rollout, resume prompt+prefix on a fresh instance: identical ids."""
    w, _ = tiny
    prompts = synth_prompts(24, TINY.vocab, 16, 300, seed=5)
    ref = _rollout(_instance(TINY, w, max_slots=32, max_seq_len=512), prompts, 160)
    src = _instance(TINY, w, max_slots=32, max_seq_len=512)
    for i, p in enumerate(prompts):
        src.generate(f"r{i}", p, target_len=160)
    partial = {}
    for _ in range(5):   # 1 prefill + up to 5*13 decode steps
        for rid, toks, _ in src.step(13):
            partial.setdefault(rid, []).extend(toks.tolist())
    ids = [f"r{i}" for i in range(len(prompts))]
    exported = src.export_partials(ids)
    for i, (pr, gen) in enumerate(exported):
        assert pr == prompts[i]
        assert gen == partial.get(f"r{i}", [])
        assert 0 < len(gen) < 160
    dst = _instance(TINY, w, max_slots=16, max_seq_len=512)   # smaller batch than the source
    resumed = _rollout(dst, prompts, 160, prefix=[g for _, g in exported])
    assert resumed == ref


@pytest.fixture(scope="module")
def mid(cuda):
    shape = small_shape(layers=2, vocab=8192)
    w = synth_hf_weights(shape, seed=0, device="cuda")
    return shape, w, Qwen2Fp32(shape, w)


def test_qwen_width_rollout_teacher_forced(mid):
    shape, w, oracle = mid
    prompts = synth_prompts(8, shape.vocab, 128, 384, seed=1)
    inst = _instance(shape, w, max_slots=16, max_seq_len=1024)
    gen = _rollout(inst, prompts, 64)
    rep = teacher_forced_compare(oracle, prompts, gen, TOL_BF16)
    print(f"1.5B-width 2L: {rep.steps} steps, exemption rate {rep.exemption_rate:.4f}")
    assert rep.ok, rep.failures[:5]


def test_qwen_width_migration_bit_exact(mid):
    shape, w, _ = mid
    prompts = synth_prompts(12, shape.vocab, 128, 384, seed=7)
    ref = _rollout(_instance(shape, w, max_slots=16, max_seq_len=1024), prompts, 300)
    src = _instance(shape, w, max_slots=16, max_seq_len=1024)
    for i, p in enumerate(prompts):
        src.generate(f"r{i}", p, target_len=300)
    for _ in range(3):
        src.step(37)
    exported = src.export_partials([f"r{i}" for i in range(len(prompts))])
    dst = _instance(shape, w, max_slots=5, max_seq_len=1024, max_prefill_rows=700)
    resumed = _rollout(dst, prompts, 300, prefix=[g for _, g in exported])
    assert resumed == ref


def test_pull_bytewise(mid):
    """The engine arena equals the host-side reference re-layout byte for byte."""
    shape, w, _ = mid
    inst = _instance(shape, w, max_slots=4, max_seq_len=256)
    ptr_, nbytes = inst.arena()
    arena = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    from paper_2510_19225_b200 import _lib
    _lib.check(_lib.lib().rlb_copy_bytes(0, arena.data_ptr(), ptr_, nbytes, None))
    torch.cuda.synchronize()
    names = [n for n, _ in hf_manifest(shape)]
    expect = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    for hf, so, do, nb in relayout_segments(shape):
        src = w[names[hf]].contiguous().view(torch.uint8).flatten()
        expect[do:do + nb] = src[so:so + nb]
    assert torch.equal(arena, expect)


def test_shadow_pull_while_serving_then_swap(tiny):
    """Double-buffered weights: pulling v2 into the shadow
    arena during a v1 rollout leaves that rollout bit-identical; after the
    swap the instance generates exactly what a fresh v2 instance does; a
    second swap (v3 into the old arena) works with the per-arena graphs."""
    from paper_2510_19225_b200._lib import RlbStateError
    w1, _ = tiny
    w2 = synth_hf_weights(TINY, seed=1, device="cuda")
    w3 = synth_hf_weights(TINY, seed=2, device="cuda")
    prompts = synth_prompts(24, TINY.vocab, 16, 48, seed=9)
    ref = {}
    for v, w in ((1, w1), (2, w2), (3, w3)):
        ref[v] = _rollout(_instance(TINY, w, max_slots=32, max_seq_len=256), prompts, 80)
    assert ref[1] != ref[2]
    inst = _instance(TINY, w1, max_slots=32, max_seq_len=256)
    for i, p in enumerate(prompts):
        inst.generate(f"r{i}", p, target_len=80)
    got = {}
    for rid, toks, _ in inst.step(16):
        got.setdefault(rid, []).extend(toks.tolist())
    inst.pull_shadow(w2, version=2)            # in flight while v1 serves
    with pytest.raises(RlbStateError):
        inst.swap_weights()                    # requests still on the instance
    for rid, toks in inst.run_to_completion().items():
        got.setdefault(rid, []).extend(toks)
    assert [got[f"r{i}"] for i in range(len(prompts))] == ref[1]
    v, state, sec = inst.shadow_status()
    assert v == 2 and state == "ready" and sec > 0
    assert inst.swap_weights() == 2 and inst.status()["weight_version"] == 2
    assert inst.shadow_status()[1] == "empty"
    assert _rollout(inst, prompts, 80) == ref[2]
    inst.pull_shadow(w3, version=3)
    assert inst.swap_weights() == 3            # no host wait: ordered on the device
    assert _rollout(inst, prompts, 80) == ref[3]
    # the shadow arena matches the fused re-layout bytewise
    from paper_2510_19225_b200 import _lib
    a_ptr, nbytes = inst.shadow_arena()
    inst.pull_shadow(w1, version=4)
    while inst.shadow_status()[1] != "ready":
        pass
    act = _instance(TINY, w1, max_slots=8, max_seq_len=256)
    p_act, n_act = act.arena()
    assert n_act == nbytes
    bufs = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    for buf, src in zip(bufs, (a_ptr, p_act)):
        _lib.check(_lib.lib().rlb_copy_bytes(0, buf.data_ptr(), src, nbytes, None))
    torch.cuda.synchronize()
    assert torch.equal(bufs[0], bufs[1])


def test_decode_profile_measured(tiny):
    """rlb_decode_profile: per batch size, device-timed decode steps that add
    up to the instance's decode accounting; it builds a ProfileTable the
    plateau rule accepts."""
    from paper_2510_19225_b200.profile import measured_profile_table
    from spotrl.balancer import estimate_plateau
    w, _ = tiny
    prompts = synth_prompts(32, TINY.vocab, 16, 48, seed=12)
    inst = _instance(TINY, w, max_slots=32, max_seq_len=256)
    inst.stats(reset=True)
    for i, p in enumerate(prompts):   # staggered targets: the batch shrinks as requests finish
        inst.generate(f"r{i}", p, target_len=20 + 4 * i)
    inst.run_to_completion(16)
    prof = inst.decode_profile()
    st = inst.stats()
    assert sum(s for _, s, _, _ in prof) == st["decode_steps"]
    assert sum(b * s for b, s, _, _ in prof) == st["decode_rows"]
    assert len(prof) >= 8 and all(sec > 0 for _, _, sec, _ in prof)
    assert all(16 <= ctx <= 256 for _, _, _, ctx in prof)
    t = measured_profile_table(prof)
    assert t.distinct_batch_sizes() == len(prof)
    assert 1 <= estimate_plateau(t, t.context_calibration) <= 32
    assert inst.decode_profile(reset=True) == prof and inst.decode_profile() == []


def test_qwen25_1_5b_full_depth_teacher_forced(cuda):
    """The config-2 model itself (28 layers, 151,936 vocab): greedy rollout on
    the B200 against the fp32 oracle, teacher-forced (bf16 tolerance 2e-2)."""
    from paper_2510_19225_b200.shapes import QWEN25_1_5B
    w = synth_hf_weights(QWEN25_1_5B, seed=0, device="cuda")
    prompts = synth_prompts(3, QWEN25_1_5B.vocab, 48, 96, seed=8)
    inst = _instance(QWEN25_1_5B, w, max_slots=8, max_seq_len=256)
    gen = _rollout(inst, prompts, 24)
    inst.close()
    oracle = Qwen2Fp32(QWEN25_1_5B, w)
    del w
    rep = teacher_forced_compare(oracle, prompts, gen, TOL_BF16)
    print(f"qwen2.5-1.5b 28L: {rep.steps} steps, exemption rate {rep.exemption_rate:.4f}")
    assert rep.ok, rep.failures[:5]
    assert rep.exemption_rate < 0.1


def test_seeding_handoff_bit_exact(tiny):
    """Seeding phase on a real local engine, hand-off to two remote B200
    instances mid-generation: every request's ids equal an
    uninterrupted rollout on one instance."""
    from spotrl.events import EventLog
    from paper_2510_19225_b200.instance import RolloutInstance
    from spotrl.manager import RolloutManager
    from paper_2510_19225_b200.runner import RolloutRunner
    from spotrl.transfer import TransferPool, build_agents
    w, _ = tiny
    prompts = synth_prompts(24, TINY.vocab, 16, 80, seed=17)
    want = _rollout(_instance(TINY, w, max_slots=32, max_seq_len=256), prompts, 90)
    m = RolloutManager(theta=8, m_b=4, log=EventLog())
    m.n_prem_cap = 2
    pool = TransferPool(build_agents(1, 2, 900e9))
    run = RolloutRunner(m, pool, flush_steps=16, max_inflight=12)
    m.begin_step(1, run.now())
    run.stage(1, w)
    run.add_local_engine("local00", _instance(TINY, w, max_slots=16, max_seq_len=256))
    for k, p in enumerate(prompts):
        run.submit(f"r{k}", p, target_len=90)
    for _ in range(2):
        run.pump()
        run.advance()
    for k in range(2):
        assert run.add_instance(f"i{k}", RolloutInstance(TINY, 0, max_slots=16, max_seq_len=256))
    assert run.end_seeding() > 0
    run.run()
    got = [m.requests[f"r{k}"].generated for k in range(len(prompts))]
    run.close()
    assert got == want


def test_qwen7b_width_rollout_and_migration(cuda):
    """7B widths (GQA group 7, 28 q / 4 kv heads, hidden 3584, ffn 18944, untied
    lm_head) at 2 layers: teacher-forced parity with the oracle and bit-exact
    migration resume -- the config 4 / 5 shape family."""
    from paper_2510_19225_b200.shapes import ModelShape
    shape = ModelShape("qwen2.5-7b-2L-v8192", vocab=8192, hidden=3584, layers=2, n_q_heads=28,
                       n_kv_heads=4, head_dim=128, ffn=18_944, tied=False)
    w = synth_hf_weights(shape, seed=3, device="cuda")
    prompts = synth_prompts(6, shape.vocab, 64, 200, seed=13)
    ref = _rollout(_instance(shape, w, max_slots=8, max_seq_len=512), prompts, 48)
    oracle = Qwen2Fp32(shape, w)
    rep = teacher_forced_compare(oracle, prompts, ref, TOL_BF16)
    print(f"7B-width 2L: {rep.steps} steps, exemption rate {rep.exemption_rate:.4f}")
    assert rep.ok, rep.failures[:5]
    src = _instance(shape, w, max_slots=8, max_seq_len=512)
    for i, p in enumerate(prompts):
        src.generate(f"r{i}", p, target_len=48)
    src.step(19)
    exported = src.export_partials([f"r{i}" for i in range(len(prompts))])
    dst = _instance(shape, w, max_slots=3, max_seq_len=512, max_prefill_rows=512)
    assert _rollout(dst, prompts, 48, prefix=[g for _, g in exported]) == ref


@pytest.mark.parametrize("n_prompts", [3, 300])
def test_qkv_two_k_blocks_per_stage_same_tokens(mid, monkeypatch, n_prompts):
    """The 64-column QKV tiles stream two K blocks per stage through 3D TMA
    boxes; the MMAs see the same tiles in the same K order, so the rollout's
    tokens equal the one-block-per-stage kernel's (RLB_QKV_KPS=1)."""
    shape, w, _ = mid
    prompts = synth_prompts(n_prompts, shape.vocab, 128, 384, seed=17)
    got = _rollout(_instance(shape, w, max_slots=512, max_seq_len=1024), prompts, 40)
    monkeypatch.setenv("RLB_QKV_KPS", "1")
    ref = _rollout(_instance(shape, w, max_slots=512, max_seq_len=1024), prompts, 40)
    assert got == ref


@pytest.mark.parametrize("n_prompts", [3, 300])
def test_o_two_k_blocks_per_stage_same_tokens(mid, monkeypatch, n_prompts):
    """The O projection's 128 x 128 split-K tiles on two-K-block stages (3D
    TMA boxes): the same partials, the same tokens (RLB_O_KPS=1 reference)."""
    shape, w, _ = mid
    prompts = synth_prompts(n_prompts, shape.vocab, 128, 384, seed=19)
    got = _rollout(_instance(shape, w, max_slots=512, max_seq_len=1024), prompts, 40)
    monkeypatch.setenv("RLB_O_KPS", "1")
    ref = _rollout(_instance(shape, w, max_slots=512, max_seq_len=1024), prompts, 40)
    assert got == ref


def test_prefill_short_pairs_same_bits(mid, monkeypatch):
    """Prefill row pairs with <= 2 pages of context run on 2-warp attention
    CTAs (the idle warp slots merged as empty partials).  Bit-level A/B:
    teacher-forced logits (rlb_score builds the same pair lists as prefill)
    are bitwise equal to the single 4-warp launch (RLB_ATTN_SPLIT=0); and a
    migration resumed on the split path continues bit-exactly."""
    shape, w, _ = mid
    prompts = synth_prompts(4, shape.vocab, 60, 300, seed=23)
    got = [_instance(shape, w, max_slots=4, max_seq_len=1024, max_prefill_rows=700).score(p)
           for p in prompts]
    with monkeypatch.context() as mp:
        mp.setenv("RLB_ATTN_SPLIT", "0")
        ref = [_instance(shape, w, max_slots=4, max_seq_len=1024, max_prefill_rows=700).score(p)
               for p in prompts]
    for a, b in zip(got, ref):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    # migrate after 20 tokens, resume (prompt + prefix prefill on the split path)
    full = _rollout(_instance(shape, w, max_slots=8, max_seq_len=1024, max_prefill_rows=700),
                    prompts, 48)
    src = _instance(shape, w, max_slots=8, max_seq_len=1024, max_prefill_rows=700, graph_steps=0)
    for i, p in enumerate(prompts):
        src.generate(f"r{i}", p, target_len=48)
    src.step(19)
    parts = src.export_partials([f"r{i}" for i in range(len(prompts))])
    dst = _instance(shape, w, max_slots=8, max_seq_len=1024, max_prefill_rows=300)
    assert _rollout(dst, prompts, 48, prefix=[g for _, g in parts]) == full


def test_numerics_plan_in_config(mid):
    """The split-K factors come from the instance config, are reported in
    status(), and a runner refuses to mix instances with different plans
    (a resume between them would not be bit-exact)."""
    from paper_2510_19225_b200.instance import RolloutInstance
    from paper_2510_19225_b200.runner import RolloutRunner
    from spotrl.events import EventLog
    from spotrl.manager import RolloutManager
    shape, w, _ = mid
    a = RolloutInstance(shape, 0, max_slots=4, max_seq_len=256)
    b = RolloutInstance(shape, 0, max_slots=4, max_seq_len=256, split_o=a_o(a) % 3 + 1)
    assert a.plan != b.plan and a.status()["plan"] == a.plan
    assert "o" + str(a_o(a)) in a.plan
    run = RolloutRunner(RolloutManager(theta=4, m_b=4, log=EventLog()))
    run.manager.n_prem_cap = 4
    run.manager.begin_step(0, 0.0)
    assert run.add_instance("a", a)
    with pytest.raises(ValueError, match="numerics plan"):
        run.add_instance("b", b)
    b.close()
    with pytest.raises(ValueError):
        RolloutInstance(shape, 0, max_slots=4, max_seq_len=256, split_o=99)


def a_o(inst):
    return int(inst.plan.split(".")[2][1:])


def test_active_weights_only_replaced_at_step_boundary(mid):
    """rlb_load_weights refuses to overwrite the serving arena
    while requests are in flight; the shadow arena + swap is the way."""
    from paper_2510_19225_b200._lib import RlbStateError
    shape, w, _ = mid
    inst = _instance(shape, w, max_slots=4, max_seq_len=512)
    inst.generate("r", synth_prompts(1, shape.vocab, 20, 20, seed=3)[0], target_len=8)
    inst.step(2)
    with pytest.raises(RlbStateError):
        inst.load_weights(w, version=2)
    inst.pull_shadow(w, version=2)
    inst.run_to_completion(8)
    assert inst.swap_weights() == 2


def _kv_bytes(inst):
    from paper_2510_19225_b200 import _lib
    p, n = inst.kv_pool()
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().rlb_copy_bytes(0, buf.data_ptr(), p, n, None))
    torch.cuda.synchronize()
    return buf


@pytest.mark.parametrize("case", ["mid-3", "mid-300", "tiny-long"])
def test_attention_tma_same_bits(request, monkeypatch, case):
    """Decode attention with K/V chunks through TMA boxes of the KV pool
    against the per-lane cp.async loads (RLB_ATTN_TMA=0): after the same
    rollout the whole paged KV pool is bytewise identical (every later
    layer's K/V depends on each earlier attention output) and so are the
    tokens.  Covers 1..300 rows, head_dim 128 and 64, multi-window rows."""
    if case.startswith("mid"):
        shape, w, _ = request.getfixturevalue("mid")
        n = int(case.split("-")[1])
        prompts = synth_prompts(n, shape.vocab, 60, 384, seed=29)
        kw, new = dict(max_slots=512, max_seq_len=512), 40
    else:
        w, _ = request.getfixturevalue("tiny")
        shape = TINY
        prompts = synth_prompts(3, TINY.vocab, 2000, 2300, seed=31)
        kw, new = dict(max_slots=4, max_seq_len=2560, max_prefill_rows=1024), 120
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("RLB_ATTN_TMA", flag)
        inst = _instance(shape, w, **kw)
        toks = _rollout(inst, prompts, new)
        out[flag] = (toks, _kv_bytes(inst))
        inst.close()
    assert out["0"][0] == out["1"][0]
    assert torch.equal(out["0"][1], out["1"][1])


def test_bucketed_decode_batches_same_tokens(tiny):
    """A long-tail batch (targets 20..200) decodes on bucketed batch sizes
    padded with scratch-slot rows and whole graphs past a row's target; every
    request's tokens equal a one-request-at-a-time rollout, and the captured
    graphs stay few."""
    w, _ = tiny
    prompts = synth_prompts(40, TINY.vocab, 8, 90, seed=43)
    import random
    rng = random.Random(3)
    targets = [rng.randint(20, 200) for _ in prompts]
    inst = _instance(TINY, w, max_slots=40, max_seq_len=320, graph_steps=8)
    for i, p in enumerate(prompts):
        inst.generate(f"r{i}", p, target_len=targets[i])
    got = inst.run_to_completion(24)
    sizes = {b for b, _, _, _ in inst.decode_profile()}
    inst.close()
    solo = _instance(TINY, w, max_slots=1, max_seq_len=320, graph_steps=0)
    for i, p in enumerate(prompts[:8]):
        solo.generate(f"s{i}", p, target_len=targets[i])
        assert solo.run_to_completion(32)[f"s{i}"] == got[f"r{i}"]
    assert all(len(got[f"r{i}"]) == targets[i] for i in range(len(prompts)))
    assert len(sizes) > 10          # many real batch sizes ...


@pytest.mark.parametrize("case", ["mid", "tiny-long"])
def test_prefill_head16_same_bits(request, monkeypatch, case):
    """Prefill attention packed by head (16 consecutive rows of one sequence
    per CTA and query head, K1h) against the pair kernel for every row
    (RLB_ATTN_HEAD16=0): teacher-forced logits bitwise equal, and after a
    rollout (varlen prefill of many sequences, odd chunk boundaries, + decode)
    the KV pool bytewise equal."""
    if case == "mid":
        shape, w, _ = request.getfixturevalue("mid")
        prompts = synth_prompts(12, shape.vocab, 30, 700, seed=37)
        kw, new = dict(max_slots=16, max_seq_len=1024, max_prefill_rows=1999), 24
    else:
        w, _ = request.getfixturevalue("tiny")
        shape = TINY
        prompts = synth_prompts(3, TINY.vocab, 2000, 2300, seed=41)
        kw, new = dict(max_slots=4, max_seq_len=2560, max_prefill_rows=1500), 16
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("RLB_ATTN_HEAD16", flag)
        inst = _instance(shape, w, **kw)
        logits = inst.score(prompts[0])
        toks = _rollout(inst, prompts, new)
        out[flag] = (logits, toks, _kv_bytes(inst))
        inst.close()
    assert np.array_equal(out["0"][0].view(np.uint32), out["1"][0].view(np.uint32))
    assert out["0"][1] == out["1"][1]
    assert torch.equal(out["0"][2], out["1"][2])


@pytest.mark.parametrize("case", ["mid", "7b-width", "odd-width"])
def test_prefill_split_sum_same_bits(request, monkeypatch, case):
    """Prefill O / down with the pair tile's splits summed on its cluster and
    added into h (EPI_SUMRES) against the [S][R][H] partial slabs summed by
    resid_norm (RLB_SUMRES=0): teacher-forced logits bitwise equal and, after
    a rollout with ragged chunks (rows not a multiple of 256), the KV pool
    bytewise equal -- so a resumed request still continues bit-identically.
    1.5B widths (splits 3 / 5) and 7B widths (splits 4 / 4, 14 n tiles)."""
    extra = {}
    if case == "mid":
        shape, w, _ = request.getfixturevalue("mid")
        n = 14
    elif case == "odd-width":
        # hidden 640: the last 256-column pair tile is half outside N; splits
        # 2 / 3 forced through the instance config
        from paper_2510_19225_b200.shapes import ModelShape
        shape = ModelShape("odd-2L-d640", vocab=4096, hidden=640, layers=2, n_q_heads=5,
                           n_kv_heads=1, head_dim=128, ffn=1792, tied=True)
        w = synth_hf_weights(shape, seed=5, device="cuda")
        n = 14
        extra = dict(split_o=2, split_down=3)
    else:
        from paper_2510_19225_b200.shapes import ModelShape
        shape = ModelShape("qwen2.5-7b-2L-v8192", vocab=8192, hidden=3584, layers=2,
                           n_q_heads=28, n_kv_heads=4, head_dim=128, ffn=18_944, tied=False)
        w = synth_hf_weights(shape, seed=3, device="cuda")
        n = 8
    prompts = synth_prompts(n, shape.vocab, 600, 900, seed=53)
    kw, new = dict(max_slots=16, max_seq_len=1024, max_prefill_rows=2999, **extra), 16
    out = {}
    monkeypatch.setenv("RLB_SUMRES_ROWS", "513")
    # slabs; running sums in L2 scratch; in TMEM; the default (TMEM for O)
    for flag in ("0", "1:0", "1:1", "1"):
        monkeypatch.setenv("RLB_SUMRES", flag[0])
        if ":" in flag:
            monkeypatch.setenv("RLB_SUMRES_TMEM", flag[2])
        else:
            monkeypatch.delenv("RLB_SUMRES_TMEM", raising=False)
        inst = _instance(shape, w, **kw)
        logits = inst.score(prompts[0])
        toks = _rollout(inst, prompts, new)
        out[flag] = (logits, toks, _kv_bytes(inst))
        inst.close()
    for flag in ("1:0", "1:1", "1"):
        assert np.array_equal(out["0"][0].view(np.uint32), out[flag][0].view(np.uint32)), flag
        assert out["0"][1] == out[flag][1], flag
        assert torch.equal(out["0"][2], out[flag][2]), flag
