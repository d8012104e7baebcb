"""RolloutRunner host logic with CPU fake instances: registration + pull,
JSQ dispatch, bulk token flushes, preemption with kept prefixes, and the
reference audits on the resulting event log."""
import random

import pytest

from oracle.audit import assert_token_conservation, assert_version_gating
from spotrl.events import EventLog
from spotrl.manager import RolloutManager
from paper_2510_19225_b200.runner import RolloutRunner
from spotrl.transfer import TransferPool, build_agents
from tests.fakes import FakeInstance, reference_continuation


def make_runner(n_inst=4, theta=64, flush=5, migration="migrate"):
    m = RolloutManager(theta=theta, m_b=4, log=EventLog(), migration=migration)
    m.n_prem_cap = n_inst
    pool = TransferPool(build_agents(1, 2, 900e9))
    run = RolloutRunner(m, pool, flush_steps=flush)
    m.begin_step(1, run.now())
    run.stage(1, {"weights": "v1"})
    for k in range(n_inst):
        assert run.add_instance(f"i{k}", FakeInstance(vocab=997, max_slots=6))
    return run


def prompts(n, seed=0):
    rng = random.Random(seed)
    return [[rng.randrange(997) for _ in range(rng.randint(3, 12))] for _ in range(n)]


@pytest.mark.parametrize("kill", [None, {12: ["i1", "i3"]}, {1: ["i0"], 20: ["i2"]}])
def test_rollout_with_preemption_completes_identically(kill):
    run = make_runner()
    ps = prompts(40)
    for k, p in enumerate(ps):
        run.submit(f"r{k}", p, target_len=30 + k % 7)
    out = run.run(kill_at=kill)
    recs = run.manager.log.records
    assert assert_token_conservation(recs) == 40
    assert assert_version_gating(recs) > 0
    probe = FakeInstance(vocab=997)
    for k, p in enumerate(ps):
        assert run.manager.requests[f"r{k}"].generated == reference_continuation(probe, p, 30 + k % 7)
    if kill:
        kept = sum(v["kept_tokens"] for key, v in out.items() if key.startswith("resume_"))
        assert kept > 0
        assert all(v["resume_ms_max"] is not None for key, v in out.items() if key.startswith("resume_"))
    run.close()


def test_recompute_policy_regenerates_from_scratch():
    run = make_runner(migration="recompute")
    ps = prompts(16, seed=3)
    for k, p in enumerate(ps):
        run.submit(f"r{k}", p, target_len=25)
    run.run(kill_at={10: ["i0"]})
    recs = run.manager.log.records
    assert assert_token_conservation(recs) == 16
    preempt_outs = [r for r in recs if r["type"] == "migrate_out" and r["reason"] == "preempt"]
    assert preempt_outs and all(r["kept_tokens"] == 0 for r in preempt_outs)
    run.close()


def test_step_boundary_swap_has_no_pull_window():
    """Version 2 is pulled into every instance's shadow arena while version 1
    still serves; begin_step(2) swaps it in and the instances are Active at 2
    immediately (no pull between step_start and instance_active)."""
    run = make_runner(n_inst=3)
    m, pool = run.manager, run.pool
    ps = prompts(18, seed=5)
    for k, p in enumerate(ps):
        run.submit(f"a{k}", p, target_len=20)
    run.pump()
    run.advance()
    run.stage(2, {"weights": "v2"})
    assert run.prefetch(2) == ["i0", "i1", "i2"]
    assert all(m.records[i].status.value == "active" and m.records[i].weight_version == 1
               for i in run.instances)
    run.run()                                  # step 1 finishes on version 1
    assert m.all_generated()
    out = run.begin_step(2)
    assert all(v["swapped"] for v in out.values()) and len(out) == 3
    assert all(m.records[i].weight_version == 2 for i in run.instances)
    assert all(inst.version == 2 for inst in run.instances.values())
    recs = m.log.records
    t_step = [r for r in recs if r["type"] == "step_start" and r["version"] == 2][0]["t"]
    swaps = [r for r in recs if r["type"] == "pull_done" and r.get("swapped")]
    assert len(swaps) == 3 and all(r["t"] >= t_step for r in swaps)
    for k, p in enumerate(prompts(12, seed=6)):
        run.submit(f"b{k}", p, target_len=15)
    run.run()
    assert assert_version_gating(m.log.records) > 0
    assert assert_token_conservation(m.log.records) == 30
    run.close()


def test_begin_step_without_prefetch_pulls_blocking():
    run = make_runner(n_inst=2)
    for k, p in enumerate(prompts(4, seed=7)):
        run.submit(f"a{k}", p, target_len=8)
    run.run()
    run.stage(2, {"weights": "v2"})
    out = run.begin_step(2)
    assert out and not any(v["swapped"] for v in out.values())
    assert all(run.manager.records[i].weight_version == 2 for i in run.instances)
    run.close()


def test_swap_refused_with_requests_in_flight():
    from paper_2510_19225_b200._lib import RlbStateError
    inst = FakeInstance()
    inst.pull_shadow(None, 2)
    inst.generate("r", [1, 2, 3], target_len=4)
    with pytest.raises(RlbStateError):
        inst.swap_weights()


def test_seeding_handoff_to_remotes():
    """Local engines serve first (ungated); when the remotes are Active,
    end_seeding hands every local request to them with its prefix, and each
    completes exactly like an uninterrupted continuation."""
    m = RolloutManager(theta=6, m_b=4, log=EventLog())
    m.n_prem_cap = 2
    pool = TransferPool(build_agents(1, 2, 900e9))
    run = RolloutRunner(m, pool, flush_steps=4, max_inflight=6)
    m.begin_step(1, run.now())
    run.stage(1, {"weights": "v1"})
    for k in range(2):
        run.add_local_engine(f"local{k:02d}", FakeInstance(vocab=997, max_slots=6))
    ps = prompts(20, seed=9)
    for k, p in enumerate(ps):
        run.submit(f"r{k}", p, target_len=25)
    for _ in range(3):                      # seeding: only the local engines serve
        run.pump()
        run.advance()
    assert all(m.owner[r].startswith("local") for r in m.owner)
    for k in range(2):
        assert run.add_instance(f"i{k}", FakeInstance(vocab=997, max_slots=6))
    handed = run.end_seeding()
    assert handed > 0 and not m.local_ids
    run.run()
    recs = m.log.records
    assert any(r["type"] == "seeding_end" and r["handed_off"] == handed for r in recs)
    assert sum(1 for r in recs if r["type"] == "migrate_out" and r["reason"] == "seed_handoff") == handed
    assert assert_token_conservation(recs) == 20
    assert assert_version_gating(recs) > 0
    probe = FakeInstance(vocab=997)
    for k, p in enumerate(ps):
        assert m.requests[f"r{k}"].generated == reference_continuation(probe, p, 25)
    run.close()


def test_preempted_instance_torn_down_off_the_resume_path():
    """A killed instance leaves the serving set at once, but its device
    teardown waits until the run ends (a dead process frees nothing on the
    survivors' critical path); the resume report splits out the host phases."""
    run = make_runner()
    victim = run.instances["i1"]
    for k, p in enumerate(prompts(24, seed=3)):
        run.submit(f"r{k}", p, target_len=25)
    seen = []
    orig = run.preempt

    def preempt(iid):
        out = orig(iid)
        seen.append((iid not in run.instances, victim.closed))
        return out

    run.preempt = preempt
    out = run.run(kill_at={8: ["i1"]})
    assert seen == [(True, False)]
    assert victim.closed
    rep = out["resume_i1"]
    assert rep["preempt_ms"] >= 0 and rep["route_submit_ms"] >= 0
    run.close()


def test_late_joiner_receives_executing_requests():
    """A spot instance registering mid-step (join_at) pulls, goes Active, and
    the reference lb_tick's executing branch moves requests above the plateau
    onto it (config 5's elastic case); every request stays exact."""
    from spotrl.balancer import MigrationKind
    from spotrl.domain import ProfileEntry, ProfileTable
    m = RolloutManager(theta=64, m_b=4, log=EventLog())
    m.n_prem_cap = 3
    pool = TransferPool(build_agents(1, 1, 900e9))
    run = RolloutRunner(m, pool, flush_steps=4, max_inflight=12)
    m.begin_step(1, run.now())
    run.stage(1, {"weights": "v1"})
    for k in range(2):
        assert run.add_instance(f"i{k}", FakeInstance(vocab=997, max_slots=12))
    ps = prompts(24, seed=13)
    for k, p in enumerate(ps):
        run.submit(f"r{k}", p, target_len=60)
    table = ProfileTable([ProfileEntry(1, 100.0), ProfileEntry(2, 190.0), ProfileEntry(4, 200.0)])
    run.run(profile=table, lb_every=1, join_at={8: [("i2", FakeInstance(vocab=997, max_slots=12))]})
    assert "i2" in m.records and m.records["i2"].status.value == "active"
    assert any(o.kind is MigrationKind.EXECUTING and o.to_instance == "i2" for o in run.lb_orders)
    recs = m.log.records
    assert assert_token_conservation(recs) == 24
    probe = FakeInstance(vocab=997)
    for k, p in enumerate(ps):
        assert m.requests[f"r{k}"].generated == reference_continuation(probe, p, 60)
    run.close()
