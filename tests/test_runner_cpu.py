"""RolloutRunner host logic with CPU fake instances: registration + pull,
JSQ dispatch, bulk token flushes, preemption with kept prefixes, and the
reference audits on the resulting event log."""
import random

import pytest

from oracle.audit import assert_token_conservation, assert_version_gating
from paper_2510_19225_b200.events import EventLog
from paper_2510_19225_b200.manager import RolloutManager
from paper_2510_19225_b200.runner import RolloutRunner
from paper_2510_19225_b200.transfer import TransferPool, build_agents
from tests.fakes import FakeInstance, reference_continuation


def make_runner(n_inst=4, theta=64, flush=5, migration="migrate"):
    m = RolloutManager(theta=theta, m_b=4, log=EventLog(), migration=migration)
    m.n_prem_cap = n_inst
    pool = TransferPool(build_agents(1, 2, 900e9))
    run = RolloutRunner(m, pool, flush_steps=flush)
    m.begin_step(1, run.now())
    pool.stage(1, source={"weights": "v1"}, now=run.now())
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
