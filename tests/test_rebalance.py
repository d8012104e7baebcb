"""Continuous rebalancer (config 5 host side): the reference's own `lb_tick`
orders applied by the runner to (fake) instances -- a long-tail rollout with
both branches firing, where every request still completes with exactly the
uninterrupted continuation."""
import random

from spotrl.balancer import MigrationKind
from spotrl.domain import ProfileEntry, ProfileTable
from spotrl.events import EventLog
from spotrl.manager import RolloutManager
from spotrl.transfer import TransferPool, build_agents

from oracle.audit import assert_token_conservation, assert_version_gating
from paper_2510_19225_b200.runner import RolloutRunner
from tests.fakes import FakeInstance, reference_continuation


def table(points, cal=0.0):
    return ProfileTable([ProfileEntry(b, t) for b, t in points], cal)


def test_longtail_rollout_with_rebalancing_is_exact():
    m = RolloutManager(theta=4, m_b=4, log=EventLog())
    m.n_prem_cap = 3
    pool = TransferPool(build_agents(1, 2, 900e9))
    run = RolloutRunner(m, pool, flush_steps=4, max_inflight=6)
    m.begin_step(1, run.now())
    run.stage(1, {"weights": "v1"})
    for k in range(3):
        assert run.add_instance(f"i{k}", FakeInstance(vocab=997, max_slots=6))
    rng = random.Random(3)
    prompts = [[rng.randrange(997) for _ in range(rng.randint(3, 9))] for _ in range(30)]
    # long tail: JSQ dispatch deals requests round-robin at first, so every
    # third (long) request lands on i0 while i1 / i2 drain their short ones
    targets = [rng.choice([90, 140]) if k % 3 == 0 else rng.choice([8, 10, 12])
               for k in range(len(prompts))]
    for k, (p, t) in enumerate(zip(prompts, targets)):
        run.submit(f"r{k}", p, target_len=t)
    plateau2 = table([(1, 100.0), (2, 190.0), (3, 195.0)])         # plateau = 2
    run.run(profile=plateau2, lb_every=1)
    kinds = {o.kind for o in run.lb_orders}
    assert kinds == {MigrationKind.PENDING, MigrationKind.EXECUTING}
    recs = m.log.records
    assert any(r["type"] == "lb_order" for r in recs)
    assert assert_token_conservation(recs) == 30
    assert assert_version_gating(recs) > 0
    probe = FakeInstance(vocab=997)
    for k, (p, t) in enumerate(zip(prompts, targets)):
        assert m.requests[f"r{k}"].generated == reference_continuation(probe, p, t)
    run.close()
