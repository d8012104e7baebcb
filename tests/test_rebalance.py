"""Continuous rebalancer (config 5 host side): the restated lb_tick against
the reference's known answers (`pkg/tests/test_balancer.py:81-128`, restated)
and the reference function itself on random registries; and a long-tail
rollout on fake instances with both branches firing, where every request
still completes with exactly the uninterrupted continuation."""
import random

import pytest

from oracle.audit import assert_token_conservation, assert_version_gating
from paper_2510_19225_b200.domain import ProfileEntry, ProfileTable
from paper_2510_19225_b200.events import EventLog
from paper_2510_19225_b200.manager import InstanceLoad, RolloutManager
from paper_2510_19225_b200.rebalance import MigrationKind, MigrationOrder, lb_tick
from paper_2510_19225_b200.runner import RolloutRunner
from paper_2510_19225_b200.transfer import TransferPool, build_agents
from tests.fakes import FakeInstance, reference_continuation


def table(points, cal=0.0):
    return ProfileTable([ProfileEntry(b, t) for b, t in points], cal)


def ex(iid, ks, gen=lambda k: 10 * k):
    return tuple((f"{iid}.e{k}", gen(k)) for k in ks)


CURVE = table([(8, 800.0), (16, 1500.0), (32, 2000.0), (64, 2060.0)])   # plateau 32


def test_pending_branch():
    reg = [InstanceLoad("A"), InstanceLoad("B", pending=("B.p0", "B.p1", "B.p2"))]
    assert lb_tick(reg, table([(1, 10), (2, 20)]), 512.0) == [
        MigrationOrder(("B.p0",), "B", "A", MigrationKind.PENDING)]


def test_executing_branch_moves_cheapest_above_plateau():
    reg = [InstanceLoad("A"), InstanceLoad("B", executing=ex("B", range(48)))]
    (o,) = lb_tick(reg, CURVE, 512.0)
    assert o.kind is MigrationKind.EXECUTING and (o.from_instance, o.to_instance) == ("B", "A")
    assert set(o.request_ids) == {f"B.e{k}" for k in range(16)}


def test_no_order_below_plateau_or_unready_or_idle():
    assert lb_tick([InstanceLoad("A"), InstanceLoad("B", executing=ex("B", range(20)))],
                   CURVE, 512.0) == []
    assert lb_tick([InstanceLoad("A"), InstanceLoad("B", executing=ex("B", range(40)))],
                   ProfileTable(), 512.0) == []
    assert lb_tick([InstanceLoad("A"), InstanceLoad("B")], table([(1, 1), (2, 2)]), 512.0) == []
    reg = [InstanceLoad("A"), InstanceLoad("B", pending=("B.p0",), executing=ex("B", range(40)))]
    assert [o.kind for o in lb_tick(reg, table([(1, 100), (2, 200), (4, 210)]), 512.0)] == \
        [MigrationKind.PENDING]
    with pytest.raises(ValueError):
        MigrationOrder(("x",), "A", "A", MigrationKind.PENDING)


def test_lb_tick_matches_reference(spotrl):
    from spotrl import balancer as rb
    from spotrl.domain import ProfileEntry as RE, ProfileTable as RT
    rng = random.Random(1)
    for _ in range(400):
        reg = []
        for k in range(rng.randint(1, 6)):
            iid = f"i{k:02d}"
            pend = tuple(f"{iid}.p{j}" for j in range(rng.randint(0, 4)))
            exe = tuple((f"{iid}.e{j}", rng.randint(0, 300)) for j in range(rng.randint(0, 12)))
            reg.append((iid, pend, exe))
        pts = [(b, rng.uniform(10, 1000) * b ** 0.5) for b in sorted(rng.sample([1, 2, 4, 8, 16], 3))]
        ours = lb_tick([InstanceLoad(i, p, e) for i, p, e in reg], table(pts), 512.0)
        theirs = rb.lb_tick([rb.InstanceLoad(i, p, e) for i, p, e in reg],
                            RT([RE(b, t) for b, t in pts]), 512.0)
        assert [(o.request_ids, o.from_instance, o.to_instance, o.kind.value) for o in ours] == \
            [(o.request_ids, o.from_instance, o.to_instance, o.kind.value) for o in theirs]


def test_longtail_rollout_with_rebalancing_is_exact():
    m = RolloutManager(theta=4, m_b=4, log=EventLog())
    m.n_prem_cap = 3
    pool = TransferPool(build_agents(1, 2, 900e9))
    run = RolloutRunner(m, pool, flush_steps=4, max_inflight=6)
    m.begin_step(1, run.now())
    pool.stage(1, source={"weights": "v1"}, now=run.now())
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
