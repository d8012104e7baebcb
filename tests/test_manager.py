"""Host manager mirror: reference semantics (pkg/tests/test_manager.py cases,
restated), the reference's own event log for a fixed call script, and -- in
the builder container -- a differential run against the unmodified reference."""
import json
import os
import sys

import pytest

from paper_2510_19225_b200.domain import InstanceStatus, RequestState, RolloutRequest, RouteLeg
from paper_2510_19225_b200.events import EventLog
from paper_2510_19225_b200.manager import GatingViolation, ManagerError, RolloutManager

GOLD = os.path.join(os.path.dirname(__file__), "golden")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "scripts"))
import manager_script  # noqa: E402


def mk(theta=2, migration="migrate", cap=4.0):
    m = RolloutManager(theta=theta, m_b=4, log=EventLog(), migration=migration)
    m.n_prem_cap = cap
    return m


def active(m, iid, version=1, now=0.0):
    m.register_instance(iid, 1, now)
    m.mark_pulling(iid, now)
    m.mark_active(iid, version, now)


def test_append_only_buffer_and_legs():
    r = RolloutRequest("r", prompt_len=5, target_len=10, group_id="g")
    with pytest.raises(ValueError, match="does not match"):
        r.append_tokens("a", [1])
    r.route_history.append(RouteLeg("a"))
    r.append_tokens("a", [1, 2, 3, 4])
    r.route_history.append(RouteLeg("b"))
    r.append_tokens("b", [5, 6, 7, 8, 9, 10])
    assert [leg.tokens for leg in r.route_history] == [4, 6]
    assert r.routed_tokens() == len(r.generated) == 10
    assert r.context_len == 15


def test_migration_keeps_prefix_and_ids():
    m = mk()
    m.begin_step(1, 0.0)
    active(m, "a")
    active(m, "b")
    m.create_request("r", 3, 10, "g", 0.0, prompt_tokens=[7, 8, 9])
    assert m.dispatch(0.0) == [("r", "a")]
    m.admit("r", "a", 0.0)
    m.on_tokens("r", "a", 4, 1.0, token_ids=[11, 12, 13, 14])
    m.migrate_out("r", 2.0, reason="lb_executing")
    assert m.requests["r"].state is RequestState.MIGRATING
    m.route_to("r", "b", 2.0)
    m.admit("r", "b", 2.0)
    m.on_tokens("r", "b", 6, 3.0)
    m.complete("r", "b", 3.0)
    req = m.requests["r"]
    assert req.generated[:4] == [11, 12, 13, 14] and len(req.generated) == 10
    assert [leg.tokens for leg in req.route_history] == [4, 6]


def test_preemption_displaces_in_creation_order_and_is_idempotent():
    m = mk(theta=10)
    m.begin_step(1, 0.0)
    active(m, "a")
    for k in range(4):
        m.create_request(f"r{k}", 3, 5, "g", 0.0)
    m.dispatch(0.0)
    m.admit("r2", "a", 0.0)
    m.admit("r0", "a", 0.0)
    displaced = m.on_preempt("a", 1.0)
    assert displaced == ["r0", "r1", "r2", "r3"]
    assert m.on_preempt("a", 1.0) == []
    assert m.records["a"].status is InstanceStatus.PREEMPTED


def test_recompute_policy_discards_on_preempt_only():
    m = mk(migration="recompute")
    m.begin_step(1, 0.0)
    active(m, "a")
    active(m, "b")
    for rid in ("x", "y"):
        m.create_request(rid, 3, 10, "g", 0.0)
    m.dispatch(0.0)
    for rid, iid in (("x", "a"), ("y", "b")):
        m.admit(rid, iid, 0.0)
        m.on_tokens(rid, iid, 3, 0.5)
    m.migrate_out("y", 1.0, reason="lb_executing")
    assert len(m.requests["y"].generated) == 3
    m.on_preempt("a", 1.0)
    assert m.requests["x"].generated == [] and m.requests["x"].route_history == []


def test_gating_and_desync_errors():
    m = mk()
    m.begin_step(1, 0.0)
    active(m, "a")
    m.create_request("r", 3, 4, "g", 0.0)
    m.dispatch(0.0)
    with pytest.raises(ManagerError, match="stream desync"):
        m.on_tokens("r", "a", 1, 0.0)          # pending, not executing
    m.admit("r", "a", 0.0)
    m.records["a"].weight_version = 0           # stale weights
    with pytest.raises(GatingViolation):
        m.on_tokens("r", "a", 1, 0.0)
    m.records["a"].weight_version = 1
    with pytest.raises(ManagerError, match="overshot"):
        m.on_tokens("r", "a", 5, 0.0)
    with pytest.raises(ValueError):
        m.on_tokens("r", "a", 2, 0.0, token_ids=[1])
    with pytest.raises(ValueError):
        m.records["a"].set_weight_version(0)


def test_stale_instance_is_not_served():
    m = mk()
    m.begin_step(2, 0.0)
    active(m, "old", version=1)
    active(m, "new", version=2)
    assert m.serving_ids() == ["new"]


def test_on_token_batch_bulk_path():
    m = mk()
    m.begin_step(1, 0.0)
    active(m, "a")
    m.create_request("r", 2, 5, "g", 0.0)
    m.create_request("s", 2, 2, "g", 0.0)
    m.dispatch(0.0)
    m.admit("r", "a", 0.0)
    m.admit("s", "a", 0.0)
    n = m.on_token_batch("a", [("r", [1, 2, 3], False), ("s", [4, 5], True)], 1.0)
    assert n == 5 and m.requests["s"].state is RequestState.COMPLETE
    assert m.requests["r"].generated == [1, 2, 3]


def _golden(policy):
    with open(os.path.join(GOLD, f"ref_manager_script_{policy}.jsonl")) as f:
        head = json.loads(f.readline())
        return head["errors"], [json.loads(line) for line in f]


@pytest.mark.parametrize("policy", ["migrate", "recompute"])
def test_reproduces_reference_event_log(policy):
    errors, records = _golden(policy)
    m = RolloutManager(theta=3, m_b=4, log=EventLog(), migration=policy)
    got_errors = manager_script.run(m)
    assert got_errors == errors
    assert json.loads(json.dumps(m.log.records)) == records


@pytest.mark.reference
def test_differential_against_reference(spotrl):
    from spotrl.events import EventLog as RefLog
    from spotrl.manager import RolloutManager as RefManager
    for seed in range(5):
        for policy in ("migrate", "recompute"):
            ref = RefManager(theta=3, m_b=4, log=RefLog(), migration=policy)
            mine = RolloutManager(theta=3, m_b=4, log=EventLog(), migration=policy)
            assert manager_script.run(ref, seed=seed) == manager_script.run(mine, seed=seed)
            assert ref.log.to_jsonl() == mine.log.to_jsonl()
