"""The real-id response buffer beside the UNMODIFIED reference manager
(`spotrl.manager.RolloutManager`): ids land in the reference's own
`RolloutRequest.generated`, every reference check still fires (and keeps
nothing on failure), migration keeps the real prefix, recompute drops it, and
the pending-depth `dispatch` routes exactly like the reference's."""
import random

import pytest
from spotrl.domain import RequestState
from spotrl.events import EventLog
from spotrl.manager import GatingViolation, ManagerError, RolloutManager

from paper_2510_19225_b200.responses import ResponseBuffer, dispatch


def mk(theta=2, migration="migrate", cap=4.0):
    m = RolloutManager(theta=theta, m_b=4, log=EventLog(), migration=migration)
    m.n_prem_cap = cap
    return m, ResponseBuffer(m)


def active(m, iid, version=1, now=0.0):
    m.register_instance(iid, 1, now)
    m.mark_pulling(iid, now)
    m.mark_active(iid, version, now)


def test_real_ids_in_reference_buffer_and_prefix_survives_migration():
    m, rb = mk()
    m.begin_step(1, 0.0)
    active(m, "a")
    active(m, "b")
    rb.create_request("r", [7, 8, 9], 10, "g", 0.0)
    assert m.requests["r"].prompt_len == 3 and rb.prompt("r") == [7, 8, 9]
    assert dispatch(m, 0.0) == [("r", "a")]
    m.admit("r", "a", 0.0)
    rb.on_tokens("r", "a", [11, 12, 13, 14], 1.0)
    m.migrate_out("r", 2.0, reason="lb_executing")
    assert rb.prefix("r") == [11, 12, 13, 14]
    m.route_to("r", "b", 2.0)
    m.admit("r", "b", 2.0)
    n = rb.on_flush("b", [("r", [21, 22, 23, 24, 25, 26], True)], 3.0)
    req = m.requests["r"]
    assert n == 6 and req.state is RequestState.COMPLETE
    assert req.generated == [11, 12, 13, 14, 21, 22, 23, 24, 25, 26]
    assert [leg.tokens for leg in req.route_history] == [4, 6]
    toks = m.log.of_type("tokens")
    assert [(r["count"], r["total"]) for r in toks] == [(4, 4), (6, 10)]
    # the reference's microbatch carries the real ids to the trainer
    mb = m.seal_microbatch(4.0, force=True)
    assert mb.responses[0].generated[-1] == 26


def test_recompute_policy_drops_the_prefix():
    m, rb = mk(migration="recompute")
    m.begin_step(1, 0.0)
    active(m, "a")
    active(m, "b")
    for rid in ("x", "y"):
        rb.create_request(rid, [1, 2, 3], 10, "g", 0.0)
    dispatch(m, 0.0)
    for rid, iid in (("x", "a"), ("y", "b")):
        m.admit(rid, iid, 0.0)
        rb.on_tokens(rid, iid, [5, 6, 7], 0.5)
    m.migrate_out("y", 1.0, reason="lb_executing")
    assert rb.prefix("y") == [5, 6, 7]
    m.on_preempt("a", 1.0)
    assert rb.prefix("x") == [] and m.requests["x"].route_history == []


def test_reference_errors_keep_nothing():
    m, rb = mk()
    m.begin_step(1, 0.0)
    active(m, "a")
    rb.create_request("r", [1, 2, 3], 4, "g", 0.0)
    dispatch(m, 0.0)
    with pytest.raises(ManagerError, match="stream desync"):
        rb.on_tokens("r", "a", [9], 0.0)              # pending, not executing
    m.admit("r", "a", 0.0)
    m.records["a"].weight_version = 0                   # stale weights
    with pytest.raises(GatingViolation):
        rb.on_tokens("r", "a", [9], 0.0)
    m.records["a"].weight_version = 1
    rb.on_tokens("r", "a", [1, 2], 0.0)
    assert m.requests["r"].generated == [1, 2]
    with pytest.raises(ManagerError, match="overshot"):
        rb.on_tokens("r", "a", [3, 4, 5], 0.0)
    with pytest.raises(ManagerError, match="completed at"):
        rb.on_flush("a", [("r", [], True)], 0.0)
    with pytest.raises(ManagerError, match="duplicate request"):
        rb.create_request("r", [1], 4, "g", 0.0)


def _scenario(seed, dispatcher):
    """Random creates / preemptions / completions / registrations; returns the log."""
    rng = random.Random(seed)
    m = RolloutManager(theta=rng.randint(1, 4), m_b=4, log=EventLog())
    m.n_prem_cap = 8
    m.begin_step(1, 0.0)
    ids = [f"i{k}" for k in range(rng.randint(1, 5))]
    for iid in ids:
        active(m, iid)
    t = 0.0
    for k in range(60):
        t += 1.0
        op = rng.random()
        if op < 0.5:
            m.create_request(f"r{k}", 4, 3, "g", t)
        elif op < 0.65:
            alive = [i for i in ids if m.records[i].status.value == "active"]
            if len(alive) > 1:
                victim = rng.choice(alive)
                for rid in sorted(m.on_preempt(victim, t), key=m.request_seq.__getitem__,
                                  reverse=True):
                    m.hold(rid, front=True)
        else:
            for iid in ids:
                q = m.pending_queues.get(iid) or []
                if q and rng.random() < 0.5:
                    rid = q[0]
                    m.admit(rid, iid, t)
                    m.on_tokens(rid, iid, 3, t)
                    m.complete(rid, iid, t)
        routed = dispatcher(m, t)
        m.log.emit(t, "dispatched", routed=[list(r) for r in routed])
    return m.log.to_jsonl()


def test_dispatch_matches_reference():
    for seed in range(40):
        assert _scenario(seed, dispatch) == _scenario(seed, RolloutManager.dispatch)
