"""Live mode on CPU: the manager server and instance processes (threads here,
fake instances) over TCP with the reference wire protocol; a connection drop
is a preemption and the displaced requests resume elsewhere; weights pulled
over W/D frames from an agent server."""
import threading

import pytest

from oracle.audit import assert_token_conservation, assert_version_gating
from spotrl.events import EventLog
from paper_2510_19225_b200.live import AgentServer, ManagerServer, serve_instance
from spotrl.manager import RolloutManager
from paper_2510_19225_b200.protocol import ProtocolError, read_frames, write_pull_request
from tests.fakes import FakeInstance, reference_continuation


def _prompts(n):
    import random
    rng = random.Random(11)
    return [[rng.randrange(997) for _ in range(rng.randint(2, 9))] for _ in range(n)]


@pytest.mark.parametrize("die", [None, 40])
def test_live_rollout_over_tcp(die):
    m = RolloutManager(theta=3, m_b=4, log=EventLog())
    m.n_prem_cap = 3
    m.begin_step(1, 0.0)
    srv = ManagerServer(m, version=1, endpoint_for=lambda iid: f"fake://{iid}", max_inflight=4)
    prompts = _prompts(18)
    for k, p in enumerate(prompts):
        srv.submit(f"r{k}", p, 12 + k % 5)
    stop = threading.Event()
    threads = []
    for k in range(3):
        inst = FakeInstance(vocab=997, max_slots=4)
        kw = {"die_after_tokens": die} if (die and k == 1) else {}
        t = threading.Thread(target=serve_instance, args=(srv.address, inst, f"i{k}"),
                             kwargs=dict(open_endpoint=lambda ep, v: ep, n_steps=3, stop=stop, **kw),
                             daemon=True)
        t.start()
        threads.append(t)
    # every instance's register message is queued before the manager starts
    # dispatching, so all three get requests (a late thread under CPU load
    # would otherwise find the work gone and never reach die_after_tokens)
    import time
    t_end = time.monotonic() + 30
    while srv.events.qsize() < 3:
        assert time.monotonic() < t_end
        time.sleep(0.01)
    srv.run_until_done(timeout=60)
    stop.set()
    srv.close()
    recs = m.log.records
    assert assert_token_conservation(recs) == 18
    assert assert_version_gating(recs) > 0
    probe = FakeInstance(vocab=997)
    for k, p in enumerate(prompts):
        assert m.requests[f"r{k}"].generated == reference_continuation(probe, p, 12 + k % 5)
    preempts = [r for r in recs if r["type"] == "preempt"]
    if die:
        assert len(preempts) == 1 and preempts[0]["instance_id"] == "i1"
        assert preempts[0]["displaced"] > 0       # they resumed on i0 / i2 (checked above)
    else:
        assert not preempts


def test_agent_pull_frames():
    agent = AgentServer(shard_bytes=1000)
    blob = bytes(range(256)) * 30
    agent.stage(3, blob)
    import socket
    host, port = agent.address
    with socket.create_connection((host, port)) as s, s.makefile("rwb") as f:
        write_pull_request(f, 3)
        f.flush()
        frames = list(read_frames(f))
    assert [k for k, _ in frames] == [b"W"] * 8 + [b"D"]
    assert b"".join(p for k, p in frames if k == b"W") == blob
    with socket.create_connection((host, port)) as s, s.makefile("rwb") as f:
        write_pull_request(f, 4)                  # not staged: EOF, no frames
        f.flush()
        assert list(read_frames(f)) == []
    agent.close()


def test_live_refuses_a_mismatched_numerics_plan():
    """An instance whose numerics plan differs from the first one's is
    refused (its connection closed -> handled as a preemption): a request
    resumed across plans would not continue bit-exactly."""
    m = RolloutManager(theta=3, m_b=4, log=EventLog())
    m.n_prem_cap = 3
    m.begin_step(1, 0.0)
    srv = ManagerServer(m, version=1, endpoint_for=lambda iid: f"fake://{iid}", max_inflight=4)
    prompts = _prompts(8)
    for k, p in enumerate(prompts):
        srv.submit(f"r{k}", p, 300)         # long enough that i1 registers mid-run
    stop = threading.Event()
    mgr = threading.Thread(target=srv.run_until_done, kwargs=dict(timeout=60), daemon=True)
    mgr.start()
    import time
    for k, plan in enumerate(["v2.q1.o3.d5.w2048.a2.p64.t0", "v2.q1.o2.d5.w2048.a2.p64.t0"]):
        inst = FakeInstance(vocab=997, max_slots=4, plan=plan)
        t = threading.Thread(target=serve_instance, args=(srv.address, inst, f"i{k}"),
                             kwargs=dict(open_endpoint=lambda ep, v: ep, n_steps=3, stop=stop),
                             daemon=True)
        t.start()
        t_end = time.monotonic() + 30
        while k == 0 and srv.plan is None:  # i0's plan is the reference one
            assert time.monotonic() < t_end
            time.sleep(0.01)
    mgr.join(timeout=90)
    assert not mgr.is_alive()
    stop.set()
    srv.close()
    recs = m.log.records
    assert [r["instance_id"] for r in recs if r["type"] == "plan_mismatch"] == ["i1"]
    assert assert_token_conservation(recs) == 8
    probe = FakeInstance(vocab=997)
    for k, p in enumerate(prompts):
        assert m.requests[f"r{k}"].generated == reference_continuation(probe, p, 300)
