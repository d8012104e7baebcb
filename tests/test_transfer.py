"""TransferPool: the reference's known answers (pkg/tests/test_transfer.py,
restated) for the modelled mode, and the measured mode driven by real pulls."""
import pytest

from paper_2510_19225_b200.transfer import TransferAgent, TransferPool, build_agents
from tests.fakes import FakeInstance

GB = 1e9


def pool(n_agents=1, egress=25 * GB):
    return TransferPool(build_agents(1, n_agents, egress))


def test_round_robin_pairing():
    p = pool(2)
    assert [p.pair_agent(f"i{k}") for k in range(4)] == ["agent-0.0", "agent-0.1"] * 2
    single = pool(1)
    assert {single.pair_agent(f"i{k}") for k in range(3)} == {"agent-0.0"}
    with pytest.raises(ValueError):
        TransferPool([])


def test_sole_pull_is_ingress_bound():
    p = pool()
    p.stage_complete(1, 0.0)
    assert p.request_pull("i0", "agent-0.0", 1, 28 * GB, 6.25 * GB, 0.0)
    (t, iid), = p.predictions()
    assert iid == "i0" and t == pytest.approx(4.48)
    job = p.finish("i0", t)
    assert job.bytes_done == job.bytes_total


def test_equal_split_and_reshare_on_finish():
    p = pool(egress=10 * GB)
    p.stage_complete(1, 0.0)
    p.request_pull("a", "agent-0.0", 1, 10 * GB, 100 * GB, 0.0)
    p.request_pull("b", "agent-0.0", 1, 20 * GB, 100 * GB, 0.0)
    assert p.jobs["a"].rate == p.jobs["b"].rate == 5 * GB
    t_a, _ = p.predictions()[0]
    assert t_a == pytest.approx(2.0)
    p.finish("a", t_a)
    assert p.jobs["b"].rate == 10 * GB
    (t_b, _), = p.predictions()
    assert t_b == pytest.approx(3.0)


def test_independent_agents():
    p = pool(2, egress=10 * GB)
    p.stage_complete(1, 0.0)
    p.request_pull("a", "agent-0.0", 1, 10 * GB, 100 * GB, 0.0)
    p.request_pull("b", "agent-0.1", 1, 10 * GB, 100 * GB, 0.0)
    assert [round(t, 6) for t, _ in p.predictions()] == [1.0, 1.0]


def test_queue_until_staged_abort_and_early_finish_guard():
    p = pool()
    assert not p.request_pull("a", "agent-0.0", 2, GB, GB, 0.0)
    assert p.predictions() == []
    assert p.stage_complete(2, 1.0) == ["a"]
    with pytest.raises(RuntimeError, match="finished early"):
        p.finish("a", 1.5)
    p.abort("a", 1.6)
    assert "a" not in p.jobs and p.predictions() == []
    with pytest.raises(ValueError, match="backwards"):
        p.stage_complete(3, 0.5)
    assert p.request_pull("b", "agent-0.0", 2, GB, GB, 2.0)
    with pytest.raises(ValueError, match="already pulling"):
        p.request_pull("b", "agent-0.0", 2, GB, GB, 2.0)


def test_measured_pull_path():
    p = TransferPool([TransferAgent("agent-0.0", "node-0", 900 * GB)])
    inst = FakeInstance()
    started = p.stage(4, source={"w": 0}, now=0.0)
    assert started == []
    assert p.request_pull("i0", "agent-0.0", 4, 0.0, float("inf"), 0.0)
    job = p.run_pull("i0", inst)
    assert inst.version == 4 and job.measured_seconds > 0 and job.measured_gbps > 0
    (t, iid), = p.predictions()
    assert iid == "i0" and t == pytest.approx(job.measured_seconds)
    assert p.finish("i0", 0.0).bytes_done == job.bytes_total
