"""Real weight bytes behind the UNMODIFIED reference `TransferPool`: staging
starts the queued pulls, a pull runs for real, `finish` goes through the
reference's own early-finish guard, preemption aborts."""
import pytest
from spotrl.transfer import TransferPool, build_agents

from paper_2510_19225_b200.transfer import WeightPlane
from tests.fakes import FakeInstance

GB = 1e9


def test_stage_run_finish_through_reference_pool():
    pool = TransferPool(build_agents(1, 2, 6.25 * GB))
    plane = WeightPlane()
    inst = FakeInstance()
    agent = pool.pair_agent("i0")
    assert not pool.request_pull("i0", agent, 4, 28 * GB, float("inf"), 0.0)   # not staged yet
    with pytest.raises(KeyError):
        plane.run(pool, "i0", inst)
    assert plane.stage(pool, 4, {"w": 0}, 1.0) == ["i0"]
    with pytest.raises(RuntimeError, match="no measured pull"):
        plane.finish(pool, "i0", 1.0)
    meas = plane.run(pool, "i0", inst)
    assert inst.version == 4 and meas.bytes == 1 << 20 and meas.gbps > 0
    # the modelled 28 GB at 6.25 GB/s would need 4.48 s: the real bytes landed
    job = plane.finish(pool, "i0", 1.001)
    assert job.bytes_done == job.bytes_total == float(1 << 20)
    assert "i0" not in pool.jobs and not pool.agents[agent].active_pulls


def test_reference_guards_still_apply():
    pool = TransferPool(build_agents(1, 1, 900 * GB))
    plane = WeightPlane()
    plane.stage(pool, 2, object(), 0.0)
    assert pool.request_pull("i0", "agent-0.0", 2, GB, float("inf"), 0.0)
    with pytest.raises(ValueError, match="already pulling"):
        pool.request_pull("i0", "agent-0.0", 2, GB, float("inf"), 0.0)
    with pytest.raises(RuntimeError, match="finished early"):
        pool.finish("i0", 0.0)                  # nothing measured: the modelled guard holds
    pool.abort("i0", 0.5)
    assert "i0" not in pool.jobs
    assert not pool.request_pull("i1", "agent-0.0", 3, GB, float("inf"), 1.0)
    with pytest.raises(KeyError):
        plane.run(pool, "i1", FakeInstance())   # queued, not started


def test_shadow_pull_collect():
    pool = TransferPool(build_agents(1, 1, 900 * GB))
    plane = WeightPlane()
    plane.stage(pool, 5, object(), 0.0)
    inst = FakeInstance()
    assert pool.request_pull("i0", "agent-0.0", 5, GB, float("inf"), 0.0)
    assert plane.run(pool, "i0", inst, shadow=True) is None
    meas = plane.collect(pool, "i0", inst)
    assert meas.shadow and meas.version == 5
    plane.finish(pool, "i0", 0.1)
    assert inst.swap_weights() == 5


def test_a_job_copies_exactly_its_version():
    """A pull started for version 2 keeps copying version 2 even if version 3
    is staged before it runs; version 2 is released once no job names it."""
    pool = TransferPool(build_agents(1, 1, 900 * GB))
    plane = WeightPlane()
    plane.stage(pool, 2, "w2", 0.0)
    assert pool.request_pull("i0", "agent-0.0", 2, GB, float("inf"), 0.0)
    plane.stage(pool, 3, "w3", 0.1)
    got = []
    inst = FakeInstance()
    inst.pull_weights = lambda src, version: (got.append((src, version)),
                                              FakeInstance.pull_weights(inst, src, version))[1]
    plane.run(pool, "i0", inst)
    assert got == [("w2", 2)]
    plane.finish(pool, "i0", 0.2)
    plane.stage(pool, 4, "w4", 0.3)
    assert sorted(plane.sources) == [4]
