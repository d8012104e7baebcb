"""Live mode on a B200: real instances behind the wire protocol.  One pulls
its weights over TCP W/D frames from an agent server (the cross-node path,
landing in a pinned buffer + GPU staging blob + fused re-layout), the other
from trainer memory; one drops its connection mid-rollout.  Every request's
ids equal a direct in-process rollout."""
import threading

import pytest
import torch

from paper_2510_19225_b200.shapes import TINY
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts

pytestmark = pytest.mark.gpu


def test_live_instances_over_tcp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.audit import assert_token_conservation
    from paper_2510_19225_b200 import _lib
    from spotrl.events import EventLog
    from paper_2510_19225_b200.instance import RolloutInstance
    from paper_2510_19225_b200.live import AgentServer, ManagerServer, TcpPulledSource, serve_instance
    from spotrl.manager import RolloutManager
    from paper_2510_19225_b200.pull import TrainerWeights

    w = synth_hf_weights(TINY, seed=0, device="cuda")
    trainer = TrainerWeights(TINY, 0, w)
    agent = AgentServer(shard_bytes=1 << 20)
    agent.stage(1, trainer.blob.cpu().numpy())

    # TCP-pulled arena == directly loaded arena, byte for byte
    direct = RolloutInstance(TINY, 0, max_slots=32, max_seq_len=512)
    direct.load_weights(w, version=1)
    src = TcpPulledSource(agent.endpoint, 1, TINY, 0)
    via_tcp = RolloutInstance(TINY, 0, max_slots=8, max_seq_len=512)
    via_tcp.load_weights(src, version=1)
    bufs = []
    for inst in (direct, via_tcp):
        p, n = inst.arena()
        b = torch.empty(n, dtype=torch.uint8, device="cuda")
        _lib.check(_lib.lib().rlb_copy_bytes(0, b.data_ptr(), p, n, None))
        bufs.append(b)
    torch.cuda.synchronize()
    assert torch.equal(bufs[0], bufs[1])

    prompts = synth_prompts(20, TINY.vocab, 8, 64, seed=41)
    targets = [40 + 7 * (k % 4) for k in range(20)]
    for k, p in enumerate(prompts):
        direct.generate(f"r{k}", p, target_len=targets[k])
    want = direct.run_to_completion(16)

    m = RolloutManager(theta=4, m_b=4, log=EventLog())
    m.n_prem_cap = 2
    m.begin_step(1, 0.0)
    ends = {"i0": agent.endpoint, "i1": "local://trainer"}
    srv = ManagerServer(m, version=1, endpoint_for=ends.__getitem__, max_inflight=6)
    for k, p in enumerate(prompts):
        srv.submit(f"r{k}", p, targets[k])

    def resolve(endpoint, version):
        if endpoint.startswith("tcp://"):
            return TcpPulledSource(endpoint, version, TINY, 0)
        return trainer

    stop = threading.Event()
    threads = []
    for iid, die in (("i0", None), ("i1", 150)):
        inst = RolloutInstance(TINY, 0, max_slots=6, max_seq_len=512)
        t = threading.Thread(target=serve_instance, args=(srv.address, inst, iid),
                             kwargs=dict(open_endpoint=resolve, n_steps=8, stop=stop,
                                         die_after_tokens=die), daemon=True)
        t.start()
        threads.append(t)
    srv.run_until_done(timeout=120)
    stop.set()
    srv.close()
    agent.close()
    recs = m.log.records
    assert assert_token_conservation(recs) == 20
    assert [r for r in recs if r["type"] == "preempt"][0]["displaced"] > 0
    for k in range(20):
        assert m.requests[f"r{k}"].generated == want[f"r{k}"]
