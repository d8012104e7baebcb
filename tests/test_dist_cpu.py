"""The N>1 host logic over gloo on CPU, at world_size 2 and 8 (the driver's
8-GPU scaling run, which gpurun cannot reach): timing reduction (max over
ranks / sums), object exchange (IPC-handle table, NCCL id), independent
per-rank rollouts with the CPU fake instance; and the 1->7 fan-out plan."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2510_19225_b200 import multi
    from spotrl.events import EventLog
    from spotrl.manager import RolloutManager
    from paper_2510_19225_b200.runner import RolloutRunner
    from tests.fakes import FakeInstance

    assert multi.dist_env() == (ws, rank, rank)
    # each rank: its own instance and prompts (weak scaling), no data-path collective
    m = RolloutManager(theta=64, m_b=4, log=EventLog())
    m.n_prem_cap = 1
    run = RolloutRunner(m, None, flush_steps=7)
    m.begin_step(1, run.now())
    run.add_instance(f"rank{rank}", FakeInstance(vocab=97, max_slots=4))
    for k in range(6):
        run.submit(f"r{rank}-{k}", [rank, k, 1, 2, 3], target_len=20 + k)
    run.run()
    tokens = sum(len(r.generated) for r in m.requests.values())
    secs = 1.0 + rank
    mx, sm = multi.reduce_max_sum([secs, float(tokens)])
    handles = multi.gather_objects({"rank": rank, "ipc": bytes([rank]) * 64})
    uid = multi.broadcast_object(b"nccl-id-from-rank0" if rank == 0 else None)
    value = multi.weak_scaling_value([sm[1]], [mx[0]])
    q.put((rank, mx, sm, [h["rank"] for h in handles], handles[1]["ipc"][:1], uid, value))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 8])
def test_gloo_plumbing(ws):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=300) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tokens_per_rank = sum(20 + k for k in range(6))
    for rank, mx, sm, order, ipc1, uid, value in results:
        assert mx[0] == float(ws) and sm[0] == ws * (ws + 1) / 2    # max / sum of seconds
        assert sm[1] == ws * tokens_per_rank              # every rank's tokens
        assert order == list(range(ws)) and ipc1 == bytes([1])
        assert uid == b"nccl-id-from-rank0"
        assert value == pytest.approx(ws * tokens_per_rank / ws)   # weak scaling: tokens / slowest


@pytest.mark.parametrize("n,rounds", [(1, 1), (3, 8), (7, 8), (7, 3)])
def test_fanout_plan_partitions_the_arena(n, rounds):
    """Scatter + all-gather slices for 1 -> n receivers: every arena byte in
    exactly one (round, receiver) slice, 16-byte aligned, in order."""
    from paper_2510_19225_b200.pull import FanoutPlan
    total = 15_231_233_024           # the 7B weight set of config 4
    plan = FanoutPlan(n, rounds, total)
    edges = [plan.slice(k, j) for k in range(rounds) for j in range(n)]
    assert edges[0][0] == 0 and edges[-1][1] == total
    for (lo, hi), (lo2, _) in zip(edges, edges[1:]):
        assert lo % 16 == 0 and lo < hi == lo2
    sizes = [hi - lo for lo, hi in edges]
    assert max(sizes) - min(sizes) <= 32
