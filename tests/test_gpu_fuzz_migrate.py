"""Fuzzed, multi-hop migration on the GPU under the unmodified reference
control plane (the reference's acceptance corpus,
`pkg/tests/test_acceptance.py:191-254`, criteria 3-4, in reduced form).

Per seed: 4 rollout instances of the tiny decoder share one B200 under
`spotrl.manager.RolloutManager` + `spotrl.transfer.TransferPool` as shipped.
At random flushes an instance is preempted and a replacement registers,
pulls the weights and becomes Active; the next victim is the instance holding
the most already-migrated requests, so requests move more than once; after
every flush the reference `lb_tick` (plateau 2) runs, moving pending requests
to empty queues and, once the queues drain, executing requests above the
plateau onto an instance that runs nothing.  Every request must end bit-identical to an
uninterrupted single-instance rollout, and the reference's own log audits
(`pkg/tests/oracles.py`) must pass."""
import random
from collections import Counter

import pytest
import torch

from oracle import audit
from paper_2510_19225_b200.shapes import TINY
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_19225_b200.instance import RolloutInstance
    w = synth_hf_weights(TINY, seed=0, device="cuda")
    prompts = synth_prompts(48, TINY.vocab, 16, 96, seed=31)
    rng = random.Random(5)
    targets = [rng.randint(60, 160) for _ in prompts]
    ref = RolloutInstance(TINY, 0, max_slots=64, max_seq_len=320, graph_steps=8)
    ref.load_weights(w, version=1)
    for k, p in enumerate(prompts):
        ref.generate(f"r{k}", p, target_len=targets[k])
    want = ref.run_to_completion(16)
    ref.close()
    return w, prompts, targets, want


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_fuzzed_multihop_migration_bit_exact(setup, seed):
    from spotrl.balancer import MigrationKind
    from spotrl.domain import ProfileEntry, ProfileTable
    from spotrl.events import EventLog
    from spotrl.manager import RolloutManager
    from spotrl.transfer import TransferPool, build_agents

    from paper_2510_19225_b200.instance import RolloutInstance
    from paper_2510_19225_b200.runner import RolloutRunner

    w, prompts, targets, want = setup
    rng = random.Random(100 + seed)
    m = RolloutManager(theta=6, m_b=8, log=EventLog())
    m.n_prem_cap = 8
    run = RolloutRunner(m, TransferPool(build_agents(1, 2, 900e9)), flush_steps=rng.choice([4, 8]),
                        model_bytes=TINY.n_bytes(), max_inflight=10)
    m.begin_step(1, run.now())
    run.stage(1, w)

    def new_instance(iid):
        inst = RolloutInstance(TINY, 0, max_slots=12, max_seq_len=320, graph_steps=rng.choice([0, 4]))
        assert run.add_instance(iid, inst)

    for k in range(4):
        new_instance(f"i{k}")
    for k, p in enumerate(prompts):
        run.submit(f"r{k}", p, target_len=targets[k])
    plateau2 = ProfileTable([ProfileEntry(1, 100.0), ProfileEntry(2, 190.0), ProfileEntry(3, 195.0)])
    kills = sorted(rng.sample(range(2, 14), 3))
    next_id = 4
    flush = 0
    late_joined = False
    while not m.all_generated():
        run.pump()
        if kills and flush >= kills[0]:
            kills.pop(0)
            moved = Counter(r["request_id"] for r in m.log.of_type("migrate_out"))
            alive = sorted(run.instances)
            victim = max(alive, key=lambda i: (sum(moved[r] for r in m.executing_sets[i]
                                                   + m.pending_queues[i]), i))
            run.preempt(victim)
            new_instance(f"i{next_id}")
            next_id += 1
            run.pump()
        if not kills and not late_joined and not m.held and \
                not any(m.pending_queues[i] for i in run.instances):
            # a late joiner once the queues are drained: it runs nothing, so
            # the reference lb_tick's executing branch moves requests onto it
            new_instance(f"i{next_id}")
            late_joined = True
        # the reference rebalancer every flush
        run.rebalance(plateau2)
        run.advance()
        flush += 1
        assert flush < 2000
    run.close()

    recs = m.log.records
    assert audit.assert_token_conservation(recs) == len(prompts)
    assert audit.assert_version_gating(recs) > 0
    hops = Counter(r["request_id"] for r in recs if r["type"] == "migrate_out")
    kinds = {o.kind for o in run.lb_orders}
    print(f"seed {seed}: {sum(hops.values())} migrations, max hops {max(hops.values())}, "
          f"lb orders {Counter(o.kind.value for o in run.lb_orders)}, audit source {audit.SOURCE}")
    assert max(hops.values()) >= 2
    assert MigrationKind.EXECUTING in kinds
    for k in range(len(prompts)):
        assert m.requests[f"r{k}"].generated == want[f"r{k}"], f"r{k} diverged"
