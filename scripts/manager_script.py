"""A fixed, seeded call script over the RolloutManager API shared by the
reference (`pkg/src/spotrl/manager.py`) and the B200 mirror
(`paper_2510_19225_b200/manager.py`).  Both must produce the same event log
and raise the same errors; tests/golden/ref_manager_script_*.jsonl holds the
reference's output.  Exercises registration (incl. cap rejection and duplicate
registration), version gating, JSQ dispatch with theta, admission, bulk
tokens, completion, LB-style migration (migrate_out + route_to), preemption
(displacement order, idempotence) and the stream-desync / overshoot errors."""
from __future__ import annotations

import random


def _try(errors: list, fn, *a, **kw):
    try:
        return fn(*a, **kw)
    except Exception as exc:  # record the error class, keep going
        errors.append(type(exc).__name__)
        return None


def run(mgr, seed: int = 3, steps: int = 3) -> list[str]:
    rng = random.Random(seed)
    errors: list[str] = []
    t = 0.0
    mgr.n_prem_cap = 3.0
    for i in range(4):                       # the 4th is rejected (cap 3)
        _try(errors, mgr.register_instance, f"i{i}", 1, t)
    _try(errors, mgr.register_instance, "i0", 1, t)   # duplicate
    for step in range(1, steps + 1):
        t += 1.0
        mgr.begin_step(step, t)
        for iid in ("i0", "i1", "i2"):
            if iid in mgr.records and mgr.records[iid].status.value != "preempted":
                mgr.mark_pulling(iid, t)
                mgr.mark_active(iid, step, t)
        for k in range(10):
            mgr.create_request(f"s{step}r{k}", 20 + k, 12 + (k % 5), f"g{k // 2}", t)
        # a stale-version instance would be gated: i2 lags one version in step 2
        if step == 2:
            mgr.records["i2"].weight_version = 1
        for _ in range(400):
            t += 0.25
            mgr.dispatch(t)
            for iid in sorted(mgr.pending_queues):
                for rid in list(mgr.pending_queues[iid]):
                    if rng.random() < 0.7:
                        mgr.admit(rid, iid, t)
            executing = [(iid, rid) for iid in sorted(mgr.executing_sets)
                         for rid in mgr.executing_sets[iid]]
            for iid, rid in executing:
                req = mgr.requests[rid]
                left = req.target_len - len(req.generated)
                k = min(left, rng.randint(0, 4))
                if k:
                    _try(errors, mgr.on_tokens, rid, iid, k, t)
                if len(req.generated) == req.target_len and req.state.value == "executing":
                    mgr.complete(rid, iid, t)
            r = rng.random()
            live = [i for i in ("i0", "i1", "i2") if i in mgr.records
                    and mgr.records[i].status.value == "active"]
            if r < 0.04 and executing:        # LB migration of an executing request
                iid, rid = executing[rng.randrange(len(executing))]
                others = [i for i in live if i != iid and mgr.records[i].weight_version == step]
                if others and mgr.requests[rid].state.value == "executing":
                    mgr.migrate_out(rid, t, reason="lb_executing")
                    mgr.route_to(rid, rng.choice(others), t)
            elif r < 0.09 and len(live) > 1:  # preemption + re-hold at the front
                victim = rng.choice(live)
                displaced = mgr.on_preempt(victim, t)
                mgr.on_preempt(victim, t)     # idempotent
                for rid in sorted(displaced, key=lambda x: mgr.request_seq[x], reverse=True):
                    mgr.hold(rid, front=True)
            for iid in ("i0", "i1", "i2"):   # replacement instance joins (pull -> active)
                if mgr.records[iid].status.value == "preempted" and rng.random() < 0.1:
                    mgr.register_instance(iid, 1, t)
                    mgr.mark_pulling(iid, t)
                    mgr.mark_active(iid, step, t)
            if all(q.state.value == "complete" for q in mgr.requests.values()
                   if q.request_id.startswith(f"s{step}")):
                break
        # error paths
        done = [rid for rid, q in mgr.requests.items() if q.state.value == "complete"]
        if done:
            _try(errors, mgr.on_tokens, done[0], "i0", 1, t)      # stream desync
    return errors
