#!/usr/bin/env python
"""Config 3: token-level migration under a synthetic preemption trace.

N rollout instances (one per visible GPU, driven from one host process with a
thread per GPU -- the C ABI releases the GIL) run config 2 each (Qwen2.5-1.5B
shape, `--prompts` prompts x `--new-tokens` tokens per instance) under the
host RolloutManager mirror.  A `.trace.jsonl` in the reference trace format
(`pkg/src/spotrl/traces.py:1-7`) preempts `--kill` instances at decode step
`--kill-at`; their requests keep every flushed token (`migrate_out`,
`pkg/src/spotrl/manager.py:336-357`), are re-routed by JSQ to the survivors
and resumed there with one varlen prefill of prompt + prefix.

Reported (one JSON line): rollout tokens/s with the preemption, per-survivor
resume prefill device time, resume ms = kill -> first post-resume token of the
last migrated request (wall, includes one flush interval), bit-exactness of
every request against an uninterrupted run (`--check`), and the reference
log audits (token conservation, single ownership, version gating) on the
event log.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=0, help="0 = one per visible GPU")
    ap.add_argument("--prompts", type=int, default=512)
    ap.add_argument("--new-tokens", type=int, default=1024)
    ap.add_argument("--kill-at", type=int, default=512)
    ap.add_argument("--kill", type=int, default=-1, help="instances to preempt (default N/4)")
    ap.add_argument("--flush-steps", type=int, default=32)
    ap.add_argument("--check", action="store_true", help="also run uninterrupted and compare")
    ap.add_argument("--shape", default="qwen2.5-1.5b")
    args = ap.parse_args()

    import torch
    from oracle.audit import assert_token_conservation, assert_version_gating
    from paper_2510_19225_b200 import _lib
    from paper_2510_19225_b200.instance import RolloutInstance
    from paper_2510_19225_b200.runner import RolloutRunner
    from paper_2510_19225_b200.shapes import SHAPES
    from paper_2510_19225_b200.synth import preemption_trace, synth_hf_weights, synth_prompts
    from spotrl.events import EventLog
    from spotrl.manager import RolloutManager
    from spotrl.traces import TraceEventKind, parse_trace
    from spotrl.transfer import TransferPool, build_agents

    shape = SHAPES[args.shape]
    n_gpu = torch.cuda.device_count()
    n = args.instances or n_gpu
    kill_n = args.kill if args.kill >= 0 else max(1, n // 4)
    ids = [f"i{k}" for k in range(n)]
    victims = ids[1::max(1, n // kill_n)][:kill_n] if kill_n else []
    trace = preemption_trace(ids, victims, args.kill_at)
    kill_at: dict[int, list[str]] = {}
    for ev in parse_trace(trace.splitlines()):
        if ev.kind is TraceEventKind.PREEMPT:
            kill_at.setdefault(int(ev.at), []).append(ev.instance_id)

    # trainer weights on GPU 0; every instance pulls them (peer reads over NVLink)
    w = synth_hf_weights(shape, seed=0, device="cuda:0")
    for d in range(1, n_gpu):
        _lib.check(_lib.lib().rlb_enable_peer(d, 0))
    extra = -(-args.prompts * kill_n // max(1, n - kill_n))
    max_slots = args.prompts + extra
    max_seq = 384 + args.new_tokens
    prompts = synth_prompts(args.prompts * n, shape.vocab, 128, 384, seed=2024)

    def build(tag):
        log = EventLog()
        m = RolloutManager(theta=args.prompts, m_b=16, log=log)
        m.n_prem_cap = n
        pool = TransferPool(build_agents(1, 1, 900e9))
        run = RolloutRunner(m, pool, flush_steps=args.flush_steps, model_bytes=shape.n_bytes())
        m.begin_step(1, run.now())
        run.stage(1, w)
        for k, iid in enumerate(ids):
            inst = RolloutInstance(shape, k % n_gpu, max_slots=max_slots, max_seq_len=max_seq,
                                   graph_steps=16)
            assert run.add_instance(iid, inst)
        for r, p in enumerate(prompts):
            run.submit(f"{tag}{r}", p, target_len=args.new_tokens)
        return run

    out = {"metric": "migration resume ms", "config": {
        "workload": f"config3: {n} instances x {args.prompts} prompts x {args.new_tokens} tokens "
                    f"({shape.name}), preempt {victims} at decode step {args.kill_at}",
        "flush_steps": args.flush_steps}}
    run = build("r")
    out["pull"] = run.pull_log
    t0 = time.perf_counter()
    stats_before = {}
    res = run.run(kill_at=kill_at)
    wall = time.perf_counter() - t0
    total = sum(len(q.generated) for q in run.manager.requests.values())
    out["rollout_tokens_per_s_wall"] = total / wall
    out["wall_s"] = wall
    out["resume"] = {k: v for k, v in res.items() if k.startswith("resume_")}
    surv = [i for i in ids if i not in victims]
    out["survivor_prefill_ms"] = {i: run.instances[i].stats()["prefill_ms"] for i in surv}
    recs = run.manager.log.records
    out["audit"] = {"requests_conserved": assert_token_conservation(recs),
                    "gated_token_events": assert_version_gating(recs)}
    migrated = {r["request_id"] for r in recs if r["type"] == "migrate_out"}
    out["migrated_requests"] = len(migrated)
    out["kept_tokens"] = sum(r["kept_tokens"] for r in recs if r["type"] == "migrate_out")
    got = {rid[1:]: q.generated for rid, q in run.manager.requests.items()}
    run.close()
    if args.check:
        ref = build("u")
        ref.run()
        want = {rid[1:]: q.generated for rid, q in ref.manager.requests.items()}
        ref.close()
        mism = [k for k in want if want[k] != got[k]]
        out["bit_exact_vs_uninterrupted"] = not mism
        out["mismatched_requests"] = len(mism)
        out["migrated_bit_exact"] = all(want[r[1:]] == got[r[1:]] for r in migrated)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
