#!/usr/bin/env python
"""Config 5: long-tail rollout with continuous load rebalancing.

N rollout instances (one per visible GPU, one host process, a thread per GPU)
serve Qwen2.5-7B-shape requests whose target lengths follow a long-tailed
distribution in [256, 8192] tokens.  Requests are placed by Alg. 2 JSQ with
delayed dispatch (`theta`), each instance admits at most `--max-inflight` of
them (the rest stay pending in the manager, like the reference GenUnit's
max_concurrency), and -- in the rebalanced run -- `lb_tick` runs every
`--lb-every` flushes (`pkg/src/spotrl/sim/engine.py:850-882`): pending
requests move to instances with empty queues, and once queues drain,
executing requests above the batching plateau move to idle instances,
resuming from prompt + prefix with one varlen prefill.

The plateau comes from the measured decode profile of the first (static)
run, exactly like the reference's `profile_prev` (`engine.py:928-939`):
`RolloutInstance.decode_profile` -> `ProfileTable` -> `estimate_plateau`.

Reported (one JSON line): makespan and tokens/s of the static and the
rebalanced run, orders by kind, migrated requests, the measured profile and
plateau, and whether every request's tokens are identical in both runs
(migration must not change a single token).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def longtail_lengths(n: int, lo: int, hi: int, seed: int) -> list[int]:
    """Lognormal response lengths (median ~2.5x lo, heavy right tail), clipped."""
    import numpy as np
    rng = np.random.default_rng(seed)
    x = rng.lognormal(mean=np.log(2.5 * lo), sigma=0.9, size=n)
    return [int(v) for v in np.clip(x, lo, hi)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=0, help="0 = one per visible GPU")
    ap.add_argument("--prompts", type=int, default=96, help="requests per instance")
    ap.add_argument("--min-len", type=int, default=256)
    ap.add_argument("--max-len", type=int, default=8192)
    ap.add_argument("--max-inflight", type=int, default=64)
    ap.add_argument("--theta", type=int, default=8)
    ap.add_argument("--flush-steps", type=int, default=32)
    ap.add_argument("--lb-every", type=int, default=2)
    ap.add_argument("--epsilon", type=float, default=0.05)
    ap.add_argument("--shape", default="qwen2.5-7b")
    ap.add_argument("--profile", choices=["calibrate", "online"], default="calibrate",
                    help="plateau from a calibration sweep at one context (default) or from the "
                         "static run's online decode profile")
    ap.add_argument("--late-join", type=int, default=0,
                    help="the last instance registers after this many decode steps (a spot "
                         "instance arriving mid-step; 0 = all from the start)")
    ap.add_argument("--kv-gb", type=float, default=0.0,
                    help="KV page pool per instance in GB (0 = max_inflight x max_seq)")
    ap.add_argument("--no-warmup", action="store_true",
                    help="skip the discarded first run (it captures the decode graphs of every "
                         "batch size, so the timed runs compare like with like)")
    args = ap.parse_args()

    import torch
    from oracle.audit import assert_token_conservation, assert_version_gating
    from paper_2510_19225_b200 import _lib
    from paper_2510_19225_b200.instance import RolloutInstance
    from paper_2510_19225_b200.profile import calibrate_profile, measured_profile_table
    from paper_2510_19225_b200.runner import RolloutRunner
    from paper_2510_19225_b200.shapes import SHAPES
    from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts
    from spotrl.balancer import MigrationKind, estimate_plateau
    from spotrl.events import EventLog
    from spotrl.manager import RolloutManager
    from spotrl.transfer import TransferPool, build_agents

    shape = SHAPES[args.shape]
    n_gpu = torch.cuda.device_count()
    n = args.instances or n_gpu
    ids = [f"i{k}" for k in range(n)]
    w = synth_hf_weights(shape, seed=0, device="cuda:0")      # trainer-held weights
    for d in range(1, n_gpu):
        _lib.check(_lib.lib().rlb_enable_peer(d, 0))
    total = args.prompts * n
    prompts = synth_prompts(total, shape.vocab, 128, 384, seed=77)
    targets = longtail_lengths(total, args.min_len, args.max_len, seed=78)
    max_seq = 384 + args.max_len
    kv_tok = 2 * shape.layers * shape.n_kv_heads * shape.head_dim * 2
    pages = int(args.kv_gb * 1e9 / (64 * kv_tok)) if args.kv_gb > 0 else 0
    instances = {iid: RolloutInstance(shape, k % n_gpu, max_slots=args.max_inflight,
                                      max_seq_len=max_seq, graph_steps=16, num_pages=pages)
                 for k, iid in enumerate(ids)}
    late = ids[-1] if args.late_join > 0 else None

    def run_once(tag, profile):
        m = RolloutManager(theta=args.theta, m_b=16, log=EventLog())
        m.n_prem_cap = n
        pool = TransferPool(build_agents(1, 1, 900e9))
        run = RolloutRunner(m, pool, flush_steps=args.flush_steps, model_bytes=shape.n_bytes(),
                            max_inflight=args.max_inflight)
        m.begin_step(1, run.now())
        run.stage(1, w)
        for iid in ids:
            instances[iid].decode_profile(reset=True)
            if iid != late:
                assert run.add_instance(iid, instances[iid])
        join = {args.late_join: [(late, instances[late])]} if late else None
        for r, (p, t) in enumerate(zip(prompts, targets)):
            run.submit(f"r{r}", p, target_len=t)
        t0 = time.perf_counter()
        run.run(profile=profile, lb_every=args.lb_every if profile is not None else 0,
                epsilon=args.epsilon, join_at=join)
        wall = time.perf_counter() - t0
        recs = m.log.records
        res = {"wall_s": wall,
               "tokens_per_s": sum(len(q.generated) for q in m.requests.values()) / wall,
               "decode_steps_max": run.decode_steps,
               "audit": {"requests_conserved": assert_token_conservation(recs),
                         "gated_token_events": assert_version_gating(recs)}}
        if profile is not None:
            res["orders"] = {k.value: sum(1 for o in run.lb_orders if o.kind is k)
                             for k in MigrationKind}
            res["moved_requests"] = {k.value: sum(len(o.request_ids) for o in run.lb_orders
                                                  if o.kind is k) for k in MigrationKind}
            res["resumed_tokens"] = sum(r["kept_tokens"] for r in recs
                                        if r["type"] == "migrate_out")
        points = [pt for iid in ids for pt in instances[iid].decode_profile()]
        got = {rid: list(q.generated) for rid, q in m.requests.items()}
        run.instances.clear()            # the instances are reused by the next run
        if run._exec is not None:
            run._exec.shutdown()
        return res, got, points

    if not args.no_warmup:
        run_once("w", None)
    static, got_static, points = run_once("s", None)
    online = measured_profile_table(points)
    if args.profile == "calibrate":
        # every batch size at one context (the instances are idle between runs)
        sizes = [b for b in (1, 2, 4, 8, 16, 32, 48, 64, 96, 128, 160, 192, 224, 256, 320, 384,
                             448, 512) if b <= args.max_inflight]
        table = calibrate_profile(instances[ids[0]], sizes, prompt_len=256, steps=32)
    else:
        table = online
    plateau = estimate_plateau(table, table.context_calibration, epsilon=args.epsilon)
    rebal, got_rebal, _ = run_once("b", table)
    same = [r for r in got_static if got_static[r] == got_rebal[r]]
    out = {"metric": "long-tail rollout makespan s", "value": rebal["wall_s"], "unit": "s",
           "higher_is_better": False,
           "config": {"workload": f"config5: {n} instances x {args.prompts} requests "
                                  f"({shape.name}), response lengths lognormal in "
                                  f"[{args.min_len}, {args.max_len}], JSQ theta={args.theta}, "
                                  f"max_inflight={args.max_inflight}, lb_tick every "
                                  f"{args.lb_every} flushes of {args.flush_steps} steps"
                                  + (f", {late} joins at decode step {args.late_join}"
                                     if late else ""),
                      "target_len_mean": sum(targets) / len(targets),
                      "target_len_max": max(targets)},
           "static": static, "rebalanced": rebal,
           "speedup": static["wall_s"] / rebal["wall_s"],
           "profile": {"source": args.profile,
                       "online_entries": [[e.batch_size, round(e.decode_throughput, 1)]
                                          for e in online.entries],
                       "entries": [[e.batch_size, round(e.decode_throughput, 1)]
                                   for e in table.entries],
                       "context_calibration": table.context_calibration,
                       "plateau": plateau, "epsilon": args.epsilon},
           "tokens_identical": len(same) == len(got_static), "requests": len(got_static)}
    for inst in instances.values():
        inst.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
