"""Host bookkeeping on the rollout path, one core:
the unmodified reference manager's token collection per token and in bulk
flushes, and migrate_out + route_to per request.

    python scripts/host_bench.py [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
B, STEPS, K = 512, 64, 64


def bench(mod_manager, mod_events, label, bulk):
    m = mod_manager.RolloutManager(theta=B, m_b=16, log=mod_events.EventLog())
    m.n_prem_cap = 2
    for iid in ("i0", "i1"):
        m.register_instance(iid, 1, 0.0)
        m.mark_active(iid, 0, 0.0)
    m.begin_step(0, 0.0)
    for r in range(B):
        m.create_request(f"r{r}", 16, STEPS * K + 1, "g", 0.0)
    m.dispatch(0.0)
    for iid in ("i0", "i1"):
        for rid in list(m.pending_queues[iid]):
            m.admit(rid, iid, 0.0)
    owner = dict(m.owner)
    out = {}
    t0 = time.perf_counter()
    for _ in range(STEPS):                        # per token: count=1, B requests, K steps
        for _k in range(K):
            for rid, iid in owner.items():
                m.on_tokens(rid, iid, 1, 0.0)
            if not bulk:
                break
        if not bulk:
            break
    dt = time.perf_counter() - t0
    n = B * (STEPS * K if bulk else 1)
    out["on_tokens_count1_tok_per_s"] = n / dt
    # bulk: count=K per request per flush
    m2 = mod_manager.RolloutManager(theta=B, m_b=16, log=mod_events.EventLog())
    m2.n_prem_cap = 2
    for iid in ("i0", "i1"):
        m2.register_instance(iid, 1, 0.0)
        m2.mark_active(iid, 0, 0.0)
    m2.begin_step(0, 0.0)
    for r in range(B):
        m2.create_request(f"r{r}", 16, STEPS * K + 1, "g", 0.0)
    m2.dispatch(0.0)
    for iid in ("i0", "i1"):
        for rid in list(m2.pending_queues[iid]):
            m2.admit(rid, iid, 0.0)
    owner2 = dict(m2.owner)
    t0 = time.perf_counter()
    for _ in range(STEPS):
        for rid, iid in owner2.items():
            m2.on_tokens(rid, iid, K, 0.0)
    dt = time.perf_counter() - t0
    out["on_tokens_bulk_k64_tok_per_s"] = B * STEPS * K / dt
    t0 = time.perf_counter()
    for rid in list(owner2)[:B // 2]:
        m2.migrate_out(rid, 0.0, reason="lb_pending" if False else "preempt")
        m2.route_to(rid, "i1" if owner2[rid] == "i0" else "i0", 0.0)
    dt = time.perf_counter() - t0
    out["migrate_out_route_to_us_per_request"] = 1e6 * dt / (B // 2)
    out["impl"] = label
    return out


def main():
    import platform
    import paper_2510_19225_b200  # noqa: F401  (puts the installed reference on sys.path)
    from spotrl import events as rev, manager as rman   # unmodified reference
    res = [bench(rman, rev, "reference spotrl", bulk=True)]
    doc = {"cpu": platform.processor() or platform.machine(), "cores": 1, "B": B,
           "flushes": STEPS, "tokens_per_flush": K, "results": res}
    print(json.dumps(doc, indent=1))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
