#!/usr/bin/env python
"""Rollout tokens/s on B200 (BASELINE.json metric), config 2 per instance.

Workload (BASELINE.json configs[1]): Qwen2.5-1.5B-shape decoder, random-init
bf16 weights (seeded), 512 synthetic prompts of length U[128, 384] per
instance, 1024 greedy new tokens each (EOS ignored), one independent instance
per GPU (weak scaling: every rank runs its own 512 prompts; no data-path
collective).  One bench "step" = one full rollout of the 512 prompts.

Printed JSON line (rank 0):
  value        generated tokens of all ranks / max-over-ranks device time of the
               rollout (CUDA events on each instance's stream: prefill + decode;
               inputs resident, host bookkeeping excluded)
  e2e          the same tokens / max-over-ranks wall time of the public-API
               calls (RolloutInstance.generate x512 + step() until done): prompt
               H2D, token-ring D2H and the host response buffer inside
  roofline     the dominant kernel (split-K paged decode attention), re-launched
               mid-rollout on the instance stream and timed with CUDA events;
               achieved = algorithmic K+V(+q,out) bytes per launch / avg duration
  cpu_baseline BASELINE.md §4, rank 0 at N=1 only, on the box's host cores:
               the fp32 CPU oracle (oracle/qwen2_fp32.py, batched greedy
               decode, all threads) on config 2 REDUCED to 16 prompts x 64
               tokens (`value`) and on config 1 in full; the CPU model; and
               the reference's own host code on the path (unmodified
               spotrl RolloutManager.on_tokens / migrate_out + route_to,
               TransferPool's modelled pull time), 1 core
`--impl reference` times only the CPU decoder (the reference has no decoder
of its own -- SURVEY.md §0 -- so its CPU path is the oracle port), each step
a batched rollout of 8 prompts x 64 tokens.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PROMPTS = 512
NEW_TOKENS = 1024
P_LO, P_HI = 128, 384
MAX_SEQ = 1408            # P_HI + NEW_TOKENS
CPU_SAMPLE = (16, 64)     # config 2 reduced: prompts x new tokens
REF_ARM_SAMPLE = (8, 64)  # --impl reference: one step = a batched rollout of this sample
NCU_ATTN_FILE = "profiles/r2_attn_mid_ncu.json"   # ncu --set full of the profiled launch
HBM_KERNELS = ("attention", "resid_norm")   # bytes-bound (others: FLOPs)   # ncu --set full capture of K1 (traffic)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--prompts", type=int, default=N_PROMPTS)
    ap.add_argument("--new-tokens", type=int, default=NEW_TOKENS)
    ap.add_argument("--flush-steps", type=int, default=64, help="decode steps per rlb_step call")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prefill-rows", type=int, default=18944,
                    help="token rows per prefill chunk (74 x 256: whole pair-tile waves)")
    ap.add_argument("--split-o", type=int, default=0, help="O split-K (0 = measured default)")
    ap.add_argument("--split-down", type=int, default=0, help="down split-K (0 = measured default)")
    ap.add_argument("--profile-at", type=float, default=0.5,
                    help="fraction of the rollout's tokens after which the kernels are profiled")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: --prompts in total, split over the ranks (default: weak, "
                         "--prompts per rank)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()

    def summary(self) -> dict:
        rows = [r for r in self.rows if len(r) >= 7 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [r for r in rows if r[6].isdigit() and int(r[6]) > 50] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in busy for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(int(r[0]) for r in busy),
                "sm_max_mhz": int(rows[0][1]), "reasons": reasons, "samples": len(busy)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


def cpu_oracle_rollout(shape, weights_cpu, n: int, new: int, lo: int, hi: int, seed: int,
                       threads: int) -> tuple[int, float]:
    """Batched greedy rollout of n prompts x new tokens on the fp32 CPU oracle:
    (generated tokens, seconds)."""
    import torch
    from oracle.qwen2_fp32 import Qwen2Fp32
    from paper_2510_19225_b200.synth import synth_prompts
    torch.set_num_threads(threads)
    oracle = Qwen2Fp32(shape, weights_cpu)
    prompts = synth_prompts(n, shape.vocab, lo, hi, seed=seed)
    t0 = time.perf_counter()
    gens = oracle.generate_batch(prompts, new)
    return sum(len(g) for g in gens), time.perf_counter() - t0


def reference_host_path() -> dict:
    """The reference's own code on the path, unmodified (`spotrl`), 1 core
    (BASELINE.md §4 item 2): token collection per token and in bulk flushes,
    migrate_out + route_to per request, and the TransferPool's modelled pull
    time for the config-2 and config-4 weight bytes at its default TCP rate."""
    import paper_2510_19225_b200  # noqa: F401  (the installed reference on sys.path)
    from spotrl.events import EventLog
    from spotrl.manager import RolloutManager
    from spotrl.transfer import TransferPool, build_agents
    B, STEPS, K = 512, 16, 64

    def manager():
        m = RolloutManager(theta=B, m_b=16, log=EventLog())
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
        return m, dict(m.owner)

    out = {"cores": 1, "impl": "spotrl (unmodified reference)"}
    m, owner = manager()
    t0 = time.perf_counter()
    for _ in range(K):
        for rid, iid in owner.items():
            m.on_tokens(rid, iid, 1, 0.0)
    out["on_tokens_count1_tok_per_s"] = B * K / (time.perf_counter() - t0)
    m, owner = manager()
    t0 = time.perf_counter()
    for _ in range(STEPS):
        for rid, iid in owner.items():
            m.on_tokens(rid, iid, K, 0.0)
    out["on_tokens_bulk_k64_tok_per_s"] = B * STEPS * K / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    for rid in list(owner)[:B // 2]:
        m.migrate_out(rid, 0.0, reason="preempt")
        m.route_to(rid, "i1" if owner[rid] == "i0" else "i0", 0.0)
    out["migrate_out_route_to_us_per_request"] = 1e6 * (time.perf_counter() - t0) / (B // 2)
    for label, nbytes in (("config2_1.5b", 3_087_428_608), ("config4_7b", 15_231_233_024)):
        pool = TransferPool(build_agents(1, 1, 25e9))
        pool.stage_complete(1, 0.0)
        pool.request_pull("i0", "agent-0.0", 1, float(nbytes), 6.25e9, 0.0)
        out[f"transferpool_modelled_pull_s_{label}"] = pool.predictions()[0][0]
    return out


def cpu_baseline(shape, threads: int) -> dict:
    """config 2 reduced (value), config 1 in full, host path."""
    from paper_2510_19225_b200.shapes import TINY
    from paper_2510_19225_b200.synth import synth_hf_weights
    n, new = CPU_SAMPLE
    w = synth_hf_weights(shape, seed=0, device="cpu")
    toks, sec = cpu_oracle_rollout(shape, w, n, new, P_LO, P_HI, seed=77, threads=threads)
    del w
    wt = synth_hf_weights(TINY, seed=0, device="cpu")
    t1, s1 = cpu_oracle_rollout(TINY, wt, 64, 128, 16, 64, seed=1, threads=threads)
    return {"value": toks / sec, "unit": "tokens/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"REDUCED config 2: {n} prompts (len U[{P_LO},{P_HI}]) x {new} greedy "
                      f"tokens, batched fp32 torch CPU oracle, {sec:.1f}s",
            "config1_full": {"value": t1 / s1, "unit": "tokens/s", "seconds": round(s1, 2),
                             "sample": "64 prompts (len U[16,64]) x 128 tokens, tiny decoder"},
            "reference_host_path": reference_host_path()}


def run_reference(args):
    """--impl reference: the CPU implementation of the path, timed on host cores."""
    from paper_2510_19225_b200.shapes import QWEN25_1_5B
    from paper_2510_19225_b200.synth import synth_hf_weights
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    w = synth_hf_weights(QWEN25_1_5B, seed=0, device="cpu")
    n, new = REF_ARM_SAMPLE
    toks = secs = 0.0
    for i in range(args.warmup + args.steps):
        t, sec = cpu_oracle_rollout(QWEN25_1_5B, w, n, new, P_LO, P_HI, seed=100 + i,
                                    threads=threads)
        if i >= args.warmup:
            toks += t
            secs += sec
    value = toks / secs
    sample = (f"{n} prompts (len U[{P_LO},{P_HI}]) x {new} greedy tokens per step, batched fp32 "
              f"torch CPU oracle, {threads} threads, {cpu_model()}")
    line = {
        "metric": "rollout tokens/s", "value": value, "unit": "tokens/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "config2: qwen2.5-1.5b-shape random-init rollout, 512 prompts x 1024 "
                               "tokens per instance (CPU arm: bounded sample, see cpu_baseline)",
                   "model": "qwen2.5-1.5b-shape", "prompt_len": f"U[{P_LO},{P_HI}]"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2510_19225_b200 import multi
    from paper_2510_19225_b200.instance import RolloutInstance
    from paper_2510_19225_b200.shapes import QWEN25_1_5B
    from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        multi.init_nccl_quiet(dist, torch, local)        # stdout stays one JSON line
    shape = QWEN25_1_5B
    n_prompts, new = args.prompts, args.new_tokens
    if args.strong:                       # fixed total work: this rank's share of the prompts
        n_prompts = args.prompts // ws + (1 if rank < args.prompts % ws else 0)
    w = synth_hf_weights(shape, seed=0, device=f"cuda:{local}")
    inst = RolloutInstance(shape, local, max_slots=n_prompts, max_seq_len=MAX_SEQ,
                           max_prefill_rows=args.prefill_rows, graph_steps=16,
                           split_o=args.split_o, split_down=args.split_down)
    pull_cold = inst.load_weights(w, version=1)    # first call: lazy module load, pool growth
    pull = inst.load_weights(w, version=1)         # the local re-layout pull itself
    prompts = synth_prompts(n_prompts, shape.vocab, P_LO, P_HI, seed=1000 + rank)
    h2d_prompt_bytes = 4 * sum(len(p) for p in prompts)

    ctx_at_profile: list[float] = []

    def rollout(tag: str, profile: bool = False):
        for i, p in enumerate(prompts):
            inst.generate(f"{tag}-{i}", p, target_len=new)
        got = 0
        prof = {}
        while True:
            out = inst.step(args.flush_steps)
            got += sum(len(t) for _, t, _ in out)
            if profile and not prof and got >= n_prompts * int(new * args.profile_at):
                # the profiled re-launches are the only region an
                # `ncu --profile-from-start off` capture sees
                torch.cuda.synchronize()
                torch.cuda.profiler.start()
                for k in ("attention", "gate_up", "down", "qkv", "o_proj", "lm_head",
                          "resid_norm"):
                    prof[k] = inst.profile_kernel(k, iters=20)
                torch.cuda.profiler.stop()
                ctx_at_profile.append(h2d_prompt_bytes / 4 / n_prompts + got / n_prompts)
            st = inst.status()
            if st["m_pending"] == 0 and st["m_exec"] == 0:
                break
        return got, prof

    for i in range(args.warmup):
        rollout(f"w{i}")
    inst.stats(reset=True)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    tokens = 0
    barrier()
    with ClockSampler(local) as clocks:
        t0 = time.perf_counter()
        for i in range(args.steps):
            got, _ = rollout(f"t{i}")
            tokens += got
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    barrier()
    st = inst.stats(reset=True)
    dev_s = (st["prefill_ms"] + st["decode_ms"]) / 1000.0
    _, prof = rollout("p", profile=True)

    agg = [dev_s, wall, float(tokens), float(st["kernel_launches"]),
           float(st["h2d_bytes"] + h2d_prompt_bytes * args.steps), float(st["d2h_bytes"])]
    mx, sm = multi.reduce_max_sum(agg, device="cuda")   # max over ranks (time), sums (work)
    dev_max, wall_max = mx[0], mx[1]
    total_tokens, launches = sm[2], int(sm[3])
    h2d_step, d2h_step = agg[4] / args.steps, agg[5] / args.steps

    if rank == 0:
        import json as _j
        peaks = {}
        try:
            peaks = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except OSError:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        nc = None
        try:
            nc = _j.load(open(os.path.join(ROOT, NCU_ATTN_FILE)))
        except (OSError, ValueError):
            pass
        att_ms, att_bytes = prof["attention"]
        traffic = traffic_src = None
        if nc:
            # the committed ncu --set full capture of this very launch (same
            # config, same profile point -> same context and algorithmic bytes)
            same = abs(nc["algorithmic_bytes"] - att_bytes) <= 1e-6 * att_bytes
            ratio = nc["dram_bytes"] / nc["algorithmic_bytes"]
            traffic = round(nc["dram_bytes"] if same else att_bytes * ratio)
            traffic_src = (f"{NCU_ATTN_FILE}: dram__bytes_read+write of the profiled launch "
                           f"(context {nc.get('context')}, {nc['duration_us']} us under ncu)"
                           + ("" if same else f", scaled by its ratio {ratio:.3f} to this launch"))
        achieved = att_bytes / (att_ms / 1e3) / 1e9
        kern = {k: {"avg_ms": round(v[0], 4), "work": v[1],
                    ("GB/s" if k in HBM_KERNELS else "TFLOP/s"):
                        round(v[1] / (v[0] / 1e3) / (1e9 if k in HBM_KERNELS else 1e12), 1)}
                for k, v in prof.items()}
        line = {
            "metric": "rollout tokens/s", "value": total_tokens / dev_max, "unit": "tokens/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * dev_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": "config2: qwen2.5-1.5b-shape random-init greedy rollout, "
                                   f"{n_prompts} prompts x {new} tokens per instance, one instance per GPU",
                       "model": "qwen2.5-1.5b-shape (random init)", "prompts_per_gpu": n_prompts,
                       "prompt_len": f"U[{P_LO},{P_HI}]", "new_tokens": new, "global_batch": n_prompts * ws,
                       "parallelism": f"independent instances x{ws}",
                       "l2": "inputs larger than L2 (3.09 GB weights + up to 20 GB KV per step)"},
            "e2e": {"value": total_tokens / wall_max, "unit": "tokens/s",
                    "h2d_bytes_per_step": int(h2d_step), "d2h_bytes_per_step": int(d2h_step)},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": "attn_mma_kernel<128> (K1, paged GQA decode attention)",
                         "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic, "traffic_source": traffic_src,
                         "bytes_per_launch": att_bytes, "avg_launch_ms": att_ms,
                         "context": round(ctx_at_profile[0], 1) if ctx_at_profile else None,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
            "kernels_mid_rollout": kern,
            "phases_ms_rank0": {"prefill": round(st["prefill_ms"], 1), "decode": round(st["decode_ms"], 1),
                                "prefill_rows": st["prefill_rows"], "decode_steps": st["decode_steps"]},
            "weight_load_local": {"bytes": pull.bytes, "seconds": pull.seconds, "GB/s": round(pull.gbps, 1),
                                  "cold_seconds": pull_cold.seconds,
                                  "note": "HBM->HBM re-layout copy: bytes read + written = 2 x bytes"},
            "clocks": clocks.summary(),
        }
        if ws == 1 and not args.no_cpu_baseline:
            del w
            line["cpu_baseline"] = cpu_baseline(shape, threads=os.cpu_count() or 1)
        print(json.dumps(line), flush=True)
    inst.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
