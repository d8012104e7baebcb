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
  cpu_baseline the fp32 CPU oracle (oracle/qwen2_fp32.py) on a bounded sample
               of the same workload, rank 0 at N=1 only
`--impl reference` times only that CPU implementation (the reference has no
decoder of its own -- SURVEY.md §0 -- so its CPU path is the oracle port).
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
CPU_SAMPLE = (4, 32)      # prompts x new tokens for the CPU oracle sample
NCU_ATTN_FILE = "profiles/r1_attn_ncu.json"
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
    ap.add_argument("--prefill-rows", type=int, default=16384, help="token rows per prefill chunk")
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


def cpu_oracle_sample(shape, weights_cpu, seed: int, threads: int) -> dict:
    """Greedy rollout of a bounded sample of the workload on the CPU oracle."""
    import torch
    from oracle.qwen2_fp32 import Qwen2Fp32
    from paper_2510_19225_b200.synth import synth_prompts
    torch.set_num_threads(threads)
    oracle = Qwen2Fp32(shape, weights_cpu)
    n, new = CPU_SAMPLE
    prompts = synth_prompts(n, shape.vocab, P_LO, P_HI, seed=seed)
    t0 = time.perf_counter()
    toks = 0
    for p in prompts:
        toks += len(oracle.generate(p, new))
    dt = time.perf_counter() - t0
    return {"value": toks / dt, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"{n} prompts (len U[{P_LO},{P_HI}]) x {new} greedy tokens, fp32 torch CPU, "
                      f"batch 1, {dt:.1f}s"}


def run_reference(args):
    """--impl reference: the CPU implementation of the path, timed on host cores."""
    import torch
    from paper_2510_19225_b200.shapes import QWEN25_1_5B
    from paper_2510_19225_b200.synth import synth_hf_weights
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    w = synth_hf_weights(QWEN25_1_5B, seed=0, device="cpu")
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(QWEN25_1_5B, w, seed=100 + i, threads=threads)
        if i >= args.warmup:
            vals.append(r)
    value = statistics.mean(v["value"] for v in vals)
    sample = vals[0]["sample"]
    line = {
        "metric": "rollout tokens/s", "value": value, "unit": "tokens/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * CPU_SAMPLE[0] * CPU_SAMPLE[1] / value,
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
                           max_prefill_rows=args.prefill_rows, graph_steps=16)
    pull = inst.load_weights(w, version=1)
    prompts = synth_prompts(n_prompts, shape.vocab, P_LO, P_HI, seed=1000 + rank)
    h2d_prompt_bytes = 4 * sum(len(p) for p in prompts)

    def rollout(tag: str, profile: bool = False):
        for i, p in enumerate(prompts):
            inst.generate(f"{tag}-{i}", p, target_len=new)
        got = 0
        prof = {}
        while True:
            out = inst.step(args.flush_steps)
            got += sum(len(t) for _, t, _ in out)
            if profile and not prof and got >= n_prompts * (new // 2):
                for k in ("attention", "gate_up", "down", "qkv", "o_proj", "lm_head",
                          "resid_norm"):
                    prof[k] = inst.profile_kernel(k, iters=20)
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
        ncu_ratio = None
        try:
            nc = _j.load(open(os.path.join(ROOT, NCU_ATTN_FILE)))
            ncu_ratio = nc["dram_bytes"] / nc["algorithmic_bytes"]
        except (OSError, KeyError, ValueError):
            pass
        att_ms, att_bytes = prof["attention"]
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
                         "traffic": (round(att_bytes * ncu_ratio) if ncu_ratio else None),
                         "traffic_source": (f"ncu --set full DRAM read+write / algorithmic bytes = "
                                            f"{ncu_ratio:.3f} on the captured launch ({NCU_ATTN_FILE}), "
                                            "scaled to this launch" if ncu_ratio else None),
                         "bytes_per_launch": att_bytes, "avg_launch_ms": att_ms,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
            "kernels_mid_rollout": kern,
            "phases_ms_rank0": {"prefill": round(st["prefill_ms"], 1), "decode": round(st["decode_ms"], 1),
                                "prefill_rows": st["prefill_rows"], "decode_steps": st["decode_steps"]},
            "weight_load_local": {"bytes": pull.bytes, "seconds": pull.seconds, "GB/s": round(pull.gbps, 1)},
            "clocks": clocks.summary(),
        }
        if ws == 1 and not args.no_cpu_baseline:
            del w
            wc = synth_hf_weights(shape, seed=0, device="cpu")
            line["cpu_baseline"] = cpu_oracle_sample(shape, wc, seed=77, threads=os.cpu_count() or 1)
        print(json.dumps(line), flush=True)
    inst.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
