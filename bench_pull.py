#!/usr/bin/env python
"""Config 4: pull-based transfer of Qwen2.5-7B-shape bf16 weights
(15,231,233,024 B, 339 HF tensors) from the trainer GPU to 1/3/7 rollout GPUs
over NVLink, with the HF -> engine re-layout fused into the copy.

Launch: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1
        bench_pull.py [--mode fanout|direct|both]
Rank 0 is the trainer (holds the HF-layout weights, publishes a cuda-ipc
endpoint = the `agent_endpoint` of protocol `pull_weights`); ranks 1..N-1 are
rollout instances that pull.  Prints one JSON line (rank 0): per-receiver and
aggregate GB/s per mode (time = first issue -> the receiver's last byte,
max over receivers), NVLink fraction of 900 GB/s, and bytewise equality of
every receiver's engine arena with the trainer's reference re-layout.
With N=1 the trainer and the receiver share one GPU (HBM copy, no NVLink).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NVLINK_GBS = 900.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["fanout", "direct", "nccl", "all"], default="all")
    ap.add_argument("--shape", default="qwen2.5-7b")
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--repeats", type=int, default=3)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from paper_2510_19225_b200 import _lib
    from paper_2510_19225_b200.instance import RolloutInstance
    from paper_2510_19225_b200.pull import (FanoutReceiver, MappedSource, NcclFanout,
                                           TrainerWeights, map_arena)
    from paper_2510_19225_b200.shapes import SHAPES
    from paper_2510_19225_b200.synth import synth_hf_weights

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("gloo")
    shape = SHAPES[args.shape]
    barrier = (lambda: dist.barrier()) if ws > 1 else (lambda: None)
    lib = _lib.lib()
    cfg = _lib.ModelCfg.from_shape(shape)

    # -- trainer: weights + reference re-layout -------------------------------
    objs = [None, None]
    trainer = None
    if rank == 0:
        w = synth_hf_weights(shape, seed=0, device=f"cuda:{local}")
        trainer = TrainerWeights(shape, local, w)
        del w
        expect = torch.empty(lib.rlb_arena_bytes(ctypes.byref(cfg)), dtype=torch.uint8,
                             device=f"cuda:{local}")
        arr = (ctypes.c_void_p * len(trainer.ptrs))(*trainer.ptrs)
        _lib.check(lib.rlb_relayout_copy(local, ctypes.byref(cfg), arr, len(trainer.ptrs),
                                         expect.data_ptr(), None))
        torch.cuda.synchronize()
        from paper_2510_19225_b200.pull import _ipc_handle
        objs = [trainer.endpoint(), _ipc_handle(expect.data_ptr())]
    if ws > 1:
        dist.broadcast_object_list(objs, src=0)
    endpoint, expect_handle = objs

    receivers = list(range(1, ws)) if ws > 1 else [0]
    is_recv = rank in receivers
    inst = src = None
    if is_recv:
        inst = RolloutInstance(shape, local, max_slots=1, max_seq_len=64, max_prefill_rows=128,
                               graph_steps=0)
        src = MappedSource(endpoint, local) if ws > 1 else None
        src_ptrs = src.ptrs if src else trainer.ptrs
    def exchange(mine):
        every = [None] * ws
        if ws > 1:
            dist.all_gather_object(every, mine)
        else:
            every = [mine]
        return [every[r] for r in receivers]

    me = receivers.index(rank) if is_recv else -1
    fan = None
    if is_recv:
        fan = FanoutReceiver(inst, me, len(receivers), args.rounds, exchange, barrier)
    else:
        exchange(None)

    results = {}
    version_ctr = [0]
    modes = ["fanout", "nccl", "direct"] if args.mode == "all" else [args.mode]
    ncf = None
    stage_s = stage_cold = None
    if ws > 1:
        def share_id(uid):
            box = [uid]
            dist.broadcast_object_list(box, src=0)
            return box[0]
        ncf = NcclFanout(local, ws, rank, share_id)
        if rank == 0:
            # the first staging pays the copy kernel's lazy module load and the
            # stream-ordered pool's first growth; the version's staging is the
            # warm one (r1 reported the cold 74 ms)
            stage_cold = ncf.stage(trainer)
            stage_s = ncf.stage(trainer)
    for mode in modes:
        times = []
        for rep in range(args.repeats + 1):     # first repetition warms up
            dt = 0.0
            if mode == "nccl" and ws > 1:
                # trainer staged the engine layout once; one NCCL broadcast lands
                # it in every receiver's arena
                barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if is_recv:
                    version_ctr[0] += 1
                    ncf.broadcast(inst, version_ctr[0])
                else:
                    ncf.broadcast(None)
                dt = time.perf_counter() - t0 if is_recv else 0.0
                barrier()
            elif is_recv and mode == "fanout":
                version_ctr[0] += 1
                dt = fan.pull(src_ptrs, version=version_ctr[0])
            elif is_recv:
                barrier()
                t0 = time.perf_counter()
                version_ctr[0] += 1
                inst.load_weights(src_ptrs, version=version_ctr[0])
                dt = time.perf_counter() - t0
                barrier()
            elif mode != "nccl":   # the trainer only serves memory; match the receivers' barriers
                for _ in range(3 if mode == "fanout" else 2):
                    barrier()
            t = torch.tensor([dt], dtype=torch.float64)
            if ws > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rep > 0:
                times.append(float(t[0]))
        nbytes = lib.rlb_arena_bytes(ctypes.byref(cfg))
        # the median repetition (each repetition: max over receivers); best and
        # worst alongside
        med = sorted(times)[len(times) // 2]
        results[mode] = {"seconds_max_over_receivers": med, "all_seconds": times,
                         "per_receiver_GBps": nbytes / med / 1e9,
                         "per_receiver_GBps_best": nbytes / min(times) / 1e9,
                         "per_receiver_GBps_worst": nbytes / max(times) / 1e9,
                         "aggregate_GBps": len(receivers) * nbytes / med / 1e9,
                         "nvlink_frac": (nbytes / med / 1e9) / NVLINK_GBS}
    # -- bytewise check ---------------------------------------------------------
    ok = torch.tensor([1], dtype=torch.int64)
    if is_recv:
        inst.mark_weights(version_ctr[0])
        aptr, nbytes = inst.arena()
        mine = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
        ref = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
        _lib.check(lib.rlb_copy_bytes(local, mine.data_ptr(), aptr, nbytes, None))
        if ws > 1:
            eptr, close = map_arena(expect_handle, local)
            _lib.check(lib.rlb_copy_bytes(local, ref.data_ptr(), eptr, nbytes, None))
            torch.cuda.synchronize()
            close()
        else:
            torch.cuda.synchronize()
            ref.copy_(expect)
        ok[0] = int(torch.equal(mine, ref))
    if ws > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"metric": "weight-pull GB/s", "config": "config4: qwen2.5-7b-shape bf16 "
                          f"({lib.rlb_arena_bytes(ctypes.byref(cfg))} B engine arena, 339 HF tensors), "
                          f"trainer GPU -> {len(receivers)} rollout GPU(s)",
                          "n_gpus": ws, "receivers": len(receivers),
                          "link": "NVLink5/NVSwitch" if ws > 1 else "local HBM (single GPU)",
                          "bytewise_equal": bool(ok[0]), "modes": results,
                          "nccl_stage_seconds": stage_s,
                          "nccl_stage_seconds_cold": stage_cold}), flush=True)
    if fan:
        fan.close()
    if src:
        src.close()
    barrier()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
