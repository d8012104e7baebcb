"""Multi-GPU plumbing: one process per GPU under torchrun.

Rollout instances are independent (no data-path collective; weak scaling,
`PAPER.md:28,56`): ranks only agree on timings (max over ranks, sums of
tokens) and exchange small control objects (CUDA-IPC handles, the NCCL unique
id of the weight fan-out).  These helpers are backend-agnostic so the same
code runs over NCCL on B200 and over gloo in the CPU tests.
"""
from __future__ import annotations

import os


def dist_env() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def reduce_max_sum(values: list[float], device=None) -> tuple[list[float], list[float]]:
    """Element-wise (max over ranks, sum over ranks) of a small float vector."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t.tolist(), t.tolist()
    mx, sm = t.clone(), t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return mx.tolist(), sm.tolist()


def gather_objects(obj) -> list:
    """Every rank's `obj`, in rank order (single process: [obj])."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def broadcast_object(obj, src: int = 0):
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return obj
    box = [obj]
    dist.broadcast_object_list(box, src=src)
    return box[0]


def weak_scaling_value(tokens_per_rank: list[float], seconds_per_rank: list[float]) -> float:
    """Whole-job throughput: tokens of all ranks / slowest rank's time."""
    return sum(tokens_per_rank) / max(seconds_per_rank)


def init_nccl_quiet(dist, torch, local_rank: int) -> None:
    """init_process_group("nccl") + one barrier with the process's stdout
    pointed at stderr, so NCCL's own start-up lines (printed with C stdio,
    e.g. "NCCL version ...") never reach the bench's one-JSON-line stdout."""
    import os
    import sys
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist.barrier()
        torch.cuda.synchronize()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
