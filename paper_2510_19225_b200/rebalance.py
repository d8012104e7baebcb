"""Continuous rebalancer decisions fed by the measured B200 decode profile.

Restates the reference's `lb_tick` (`pkg/src/spotrl/balancer.py:129-185`) and
its order type (`MigrationKind`, `MigrationOrder`, `balancer.py:38-78`) so the
B200 runner can apply them to real instances (config 5): the
pending branch moves one queued request from the most backlogged instance to
an instance whose queue is empty; once every queue is drained, the executing
branch moves the requests above the batching plateau (cheapest prefixes
first) from the busiest instance to an idle one.  The plateau comes from
`profile.estimate_plateau` on a `ProfileTable` built from measured device
time (`RolloutInstance.decode_profile`).  Pure decisions over a snapshot;
`RolloutRunner.rebalance` applies them.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Callable, Sequence

from .domain import ProfileTable
from .manager import InstanceLoad
from .profile import ProfileNotReadyError, estimate_plateau


class MigrationKind(enum.Enum):
    PENDING = "pending"
    EXECUTING = "executing"


@dataclass(frozen=True)
class MigrationOrder:
    request_ids: tuple[str, ...]
    from_instance: str
    to_instance: str
    kind: MigrationKind

    def __post_init__(self) -> None:
        if not self.request_ids:
            raise ValueError("empty migration order")
        if self.from_instance == self.to_instance:
            raise ValueError(f"self-migration on {self.from_instance}")


def lb_tick(registry: Sequence[InstanceLoad], profile: ProfileTable, current_mean_context: float,
            *, epsilon: float = 0.05,
            context_factor: Callable[[float], float] | None = None) -> list[MigrationOrder]:
    """One rebalancer pass: at most one order.

    1. Some queue empty while another is backlogged: move the backlogged
       instance's oldest pending request (most pending first, lowest id on
       ties) to the lowest-id instance with an empty queue.
    2. Otherwise, if some instance executes nothing: take the instance with
       the most executing requests (lowest id on ties) and move its requests
       beyond the plateau -- fewest generated tokens first, then request id --
       to the lowest-id idle instance.  Skipped while the profile is not ready.
    """
    if not registry:
        return []
    empty_q = sorted((ld for ld in registry if ld.m_pending == 0), key=lambda ld: ld.instance_id)
    backlog = [ld for ld in registry if ld.m_pending > 0]
    if empty_q and backlog:
        src = min(backlog, key=lambda ld: (-ld.m_pending, ld.instance_id))
        return [MigrationOrder((src.pending[0],), src.instance_id, empty_q[0].instance_id,
                               MigrationKind.PENDING)]
    idle = sorted((ld for ld in registry if ld.m_exec == 0), key=lambda ld: ld.instance_id)
    if not idle:
        return []
    src = min(registry, key=lambda ld: (-ld.m_exec, ld.instance_id))
    if src.m_exec == 0:
        return []
    try:
        plateau = estimate_plateau(profile, current_mean_context, epsilon=epsilon,
                                   context_factor=context_factor)
    except ProfileNotReadyError:
        return []
    surplus = src.m_exec - plateau
    if surplus <= 0:
        return []
    movers = sorted(src.executing, key=lambda item: (item[1], item[0]))[:surplus]
    return [MigrationOrder(tuple(rid for rid, _ in movers), src.instance_id, idle[0].instance_id,
                           MigrationKind.EXECUTING)]
