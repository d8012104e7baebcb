"""Response buffer and instance records of the rollout path.

Mirrors the reference value types the path touches
(`pkg/src/spotrl/domain.py:13-90`): `RequestState`, `InstanceStatus`,
`RouteLeg`, `RolloutRequest` (append-only `generated`, per-leg token counts,
`context_len`), `InstanceRecord` (monotone weight version).  Same names, same
fields, same errors.  One addition for the B200 path: a request can carry its
real `prompt_tokens`, because a migrated request is resumed from prompt +
generated ids (the reference stores only `prompt_len` and fabricates ids,
`pkg/src/spotrl/manager.py:307-308`).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field


class RequestState(enum.Enum):
    UNROUTED = "unrouted"
    PENDING = "pending"
    EXECUTING = "executing"
    COMPLETE = "complete"
    MIGRATING = "migrating"


class InstanceStatus(enum.Enum):
    PROVISIONING = "provisioning"
    PULLING_WEIGHTS = "pulling_weights"
    ACTIVE = "active"
    PREEMPTED = "preempted"


@dataclass
class RouteLeg:
    """One hop of a request's routing history and the tokens produced there."""

    instance_id: str
    tokens: int = 0


@dataclass
class RolloutRequest:
    """One prompt's generation job; `generated` only grows, and its length is
    always the sum of `route_history` leg counts."""

    request_id: str
    prompt_len: int
    target_len: int
    group_id: str
    generated: list[int] = field(default_factory=list)
    state: RequestState = RequestState.UNROUTED
    migrating_from: str | None = None
    route_history: list[RouteLeg] = field(default_factory=list)
    prompt_tokens: list[int] | None = None

    def append_tokens(self, instance_id: str, tokens: list[int]) -> None:
        legs = self.route_history
        if not legs or legs[-1].instance_id != instance_id:
            raise ValueError(
                f"{self.request_id}: token stream from {instance_id} does not match "
                f"current route leg"
            )
        self.generated.extend(tokens)
        legs[-1].tokens += len(tokens)

    @property
    def context_len(self) -> int:
        return self.prompt_len + len(self.generated)

    def routed_tokens(self) -> int:
        return sum(leg.tokens for leg in self.route_history)

    @property
    def remaining(self) -> int:
        return self.target_len - len(self.generated)


@dataclass
class InstanceRecord:
    """Liveness, weight version and queue depths of one rollout instance."""

    instance_id: str
    gpu_count: int
    status: InstanceStatus = InstanceStatus.PROVISIONING
    weight_version: int = 0
    m_pending: int = 0
    m_exec: int = 0
    cumulative_busy_time: float = 0.0
    joined_at: float = 0.0
    preempted_at: float | None = None

    def set_weight_version(self, version: int) -> None:
        if version < self.weight_version:
            raise ValueError(
                f"{self.instance_id}: weight version {version} < {self.weight_version}"
            )
        self.weight_version = version


@dataclass(frozen=True)
class ProfileEntry:
    """One point of the batch-size -> decode-throughput curve
    (`pkg/src/spotrl/domain.py:130-133`); tokens/sec of the whole instance."""

    batch_size: int
    decode_throughput: float


@dataclass
class ProfileTable:
    """Online decode profile (`pkg/src/spotrl/domain.py:136-148`).  On B200 it
    is built from measured device time per batch size
    (`RolloutInstance.decode_profile`, `profile.measured_profile_table`);
    `context_calibration` is the mean context length the points were taken at."""

    entries: list[ProfileEntry] = field(default_factory=list)
    context_calibration: float = 0.0

    def distinct_batch_sizes(self) -> int:
        return len({e.batch_size for e in self.entries})
