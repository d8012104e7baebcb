"""Real token ids in the reference response buffer.

The reference's `RolloutManager` (`pkg/src/spotrl/manager.py`) is used
unmodified.  Its token collection carries counts only: `on_tokens(request_id,
instance_id, count, now)` (`manager.py:295-314`) checks ownership, gating and
overshoot, then appends placeholder ids `range(start, start + count)`
(`manager.py:307-308`), because the simulator has no model; `create_request`
(`manager.py:170-189`) stores `prompt_len`, not the prompt.

The B200 path produces real ids, and a migrated request must be resumed from
prompt + generated ids (`protocol.py:75-81`).  `ResponseBuffer` sits beside
the manager:

  * prompt ids live in a table keyed by `request_id` (the reference
    `RolloutRequest` has no field for them, `domain.py:36-49`);
  * a flush of an instance goes through the reference `on_tokens` with its
    count first -- every check and the `tokens` event are the reference's --
    and only after it accepted the tokens are the placeholder ids it appended
    overwritten in place with the ids the GPU produced.  So the reference's
    own `RolloutRequest.generated`, route legs, microbatches
    (`seal_microbatch`) and migration prefixes (`migrate_out` keeps the
    list, recompute clears it, `manager.py:336-357`) all carry real ids.

`dispatch` routes held requests with the reference's `select_instance`
(`balancer.py:80-92`) and `route_to` (`manager.py:258-259`).  It is the
reference `dispatch` loop (`manager.py:208-222`) with one change: the
snapshot `select_instance` sees is each serving instance's pending-queue
depth (taken once, bumped as requests are routed), because JSQ reads
`m_pending` alone -- the reference rebuilds every serving instance's
pending and executing lists for each routed request, O(routed x executing),
which costs ~1 s when 1,024 requests are re-routed onto survivors running
3,072 (config 3).  Routing decisions and `route` events are identical
(`tests/test_responses.py::test_dispatch_matches_reference`).
"""
from __future__ import annotations

from typing import Iterable

from spotrl.balancer import MUST_WAIT, select_instance
from spotrl.manager import ManagerError, RolloutManager


class ResponseBuffer:
    """Prompt ids + real generated ids for the requests of one manager."""

    def __init__(self, manager: RolloutManager):
        self.manager = manager
        self.prompts: dict[str, list[int]] = {}

    # -- requests ---------------------------------------------------------------

    def create_request(self, request_id: str, prompt_tokens: list[int], target_len: int,
                       group_id: str, now: float):
        """`manager.create_request` + the prompt ids for later (re)submission."""
        req = self.manager.create_request(request_id, len(prompt_tokens), target_len,
                                          group_id, now)
        self.prompts[request_id] = [int(t) for t in prompt_tokens]
        return req

    def prompt(self, request_id: str) -> list[int]:
        return self.prompts[request_id]

    def prefix(self, request_id: str) -> list[int]:
        """Ids kept so far (the resume prefix): the reference request's list."""
        return list(self.manager.requests[request_id].generated)

    # -- token collection ---------------------------------------------------------

    def on_tokens(self, request_id: str, instance_id: str, ids, now: float) -> None:
        """Reference `on_tokens(count=len(ids))`, then the real ids in place of
        its placeholders.  If the reference raises (stream desync, gating
        violation, overshoot), nothing of this flush is kept."""
        ids = [int(t) for t in ids]
        if not ids:
            return
        gen = self.manager.requests[request_id].generated
        start = len(gen)
        self.manager.on_tokens(request_id, instance_id, len(ids), now)
        if len(gen) != start + len(ids):
            raise ManagerError(f"{request_id}: response buffer out of step with the manager")
        gen[start:] = ids

    def on_flush(self, instance_id: str, batch: Iterable, now: float) -> int:
        """One flush of an instance: (request_id, ids, done) per request with
        news.  Tokens first, then `complete` for requests that reached their
        target.  Returns the token count."""
        n = 0
        for request_id, ids, done in batch:
            if len(ids):
                self.on_tokens(request_id, instance_id, ids, now)
                n += len(ids)
            if done:
                self.manager.complete(request_id, instance_id, now)
        return n


class _QueueDepth:
    """What `select_instance` reads of an `InstanceLoad`: id and pending depth."""

    __slots__ = ("instance_id", "m_pending")

    def __init__(self, instance_id: str, m_pending: int):
        self.instance_id = instance_id
        self.m_pending = m_pending


def dispatch(manager: RolloutManager, now: float) -> list[tuple[str, str]]:
    """Route held requests while some serving instance is below theta (the
    reference `dispatch` decision over pending-queue depths; see module doc).
    Routing does not change which instances serve, so the serving set is
    taken once and the chosen instance's depth is bumped in place."""
    routed: list[tuple[str, str]] = []
    if not manager.held:
        return routed
    serving = manager.serving_ids()
    if not serving:
        return routed
    loads = [_QueueDepth(i, len(manager.pending_queues[i])) for i in serving]
    by_id = {d.instance_id: d for d in loads}
    while manager.held:
        choice = select_instance(loads, manager.theta)
        if choice is MUST_WAIT:
            break
        request_id = manager.held.popleft()
        manager.route_to(request_id, choice, now)
        by_id[choice].m_pending += 1
        routed.append((request_id, choice))
    return routed
