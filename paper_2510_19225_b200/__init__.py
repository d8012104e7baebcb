"""B200-native rollout data path of RLBoost behind the reference's own API.

The control plane is the UNMODIFIED reference package `spotrl`
(`/root/reference/pkg/src/spotrl`): `RolloutManager`, `TransferPool`, the
domain types, the balancer decisions and the wire protocol are imported, not
restated.  This package adds only what the B200 path needs beside them (the
C-ABI instance, the real-id response buffer, the NVLink weight plane, the
runner that drives instances under the reference manager).

`spotrl` is resolved from `sys.path` first, then from `<repo>/baseline/_ref`
(where `__graft_entry__.build()` installs the reference from its own sources;
that directory travels to GPU boxes with the repo snapshot), then -- in the
builder container only -- from the reference source tree itself.  Without
the reference package the product refuses to import.
"""
from __future__ import annotations

import os
import sys


def _ensure_spotrl() -> None:
    try:
        import spotrl  # noqa: F401
        return
    except ImportError:
        pass
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # the installed copy first; in the builder container the reference's own
    # source tree (read-only) if build() has not installed it yet
    for ref in (os.path.join(root, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(ref, "spotrl")) and ref not in sys.path:
            sys.path.append(ref)
            break
    try:
        import spotrl  # noqa: F401,F811
    except ImportError as exc:
        raise ImportError(
            "the reference control plane `spotrl` is not importable; run "
            "`python __graft_entry__.py` (build() installs it into baseline/_ref) or "
            "`pip install --target baseline/_ref <copy of /root/reference/pkg>`") from exc


_ensure_spotrl()
