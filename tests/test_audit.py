"""The control-plane oracle (oracle/audit.py) pinned against the reference
simulator's own logs and the counts its oracles derived from them
(tests/golden/ref_sim_*.jsonl.gz, made by scripts/make_golden.py)."""
import copy
import gzip
import json
import os

import pytest

from oracle.audit import (restated_assert_token_conservation as assert_token_conservation,
                          restated_assert_version_gating as assert_version_gating,
                          restated_audit_requests as audit_requests)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(policy):
    with gzip.open(os.path.join(GOLD, f"ref_sim_{policy}.jsonl.gz"), "rt") as f:
        facts = json.loads(f.readline())["facts"]
        return facts, [json.loads(line) for line in f]


@pytest.mark.parametrize("policy", ["migrate", "recompute"])
def test_restatement_reproduces_reference_counts(policy):
    facts, recs = load(policy)
    assert assert_token_conservation(recs) == facts["requests"]
    assert assert_version_gating(recs) == facts["gated_token_events"]
    assert len([r for r in recs if r["type"] == "preempt"]) == facts["preemptions"]


def test_detects_corruptions():
    _, recs = load("migrate")
    tok = next(i for i, r in enumerate(recs) if r["type"] == "tokens")
    bad = copy.deepcopy(recs)
    bad[tok]["count"] += 1
    with pytest.raises(AssertionError):
        assert_token_conservation(bad)
    bad = copy.deepcopy(recs)
    bad[tok]["instance_id"] = "nobody"
    with pytest.raises(AssertionError):
        audit_requests(bad)
    remote = next(i for i, r in enumerate(recs)
                  if r["type"] == "tokens" and not r["instance_id"].startswith("local"))
    bad = copy.deepcopy(recs)
    bad[remote]["version"] = -1
    with pytest.raises(AssertionError):
        assert_version_gating(bad)
    comp = next(i for i, r in enumerate(recs) if r["type"] == "complete")
    bad = recs[:comp] + recs[comp + 1:]
    with pytest.raises(AssertionError):
        assert_token_conservation(bad)


def test_restatement_agrees_with_reference_oracles():
    from oracle import audit
    ref = audit.reference_oracles()
    if ref is None:
        pytest.skip("reference oracles not installed (run __graft_entry__.build())")
    assert audit.SOURCE == "reference" and audit.assert_token_conservation is ref.assert_token_conservation
    for policy in ("migrate", "recompute"):
        _, recs = load(policy)
        assert ref.assert_token_conservation(recs) == audit.restated_assert_token_conservation(recs)
        assert ref.assert_version_gating(recs) == audit.restated_assert_version_gating(recs)
