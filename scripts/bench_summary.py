"""One-line summary of a bench.py JSON line on stdin (tuning runs)."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
ph = d["phases_ms_rank0"]
k = {n: round(v["avg_ms"] * 1e3, 1) for n, v in d["kernels_mid_rollout"].items()}
print(tag, round(d["value"]), "decode ms/step", round(ph["decode"] / ph["decode_steps"], 3),
      "prefill ms", ph["prefill"], k)
