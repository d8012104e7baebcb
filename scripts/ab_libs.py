"""Bitwise A/B of librlb builds that must not change a row's bits: for each
library (RLB_LIB) a child process runs the same prefill-heavy rollout +
teacher-forced score on the full 1.5B shape and prints a digest of the whole
KV pool, the tokens and the logits; the digests must match.

    python scripts/ab_libs.py paper_2510_19225_b200/librlb.so paper_2510_19225_b200/librlb_x.so
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, sys
sys.path.insert(0, %r)
import torch
from paper_2510_19225_b200 import _lib
from paper_2510_19225_b200.instance import RolloutInstance
from paper_2510_19225_b200.shapes import QWEN25_1_5B as S
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts
w = synth_hf_weights(S, seed=0, device="cuda")
inst = RolloutInstance(S, 0, max_slots=64, max_seq_len=1408, max_prefill_rows=4096)
inst.load_weights(w, version=1)
prompts = synth_prompts(48, S.vocab, 128, 1100, seed=5)
logits = inst.score(prompts[0])
for i, p in enumerate(prompts):
    inst.generate(f"r{i}", p, target_len=24)
got = inst.run_to_completion(16)
p, n = inst.kv_pool()
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
_lib.check(_lib.lib().rlb_copy_bytes(0, buf.data_ptr(), p, n, None))
torch.cuda.synchronize()
h = hashlib.sha256()
for k in range(0, n, 1 << 30):
    h.update(buf[k:k + (1 << 30)].cpu().numpy().tobytes())
print(json.dumps({"kv": h.hexdigest(), "tokens": hashlib.sha256(json.dumps(got, sort_keys=True).encode()).hexdigest(),
                  "logits": hashlib.sha256(logits.tobytes()).hexdigest()}))
""" % ROOT

out = {}
for lib in sys.argv[1:]:
    env = dict(os.environ, RLB_LIB=os.path.join(ROOT, lib))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    out[lib] = json.loads(line[-1]) if line else {"error": r.stderr[-500:]}
ref = next(iter(out.values()))
print(json.dumps({"results": out, "identical": all(v == ref for v in out.values())}, indent=1))
