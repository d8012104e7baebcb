"""Mid-rollout kernel timings of the config-2 decode step plus the CTA-0
latency breakdown of each projection (RLB_GEMM_DBG)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RLB_GEMM_DBG"] = "1"
from paper_2510_19225_b200.instance import RolloutInstance
from paper_2510_19225_b200.shapes import QWEN25_1_5B
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts
w = synth_hf_weights(QWEN25_1_5B, seed=0, device="cuda:0")
inst = RolloutInstance(QWEN25_1_5B, 0, max_slots=512, max_seq_len=1408, graph_steps=16)
inst.load_weights(w, version=1)
for i, p in enumerate(synth_prompts(512, QWEN25_1_5B.vocab, 128, 384, seed=3)):
    inst.generate(f"r{i}", p, target_len=600)
for _ in range(10):
    inst.step(32)
for k in ("qkv", "o_proj", "gate_up", "down", "lm_head", "attention", "resid_norm"):
    ms, work = inst.profile_kernel(k, iters=20)
    print(f"{k:10s} {ms * 1e3:7.2f} us", flush=True)
