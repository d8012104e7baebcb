"""Per-kernel device time of a small-batch decode step (the long-tail regime
of config 5): one instance, `b` live requests, then rlb_profile_kernel on the
step's row count.  Prints us per launch and GB/s of weight bytes streamed.

    python scripts/small_batch_kernels.py --shape qwen2.5-7b --batches 1,8,64
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_19225_b200.instance import RolloutInstance  # noqa: E402
from paper_2510_19225_b200.shapes import SHAPES  # noqa: E402
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="qwen2.5-7b")
    ap.add_argument("--batches", default="1,8,64")
    args = ap.parse_args()
    s = SHAPES[args.shape]
    w = synth_hf_weights(s, seed=0, device="cuda:0")
    H, F, V = s.hidden, s.ffn, s.vocab
    qkv = (s.n_q_heads + 2 * s.n_kv_heads) * s.head_dim
    wbytes = {"qkv": 2 * qkv * H, "o_proj": 2 * H * s.n_q_heads * s.head_dim,
              "gate_up": 2 * 2 * F * H, "down": 2 * H * F, "lm_head": 2 * V * H}
    for b in map(int, args.batches.split(",")):
        inst = RolloutInstance(s, 0, max_slots=max(b, 8), max_seq_len=1024, graph_steps=16)
        inst.load_weights(w, version=1)
        for i, p in enumerate(synth_prompts(b, s.vocab, 128, 384, seed=b)):
            inst.generate(f"r{i}", p, target_len=400)
        for _ in range(4):
            inst.step(16)
        tot = 0.0
        line = []
        for k in ("qkv", "attention", "o_proj", "resid_norm", "gate_up", "down", "lm_head"):
            ms, _ = inst.profile_kernel(k, iters=50)
            us = ms * 1e3
            per_layer = 2 if k == "resid_norm" else 1
            if k != "lm_head":
                tot += us * per_layer * s.layers
            else:
                tot += us
            gbs = f" {wbytes[k] / (ms * 1e-3) / 1e9:6.0f} GB/s" if k in wbytes else ""
            line.append(f"{k} {us:6.1f} us{gbs}")
        print(f"{s.name} b={b}: " + " | ".join(line) + f" || sum {tot / 1e3:.3f} ms/step", flush=True)
        inst.close()


if __name__ == "__main__":
    main()
