"""Token dump for A/B bit-identity checks of a kernel change.

    RLB_LIB=paper_2510_19225_b200/librlb_prev.so python scripts/ab_tokens.py prev
    python scripts/ab_tokens.py new && python scripts/ab_tokens.py --compare prev new

Runs config-2 shapes (Qwen2.5-1.5B, 128 prompts x 96 tokens, varlen prefill
and batched decode) plus a mid-generation resume of every 4th request, and
writes all generated ids to gpurun_out/ab_<tag>.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


def run(tag):
    from paper_2510_19225_b200.instance import RolloutInstance
    from paper_2510_19225_b200.shapes import QWEN25_1_5B
    from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts
    w = synth_hf_weights(QWEN25_1_5B, seed=0, device="cuda:0")
    inst = RolloutInstance(QWEN25_1_5B, 0, max_slots=128, max_seq_len=512, graph_steps=16)
    inst.load_weights(w, version=1)
    prompts = synth_prompts(128, QWEN25_1_5B.vocab, 100, 300, seed=7)
    for i, p in enumerate(prompts):
        inst.generate(f"r{i}", p, target_len=96)
    got = inst.run_to_completion()
    # resume: prompt + first 40 generated ids as prefix, continue to 96
    for i in range(0, 128, 4):
        inst.generate(f"m{i}", prompts[i], got[f"r{i}"][:40], target_len=96)
    got.update(inst.run_to_completion())
    os.makedirs(OUT, exist_ok=True)
    np.savez(os.path.join(OUT, f"ab_{tag}.npz"), **{k: np.asarray(v, np.int32) for k, v in got.items()})
    resumed = sum(got[f"m{i}"] == got[f"r{i}"][40:] for i in range(0, 128, 4))
    print(f"{tag}: {len(got)} sequences, resume bit-exact {resumed}/32")


def compare(a, b):
    A = np.load(os.path.join(OUT, f"ab_{a}.npz"))
    B = np.load(os.path.join(OUT, f"ab_{b}.npz"))
    diff = [k for k in A.files if not np.array_equal(A[k], B[k])]
    print(f"{a} vs {b}: {len(A.files)} sequences, {len(diff)} differ {diff[:8]}")
    return 0 if not diff else 1


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        sys.exit(compare(sys.argv[2], sys.argv[3]))
    run(sys.argv[1])
