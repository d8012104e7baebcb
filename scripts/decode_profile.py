"""Measured batch-size -> decode-throughput curve of one B200 instance (config
2 shape) and the plateau the reference's rule picks from it.

    python scripts/decode_profile.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_19225_b200.instance import RolloutInstance
from paper_2510_19225_b200.profile import measured_profile_table
from spotrl.balancer import estimate_plateau
from paper_2510_19225_b200.shapes import SHAPES
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts

BATCHES = [1, 2, 4, 8, 16, 32, 64, 128, 192, 256, 384, 512]
NEW = 96


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?")
    ap.add_argument("--shape", default="qwen2.5-1.5b")
    ap.add_argument("--batches", default=",".join(map(str, BATCHES)))
    args = ap.parse_args()
    out = args.out
    shape = SHAPES[args.shape]
    w = synth_hf_weights(shape, seed=0, device="cuda:0")
    inst = RolloutInstance(shape, 0, max_slots=512, max_seq_len=512, graph_steps=16)
    inst.load_weights(w, version=1)
    points = []
    for b in map(int, args.batches.split(",")):
        prompts = synth_prompts(b, shape.vocab, 128, 384, seed=b)
        for rep in range(2):      # first pass captures the graphs
            inst.decode_profile(reset=True)
            for i, p in enumerate(prompts):
                inst.generate(f"b{b}-{rep}-{i}", p, target_len=NEW)
            inst.run_to_completion(64)
        pts = [pt for pt in inst.decode_profile(reset=True) if pt[0] == b]
        points += pts
        s, sec = sum(p[1] for p in pts), sum(p[2] for p in pts)
        print(f"b={b:4d} steps={s:4d} {1e3 * sec / s:7.3f} ms/step {b * s / sec:10.0f} tok/s",
              flush=True)
    t = measured_profile_table(points)
    res = {"shape": shape.name, "new_tokens": NEW, "prompt_len": "U[128,384]",
           "context_calibration": t.context_calibration,
           "entries": [{"batch_size": e.batch_size, "decode_tokens_per_s": e.decode_throughput}
                       for e in t.entries],
           "plateau": {str(eps): estimate_plateau(t, t.context_calibration, epsilon=eps)
                       for eps in (0.01, 0.05, 0.1)}}
    print(json.dumps(res["plateau"]))
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
