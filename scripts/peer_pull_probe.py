"""Single-process probes for ncu: the fused re-layout pull reading trainer
weights on GPU 1 over NVLink into an instance arena on GPU 0 (K7), and the
migration compaction kernel (K5) on a config-2-sized export."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_19225_b200 import _lib
from paper_2510_19225_b200.instance import RolloutInstance
from paper_2510_19225_b200.pull import TrainerWeights
from paper_2510_19225_b200.shapes import QWEN25_1_5B, QWEN25_7B
from paper_2510_19225_b200.synth import synth_hf_weights, synth_prompts

shape = QWEN25_7B if "--7b" in sys.argv else QWEN25_1_5B
if torch.cuda.device_count() > 1:
    w = synth_hf_weights(shape, seed=0, device="cuda:1")
    tw = TrainerWeights(shape, 1, w)
    del w
    _lib.check(_lib.lib().rlb_enable_peer(0, 1))
    inst = RolloutInstance(shape, 0, max_slots=8, max_seq_len=256)
    for i in range(3):
        r = inst.load_weights(tw, version=i + 1)
        print(f"peer pull {shape.name}: {r.bytes / 1e9:.2f} GB in {r.seconds * 1e3:.2f} ms = "
              f"{r.bytes / r.seconds / 1e9:.1f} GB/s", flush=True)
    inst.close()
# K5: export 512 partial responses mid-rollout
shape = QWEN25_1_5B
w = synth_hf_weights(shape, seed=0, device="cuda:0")
inst = RolloutInstance(shape, 0, max_slots=512, max_seq_len=1408, graph_steps=16)
inst.load_weights(w, version=1)
for i, p in enumerate(synth_prompts(512, shape.vocab, 128, 384, seed=5)):
    inst.generate(f"r{i}", p, target_len=1024)
for _ in range(8):
    inst.step(64)
ids = [f"r{i}" for i in range(512)]
for rep in range(3):
    t0 = time.perf_counter()
    ex = inst.export_partials(ids)
    dt = time.perf_counter() - t0
    print(f"export_partials #{rep}: {len(ex)} requests, {sum(len(a) + len(b) for a, b in ex)} ids, "
          f"{dt * 1e3:.2f} ms wall", flush=True)
