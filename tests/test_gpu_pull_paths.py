"""Weight-pull data paths on one B200: the fan-out's range slices of the fused
re-layout, and a CUDA-IPC pull from another process (the `cuda-ipc://`
agent endpoint of `pull_weights`) -- both must land the same arena bytes as
the direct fused re-layout."""
import os
import subprocess
import sys

import pytest
import torch

from paper_2510_19225_b200.shapes import small_shape
from paper_2510_19225_b200.synth import synth_hf_weights

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_19225_b200.instance import RolloutInstance
    shape = small_shape(layers=2, vocab=8192)
    w = synth_hf_weights(shape, seed=5, device="cuda")
    inst = RolloutInstance(shape, 0, max_slots=4, max_seq_len=256)
    inst.load_weights(w, version=1)
    return shape, w, inst


def _arena_bytes(inst):
    from paper_2510_19225_b200 import _lib
    p, n = inst.arena()
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().rlb_copy_bytes(0, buf.data_ptr(), p, n, None))
    torch.cuda.synchronize()
    return buf


def test_relayout_range_slices_compose(setup):
    import ctypes
    from paper_2510_19225_b200 import _lib
    from paper_2510_19225_b200.instance import RolloutInstance
    shape, w, inst = setup
    want = _arena_bytes(inst)
    dst = RolloutInstance(shape, 0, max_slots=4, max_seq_len=256)
    p, n = dst.arena()
    ptrs = dst._source_ptrs(w)
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    cfg = _lib.ModelCfg.from_shape(shape)
    cuts = [0, 16 * 12345, 16 * 999_999, n // 2 // 16 * 16, n]
    for lo, hi in zip(cuts, cuts[1:]):
        _lib.check(_lib.lib().rlb_relayout_copy_range(0, ctypes.byref(cfg), arr, len(ptrs), p, lo, hi,
                                                      None))
    torch.cuda.synchronize()
    assert torch.equal(_arena_bytes(dst), want)


CHILD = r"""
import os, sys, hashlib
sys.path.insert(0, os.environ["ROOT"])
import torch
from paper_2510_19225_b200.instance import RolloutInstance
from paper_2510_19225_b200.pull import MappedSource
from paper_2510_19225_b200.shapes import small_shape
from paper_2510_19225_b200 import _lib
shape = small_shape(layers=2, vocab=8192)
src = MappedSource(os.environ["ENDPOINT"], 0)
inst = RolloutInstance(shape, 0, max_slots=4, max_seq_len=256)
inst.pull_weights(src, 1)
p, n = inst.arena()
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
_lib.check(_lib.lib().rlb_copy_bytes(0, buf.data_ptr(), p, n, None))
torch.cuda.synchronize()
print("SHA", hashlib.sha256(buf.cpu().numpy().tobytes()).hexdigest())
src.close()
"""


def test_cuda_ipc_pull_from_another_process(setup):
    import hashlib
    from paper_2510_19225_b200.pull import TrainerWeights
    shape, w, inst = setup
    tw = TrainerWeights(shape, 0, w)
    env = dict(os.environ, ROOT=ROOT, ENDPOINT=tw.endpoint())
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    got = [l.split()[1] for l in out.stdout.splitlines() if l.startswith("SHA ")][0]
    want = hashlib.sha256(_arena_bytes(inst).cpu().numpy().tobytes()).hexdigest()
    assert got == want
