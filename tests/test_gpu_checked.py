"""The GPU parity and migration tests again on librlb_checked.so: every page
id, slot, position and sequence length the kernels take from device tables
is bounds-checked on the device (RLB_CHECKED; a failed check traps).  This
pool does not allow compute-sanitizer, so the checked build is the
out-of-bounds evidence for the kernels."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2510_19225_b200", "librlb_checked.so")


def test_engine_suite_on_checked_build():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(CHECKED):
        pytest.skip("librlb_checked.so not built (make checked)")
    env = dict(os.environ, RLB_LIB=CHECKED)
    sel = ["tests/test_gpu_engine.py", "tests/test_gpu_edges.py", "tests/test_gpu_fuzz_migrate.py",
           "tests/test_gpu_kernels.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *sel],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    print(tail)
    assert r.returncode == 0, tail
    assert "RLB device check failed" not in r.stdout + r.stderr
