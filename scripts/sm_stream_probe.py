"""Weight streaming rate of the K2 GEMM at few rows: M=1 (a 128-row A box of
which 127 rows are out of bounds) vs M=128 (a full A box), per CTA count."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19225_b200 import _lib  # noqa: E402

lib = _lib.lib()
for K in (3584,):
    for M in (1, 128):
        for ntile in (18, 36, 72, 144, 296):
            bn = 128
            N = ntile * bn
            ms = ctypes.c_double()
            _lib.check(lib.rlb_bench_gemm(0, M, N, K, 0, bn, 1, 128, 30, ctypes.byref(ms)))
            us = ms.value * 1e3
            wb = N * K * 2
            print(f"M={M:3d} K={K} ctas={ntile:4d}: {us:8.2f} us  weights {wb/us/1e3:7.0f} GB/s  "
                  f"per-CTA {wb/ntile/us/1e3:6.1f} GB/s", flush=True)
