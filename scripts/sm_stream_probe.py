import ctypes, os, sys
sys.path.insert(0, "/root/repo")
from paper_2510_19225_b200 import _lib
lib = _lib.lib()
for K in (3584, 18944):
    for ntile in (9, 18, 36, 72, 144, 148, 296):
        for bn in (128,):
            N = ntile * bn
            ms = ctypes.c_double()
            _lib.check(lib.rlb_bench_gemm(0, 1, N, K, 0, bn, 1, 128, 30, ctypes.byref(ms)))
            us = ms.value * 1e3
            wb = N * K * 2
            print(f"K={K} ctas={ntile:4d} bn={bn}: {us:8.2f} us  total {wb/us/1e3:7.0f} GB/s  per-CTA {wb/ntile/us/1e3:6.1f} GB/s", flush=True)
