"""GEMM microbenchmark sweep (tile width / split-K / M) on one B200 via rlb_bench_gemm."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19225_b200 import _lib  # noqa: E402

CASES = [  # name, M, N, K, epilogue, block_n, splits
    ("tiny-k64", 512, 128, 64, 3, 128, 1),
    ("qkv", 512, 2048, 1536, 5, 128, 1), ("qkv s2", 512, 2048, 1536, 5, 128, 2),
    ("qkv s4", 512, 2048, 1536, 5, 128, 4),
    ("o s1", 512, 1536, 1536, 5, 128, 1), ("o s4", 512, 1536, 1536, 5, 128, 4),
    ("o s6", 512, 1536, 1536, 5, 128, 6),
    ("gate_up", 512, 17920, 1536, 2, 256, 1), ("gate_up bn128", 512, 17920, 1536, 2, 128, 1),
    ("down s5", 512, 1536, 8960, 5, 128, 5), ("down s4", 512, 1536, 8960, 5, 128, 4),
    ("lm_head", 512, 151936, 1536, 4, 256, 1),
    ("prefill gate_up", 1024, 17920, 1536, 2, 256, 1), ("prefill gate_up 4k", 4096, 17920, 1536, 2, 256, 1),
    ("prefill down s5", 1024, 1536, 8960, 5, 128, 5), ("prefill qkv s4", 1024, 2048, 1536, 5, 128, 4),
]


def main():
    lib = _lib.lib()
    for name, M, N, K, epi, bn, sp in CASES:
        ms = ctypes.c_double()
        _lib.check(lib.rlb_bench_gemm(0, M, N, K, epi, bn, sp, 256, 50, ctypes.byref(ms)))
        tf = 2.0 * M * N * K / (ms.value * 1e-3) / 1e12
        print(f"{name:22s} M={M:5d} N={N:6d} K={K:5d} bn={bn} s={sp}: {ms.value * 1e3:8.2f} us  {tf:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
