"""Split-K projections (down / O) on single-SM tiles vs persistent 2-SM pair
tiles writing fp32 partials, via rlb_bench_gemm (zero data, CUDA events)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19225_b200 import _lib  # noqa: E402

CASES = [  # name, M, N, K, splits
    ("down", 512, 1536, 8960, 5), ("down", 512, 1536, 8960, 6), ("down", 512, 1536, 8960, 7),
    ("down", 512, 1536, 8960, 4), ("down", 384, 1536, 8960, 5),
    ("o", 512, 1536, 1536, 3), ("o", 512, 1536, 1536, 6),
    ("down prefill", 16384, 1536, 8960, 5), ("o prefill", 16384, 1536, 1536, 3),
    ("7b down", 256, 3584, 18944, 4), ("7b o", 256, 3584, 3584, 4),
]


def run(lib, M, N, K, epi, bn, sp, bm, pair):
    if pair:
        os.environ["RLB_GEMM_PAIR"] = "2"
    else:
        os.environ.pop("RLB_GEMM_PAIR", None)
    ms = ctypes.c_double()
    _lib.check(lib.rlb_bench_gemm(0, M, N, K, epi, bn, sp, bm, 50, ctypes.byref(ms)))
    return ms.value * 1e3


def main():
    lib = _lib.lib()
    for name, M, N, K, sp in CASES:
        one = run(lib, M, N, K, 5, 128, sp, 256, False)
        cl = run(lib, M, N, K, 1, 128, sp, 256, False) if sp <= 8 else float("nan")
        pr = run(lib, M, N, K, 5, 128, sp, 256, True)
        tf = lambda us: 2.0 * M * N * K / (us * 1e-6) / 1e12  # noqa: E731
        print(f"{name:13s} M={M:5d} N={N:5d} K={K:5d} s={sp}: 1-SM partials {one:7.2f} us "
              f"({tf(one):6.1f} TF/s)  1-SM cluster-resadd {cl:7.2f} us  pair partials {pr:7.2f} us "
              f"({tf(pr):6.1f} TF/s)", flush=True)


if __name__ == "__main__":
    main()
