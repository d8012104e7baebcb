"""Small-M behaviour of the decode GEMMs: time per shape and tile width at
M = 1..512, and whether the UMMA N (block_n) or tile height changes a row's
bits (it must not: the engine picks them per batch size)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_19225_b200 import _lib
from paper_2510_19225_b200.instance import gemm
lib = _lib.lib()
ms = ctypes.c_double()
# name: (N, K, epilogue, block_n, splits, block_m)
CASES = {"qkv": (2048, 1536, 3, 128, 1, 128), "o": (1536, 1536, 5, 128, 3, 256),
         "gate_up": (17920, 1536, 2, 256, 1, 256), "gate_up_bn128": (17920, 1536, 2, 128, 1, 256),
         "gate_up_bn128_m128": (17920, 1536, 2, 128, 1, 128),
         "down": (1536, 8960, 1, 128, 5, 256), "down_m128": (1536, 8960, 1, 128, 5, 128),
         "lm_head": (151936, 1536, 4, 256, 1, 256), "lm_head_bn128": (151936, 1536, 4, 128, 1, 256),
         "lm_head_bn128_m128": (151936, 1536, 4, 128, 1, 128)}
for M in (1, 16, 64, 128, 256, 512):
    row = []
    for name, (N, K, epi, bn, sp, bm) in CASES.items():
        _lib.check(lib.rlb_bench_gemm(0, M, N, K, epi, bn, sp, bm, 50, ctypes.byref(ms)))
        row.append(f"{name} {ms.value * 1e3:6.1f}")
    print(f"M={M:4d}: " + " | ".join(row), flush=True)
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(512, 1536, generator=g, device="cuda").bfloat16()
B = (0.05 * torch.randn(2048, 1536, generator=g, device="cuda")).bfloat16()
o128 = gemm(0, A, B, epilogue=3, block_n=128)
o256 = gemm(0, A, B, epilogue=3, block_n=256)
o128m = gemm(0, A, B, epilogue=3, block_n=128, block_m=128)
print("bn128 vs bn256 bit-identical:", torch.equal(o128, o256),
      "max diff", float((o128 - o256).abs().max()))
print("bm256 vs bm128 bit-identical:", torch.equal(o128, o128m))
one = gemm(0, A[:1].contiguous(), B, epilogue=3, block_n=256)
print("M=1 row bit-identical to its M=512 row:", torch.equal(one[0], o256[0]))
