"""Per-CTA latency breakdown (globaltimer stamps of CTA 0) and average time of
the decode-step GEMM shapes; RLB_GEMM_DBG=1 prints the breakdown."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19225_b200 import _lib
lib = _lib.lib()
ms = ctypes.c_double()
# name: (M, N, K, epilogue, block_n, splits, block_m); epilogue 5 = fp32 partials,
# 1 = residual add (split-K reduced in a cluster)
CASES = {"qkv": (512, 2048, 1536, 5, 128, 2, 256), "qkv_m128": (512, 2048, 1536, 3, 128, 1, 128),
         "o": (512, 1536, 1536, 5, 128, 3, 256), "o_resadd_m128": (512, 1536, 1536, 1, 128, 1, 128),
         "o_resadd_m128_s2": (512, 1536, 1536, 1, 128, 2, 128),
         "gate_up": (512, 17920, 1536, 2, 256, 1, 256), "gate_up_m128": (512, 17920, 1536, 2, 256, 1, 128),
         "down": (512, 1536, 8960, 5, 128, 5, 256), "down_resadd": (512, 1536, 8960, 1, 128, 5, 256),
         "down_resadd_m128_s4": (512, 1536, 8960, 1, 128, 4, 128),
         "lm_head": (512, 151936, 1536, 4, 256, 1, 256)}
for name, case in CASES.items():
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    _lib.check(lib.rlb_bench_gemm(0, *case, 50, ctypes.byref(ms)))
    print(f"{name:22s} {case} {ms.value * 1e3:8.2f} us", flush=True)
