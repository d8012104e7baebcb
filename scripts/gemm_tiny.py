import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19225_b200 import _lib
lib = _lib.lib()
ms = ctypes.c_double()
for case in [(512, 128, 64, 3, 128, 1), (512, 2048, 1536, 5, 128, 4), (4096, 17920, 1536, 2, 256, 1)]:
    _lib.check(lib.rlb_bench_gemm(0, *case, 256, 10, ctypes.byref(ms)))
    print(case, ms.value * 1e3, "us")
