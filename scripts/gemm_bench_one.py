"""One decode-GEMM shape through hc_gemm_bench (for ncu): M N K epi mode reps."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_01792_b200._native import lib, check  # noqa: E402

M, N, K, epi, mode, reps = (int(x) for x in sys.argv[1:7])
us = C.c_double()
check(lib().hc_gemm_bench(M, N, K, epi, mode, reps, C.byref(us)))
print(f"{us.value:.2f} us/launch, {N * K * 2 / us.value / 1e3:.0f} GB/s of weights")
