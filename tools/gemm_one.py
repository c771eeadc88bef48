"""One tcgen05 GEMM shape, for ncu: python tools/gemm_one.py M N K a_view b_view act iters"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09237_b200 as mb  # noqa: E402

M, N, K, av, bv, act, iters = (int(x) for x in sys.argv[1:8])
ms = C.c_double()
assert mb.LIB.morlax_gemm_bench(M, N, K, av, bv, act, iters, C.byref(ms)) == 0, mb.LIB.morlax_last_error()
print(f"{M}x{N}x{K} act{act}: {ms.value * 1e3:.1f} us, {2.0 * M * N * K / (ms.value * 1e-3) / 1e12:.1f} TFLOP/s")
