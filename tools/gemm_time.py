"""Standalone time of the update's GEMM shapes (morlax_gemm_bench, 50 launches each)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09237_b200 as mb  # noqa: E402

SHAPES = [("fwd_L1", 65536, 256, 256, 0, 0, 1), ("dX_L1", 65536, 256, 256, 0, 1, 2), ("theta", 80664, 128, 256, 0, 0, 0)]
ms = C.c_double()
out = []
for name, M, N, K, av, bv, act in SHAPES:
    mb.LIB.morlax_gemm_bench(M, N, K, av, bv, act, 50, C.byref(ms))
    out.append("%s %.2f us" % (name, ms.value * 1e3))
print(" | ".join(out))
