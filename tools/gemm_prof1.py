"""One launch of each GEMM shape with the -DMB_GEMM_PROF role timing (CTA 0)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09237_b200 as mb  # noqa: E402

SHAPES = [("fwd L1", 73728, 256, 256, 0, 0, 1), ("dX L1", 73728, 256, 256, 0, 1, 2), ("theta", 80664, 128, 256, 0, 0, 0)]
ms = C.c_double()
for name, M, N, K, av, bv, act in SHAPES:
    print("==", name, flush=True)
    mb.LIB.morlax_gemm_bench(M, N, K, av, bv, act, 1, C.byref(ms))
