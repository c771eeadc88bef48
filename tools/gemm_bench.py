"""tcgen05 GEMM microbenchmark (img_gemm.cu) on the training step's shapes."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09237_b200 as mb  # noqa: E402

SHAPES = [  # (name, M, N, K, a_view, b_view, act)
    ("fwd L1 (rows x 256 x 256, tanh)", 73728, 256, 256, 0, 0, 1),
    ("fwd L0 (rows x 256 x 45)", 73728, 256, 45, 0, 0, 1),
    ("dX L1 (rows x 256 x 256, tanh')", 73728, 256, 256, 0, 1, 2),
    ("dW L1 (256 x 256 x 640 rows)", 256, 256, 640, 1, 1, 0),
    ("theta (P x G x F)", 80664, 128, 256, 0, 0, 0),
    ("dM (P x F x G)", 80664, 256, 128, 1, 1, 0),
    ("big square 16384^2 x 4096", 16384, 256, 4096, 0, 0, 0),
]
for name, M, N, K, av, bv, act in SHAPES:
    ms = C.c_double()
    rc = mb.LIB.morlax_gemm_bench(M, N, K, av, bv, act, 20, C.byref(ms))
    assert rc == 0, mb.LIB.morlax_last_error()
    tf = 2.0 * M * N * K / (ms.value * 1e-3) / 1e12
    print(f"{name:40s} {ms.value * 1e3:9.1f} us  {tf:7.1f} TFLOP/s")
