import ctypes as C, os, sys
sys.path.insert(0, '/root/repo')
import paper_2603_09237_b200 as mb
for name, M, N, K, av, bv, act in [
    ("fwd  b0 act1", 73728, 256, 256, 0, 0, 1),
    ("fwd  b0 act0", 73728, 256, 256, 0, 0, 0),
    ("dX   b1 act2", 73728, 256, 256, 0, 1, 2),
    ("dX   b1 act1", 73728, 256, 256, 0, 1, 1),
    ("dX   b1 act0", 73728, 256, 256, 0, 1, 0),
    ("a1b1 act0", 73728, 256, 256, 1, 1, 0),
    ("fwd BN128 b0 act1", 73728, 128, 256, 0, 0, 1),
    ("fwd BN128 b1 act1", 73728, 128, 256, 0, 1, 1),
    ("K512 b0 act1", 73728, 256, 512, 0, 0, 1),
    ("K1024 b0 act0", 73728, 256, 1024, 0, 0, 0),
]:
    ms = C.c_double()
    assert mb.LIB.morlax_gemm_bench(M, N, K, av, bv, act, 20, C.byref(ms)) == 0
    print(f"{name:22s} {ms.value*1e3:8.1f} us {2.0*M*N*K/(ms.value*1e-3)/1e12:7.1f} TF")
