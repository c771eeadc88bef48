"""tcgen05 GEMM (img_gemm.cu) vs an fp64 numpy reference on bf16-rounded
operands, for every operand major-ness the training step uses and ragged
sizes (tile tails in M, N and K)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bf16(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16  # round-to-nearest-even
    return u.astype(np.uint32).view(np.float32)


def run(mb, M, N, K, a_kmajor, b_kmajor, use_tc, seed=0):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(K, N)).astype(np.float32)
    Ab = np.ascontiguousarray(A if a_kmajor else A.T)      # K-major: [M][K]; MN-major: [K][M]
    Bb = np.ascontiguousarray(B.T if b_kmajor else B)      # K-major: [N][K]; MN-major: [K][N]
    am, ak = (K, 1) if a_kmajor else (1, M)
    bk, bn = (1, K) if b_kmajor else (N, 1)
    out = np.zeros((M, N), np.float32)
    rc = mb.LIB.morlax_gemm_test(M, N, K, Ab.ctypes.data_as(C.c_void_p), C.c_long(am), C.c_long(ak),
                                 Bb.ctypes.data_as(C.c_void_p), C.c_long(bk), C.c_long(bn),
                                 out.ctypes.data_as(C.c_void_p), use_tc)
    assert rc == 0, mb.LIB.morlax_last_error()
    ref = bf16(A).astype(np.float64) @ bf16(B).astype(np.float64) if use_tc else \
        A.astype(np.float64) @ B.astype(np.float64)
    return out, ref


@pytest.fixture(scope="module")
def mb():
    import paper_2603_09237_b200 as mb
    return mb


@pytest.mark.parametrize("a_k,b_k", [(1, 1), (0, 1), (1, 0), (0, 0)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 256, 200), (77, 12, 45), (128, 48, 512),
                                   (1000, 6, 256), (64, 200, 16),
                                   # 256-wide tiles over several row tiles, a partial N tile, a long K loop
                                   (640, 256, 384), (384, 200, 128), (1024, 256, 1024)])
def test_tc_gemm_matches_bf16_reference(mb, M, N, K, a_k, b_k):
    out, ref = run(mb, M, N, K, a_k, b_k, 1)
    err = np.abs(out - ref).max() / max(1.0, np.abs(ref).max())
    assert err < 1e-5, (err, np.abs(out - ref).max())
