"""GPU unit test of the in-kernel block GEMM building blocks (SIMT FP32 and tcgen05
3xTF32 / 1xTF32) against an FP64 numpy product, over the shapes and transpositions the
fused per-centre kernels use (ragged M/N/K, M > 128, N > 256)."""
import ctypes as C

import numpy as np
import pytest

import paper_2604_07276_b200 as nb

pytestmark = pytest.mark.gpu

SHAPES = [(90, 256, 128), (90, 90, 128), (90, 128, 90), (123, 96, 123), (17, 16, 8), (160, 256, 256),
          (200, 130, 70), (1, 1, 1), (128, 512, 32)]


def run(mode, ta, tb, A, B):
    L = nb.lib()
    L.nnmd_b200_selftest_gemm.argtypes = [C.c_int] * 6 + [C.POINTER(C.c_float)] * 3
    M = A.shape[1] if ta else A.shape[0]
    K = A.shape[0] if ta else A.shape[1]
    N = B.shape[0] if tb else B.shape[1]
    A32 = np.ascontiguousarray(A, dtype=np.float32)
    B32 = np.ascontiguousarray(B, dtype=np.float32)
    Cm = np.zeros((M, N), dtype=np.float32)
    fp = C.POINTER(C.c_float)
    rc = L.nnmd_b200_selftest_gemm(mode, ta, tb, M, N, K, A32.ctypes.data_as(fp), B32.ctypes.data_as(fp),
                                   Cm.ctypes.data_as(fp))
    assert rc == 0, L.nnmd_b200_last_error()
    return Cm


@pytest.mark.parametrize("mode,tol", [(0, 5e-6), (1, 3e-5), (2, 2e-3)])
@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("shape", SHAPES)
def test_block_gemm(mode, tol, ta, tb, shape):
    M, N, K = shape
    rng = np.random.default_rng(M * 1000 + N * 10 + K)
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    ref = A.astype(np.float32).astype(np.float64) @ B.astype(np.float32).astype(np.float64)
    got = run(mode, ta, tb, A.T.copy() if ta else A, B.T.copy() if tb else B)
    scale = np.sqrt(K) * 1.0
    err = np.abs(got - ref).max() / scale
    assert err <= tol, (mode, ta, tb, shape, err)
