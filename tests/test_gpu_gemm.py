"""Dense-transform GEMMs (K4/K7) through the C ABI: the SIMT FP32 kernels
and the tcgen05 TF32 kernels against a float64 numpy reference of the same
op, at the shapes of the BASELINE configs (odd widths included)."""

import numpy as np
import pytest

from paper_2311_14898_b200 import _native as N

pytestmark = pytest.mark.gpu


def _gemm(op, prec, A, W, G, M, K, Nn):
    rows, cols = (K, Nn) if op == 3 else ((M, K) if op == 2 else (M, Nn))
    C = np.zeros((rows, cols), np.float32)
    N.call("ht_gemm_test", op, prec, N.ptr(A), N.ptr(W), N.ptr(G), N.ptr(C), M, K, Nn)
    return C


def _ref(op, A, W, G):
    A64, W64 = A.astype(np.float64), None if W is None else W.astype(np.float64)
    G64 = None if G is None else G.astype(np.float64)
    if op == 0:
        return np.maximum(A64 @ W64, 0)
    if op == 1:
        return np.where(A64 @ W64 > 0, G64, 0)
    if op == 2:
        return A64 @ W64.T
    return A64.T @ G64


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


SHAPES = [(1000, 64, 128), (777, 100, 256), (5000, 256, 256), (300, 256, 47), (129, 128, 16),
          (4096, 200, 128), (64, 32, 172)]


@pytest.mark.parametrize("M,K,Nn", SHAPES)
@pytest.mark.parametrize("op", [0, 1, 2, 3])
@pytest.mark.parametrize("prec", [0, 1])
def test_gemm_ops(op, prec, M, K, Nn):
    rng = np.random.default_rng(M + K + Nn + op)
    A = rng.standard_normal((M, Nn if op == 2 else K)).astype(np.float32)
    W = (rng.standard_normal((K, Nn)) / np.sqrt(K)).astype(np.float32)
    G = rng.standard_normal((M, Nn)).astype(np.float32)
    C = _gemm(op, prec, A, W, G, M, K, Nn)
    R = _ref(op, A, W, G)
    if op == 1:
        # compare where the mask decision is not on a rounding knife edge
        z = A.astype(np.float64) @ W.astype(np.float64)
        safe = np.abs(z) > 1e-4 * np.abs(z).max()
        C, R = C[safe], R[safe]
    # SIMT FP32 and 3xTF32 (ops 0/1) are FP32-accurate; 1xTF32 (ops 2/3)
    # carries the 10-bit TF32 mantissa
    tol = 1e-5 if (prec == 0 or op in (0, 1)) else 3e-3
    assert _rel(C, R) < tol, (op, prec, M, K, Nn, _rel(C, R))


def test_tc_recompute_is_bitwise_stable():
    """The backward recompute of z must reproduce the forward bits (the
    reference's hybrid == store-all guarantee, engine.py:163-171)."""
    rng = np.random.default_rng(1)
    M, K, Nn = 3000, 256, 256
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, Nn)) / 16).astype(np.float32)
    h1 = _gemm(0, 1, A, W, None, M, K, Nn)
    h2 = _gemm(0, 1, A, W, None, M, K, Nn)
    np.testing.assert_array_equal(h1, h2)
    G = np.ones((M, Nn), np.float32)
    gz = _gemm(1, 1, A, W, G, M, K, Nn)
    np.testing.assert_array_equal(gz > 0, h1 > 0)
