"""Dense-transform GEMMs (K4/K7) through the C ABI: the SIMT FP32 kernels
and the tcgen05 TF32 kernels against a float64 numpy reference of the same
op, at the shapes of the BASELINE configs (odd widths included)."""

import numpy as np
import pytest

from paper_2311_14898_b200 import _native as N

pytestmark = pytest.mark.gpu


def _gemm(op, prec, A, W, G, M, K, Nn):
    rows, cols = (K, Nn) if op == 3 else ((M, K) if op in (2, 4) else (M, Nn))
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


def _tf32_rna(x):
    """cvt.rna.tf32.f32: round to the 10-bit mantissa, ties away from zero."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return ((u + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.parametrize("M,K,Nn", [(5000, 256, 256), (777, 100, 256), (300, 256, 48),
                                    (4096, 200, 128), (129, 172, 32)])
def test_masked_gemm_equals_mask_then_gemm(M, K, Nn):
    """The backward's gz . W^T with the ReLU' mask formed inside the tcgen05
    GEMM (TMA loads of the g and h tiles, gz stored from the masked stage):
    the product is bitwise the unfused mask-then-GEMM's, gz is g * [h > 0]
    TF32-rounded (RNA; k_tc_wgrad rounds its operands the same way)."""
    rng = np.random.default_rng(M + K)
    h = np.maximum(rng.standard_normal((M, Nn)), 0).astype(np.float32)
    g = rng.standard_normal((M, Nn)).astype(np.float32)
    W = (rng.standard_normal((K, Nn)) / np.sqrt(Nn)).astype(np.float32)
    gz = np.where(h > 0, g, 0).astype(np.float32)
    C = _gemm(4, 1, h, W, g, M, K, Nn)
    np.testing.assert_array_equal(C, _gemm(2, 1, gz, W, None, M, K, Nn))
    np.testing.assert_array_equal(_gemm(5, 1, h, W, g, M, K, Nn), _tf32_rna(gz))
    assert _rel(C, gz.astype(np.float64) @ W.astype(np.float64).T) < 3e-3


def test_pair_gemm_matches_single_cta():
    """HT_PAIR=1: 3xTF32 row GEMMs with N > 128 run on CTA pairs
    (cta_group::2, M = 256 MMAs, each SM staging half of the weights); the
    default runs one CTA per 128-row tile.
    Same operands, same k order, same three products per k step: the
    outputs agree to FP32 accumulation-order noise (checked bitwise-or-1ulp),
    including tiles whose second half lies past the last row."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, sys\n"
        "import importlib.util as u\n"
        "sp = u.spec_from_file_location('tgg', %r)\n"
        "m = u.module_from_spec(sp); sp.loader.exec_module(m); _gemm = m._gemm\n"
        "out = []\n"
        "for M, K, Nn in [(1000, 64, 256), (777, 100, 256), (129, 128, 200), (300, 256, 172)]:\n"
        "    rng = np.random.default_rng(M)\n"
        "    A = rng.standard_normal((M, K)).astype(np.float32)\n"
        "    W = (rng.standard_normal((K, Nn)) / np.sqrt(K)).astype(np.float32)\n"
        "    G = rng.standard_normal((M, Nn)).astype(np.float32)\n"
        "    out += [_gemm(0, 1, A, W, None, M, K, Nn), _gemm(1, 1, A, W, G, M, K, Nn)]\n"
        "np.savez(sys.argv[1], *out)\n") % os.path.abspath(__file__)
    import tempfile
    res = {}
    with tempfile.TemporaryDirectory() as td:
        for flag in ("0", "1"):
            f = os.path.join(td, "o%s.npz" % flag)
            env = dict(os.environ, HT_PAIR=flag)
            subprocess.run([sys.executable, "-c", code, f], check=True, env=env, timeout=600)
            z = np.load(f)
            res[flag] = [z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))]
    for a, b in zip(res["0"], res["1"]):
        ulp = np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))
        assert ulp.max() <= 1, ulp.max()
