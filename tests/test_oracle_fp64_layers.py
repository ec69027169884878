"""The whole-graph fp64 layer restatements the full-size GPU parity tests
use (oracle.gcn_layer_fp64 / gat_layer_fp64 / masked_xent_fp64) agree with
the golden-pinned per-chunk oracle kernels on a small graph (one chunk =
the whole graph, m = n = 1)."""

import numpy as np

from oracle import hongtu_oracle as O


def _graph(V=300, E=2400, seed=5):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, V, size=E)
    dst = rng.integers(0, V, size=E)
    # a hub source and an isolated destination
    src[:200] = 7
    dst[dst == 11] = 12
    return O.build_graph(src, dst, V)


def test_gcn_layer_fp64_matches_chunk_kernels():
    g = _graph()
    V = g["num_vertices"]
    rng = np.random.default_rng(1)
    h = rng.standard_normal((V, 12))
    W = rng.standard_normal((12, 8))
    gout = rng.standard_normal((V, 8))
    ch = O.chunk_of(g, np.arange(V))
    h_out, agg, _ = O.gcn_chunk_forward(ch, h[ch["sources"]], W)
    gnbr, gW = O.gcn_chunk_backward(ch, agg, gout, W)
    r = O.gcn_layer_fp64(O.adjacency_fp64(g), h, W, gout)
    np.testing.assert_allclose(r["agg"], agg, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(r["h_out"], h_out, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(r["grad_W"], gW, rtol=1e-12, atol=1e-12)
    gh = np.zeros((V, 12))
    gh[ch["sources"]] = gnbr
    np.testing.assert_allclose(r["grad_h"], gh, rtol=1e-12, atol=1e-12)


def test_gat_layer_fp64_matches_chunk_kernels():
    g = _graph()
    V = g["num_vertices"]
    rng = np.random.default_rng(2)
    h = rng.standard_normal((V, 12))
    W = rng.standard_normal((12, 8)) * 0.3
    a = rng.standard_normal(16) * 0.3
    gout = rng.standard_normal((V, 8))
    ch = O.chunk_of(g, np.arange(V))
    h_out, _ = O.gat_chunk_forward(ch, h[ch["sources"]], h, W, a)
    gnbr, gdst, gW, ga = O.gat_chunk_backward(ch, h[ch["sources"]], h, gout, W, a)
    r = O.gat_layer_fp64(g, h, W, a, grad_out=gout, block=500)
    np.testing.assert_allclose(r["h_out"], h_out, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(r["grad_W"], gW, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(r["grad_a"], ga, rtol=1e-11, atol=1e-11)
    gh = gdst.copy()
    gh[ch["sources"]] += gnbr
    np.testing.assert_allclose(r["grad_h"], gh, rtol=1e-11, atol=1e-11)


def test_masked_xent_fp64():
    rng = np.random.default_rng(3)
    z = rng.standard_normal((50, 6)).astype(np.float32)
    y = rng.integers(0, 6, 50)
    m = rng.random(50) < 0.4
    l32, g32 = O.softmax_xent(z.astype(np.float64), y, m)
    l64, g64 = O.masked_xent_fp64(z, y, m)
    assert l32 == l64
    np.testing.assert_array_equal(g32, g64)
