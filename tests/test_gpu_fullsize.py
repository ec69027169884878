"""Parity at the bench's full size (BASELINE config 2: 2.4M vertices, ~62M
edges, 3-layer GCN 100-256-256-47, m = n = 1, TF32) through properties that
do not need a full CPU epoch:

* forward aggregation rows of sampled destinations are bitwise the
  sequential multiply-then-add over their CSC in-edges (np.add.at,
  src/engine.py:139);
* h^{l+1} = max(agg^l . W^l, 0) on sampled rows (3xTF32: FP32-accurate);
* grad_h^L rows are the masked softmax-CE gradient of h^L (src/engine.py:297-320);
* the last layer's dW = agg^{L-1}^T (grad_h^L * 1[h^L > 0]) over all 2.4M
  rows against float64 (1xTF32: the north star's 1e-3);
* W_new = W - lr * dW bitwise (src/engine.py:328-344);
* the HBM store and the pinned host store give bitwise the same epoch;
* layer by layer against the fp64 oracle fed with the GPU's own layer
  inputs h^l and output gradients grad_h^{l+1} (so each layer is checked
  alone, at the north star's 1e-3): every layer's h^{l+1} and dW, grad_h^l
  on sampled rows plus the 20 highest out-degree sources (the hub pieces of
  the transposed aggregation), the loss and grad_h^L - for the GCN (whose
  narrow last layer runs project-first, z = A.(h.W), against the oracle's
  (A.h).W) and for the bench's GAT (256-128-128-64, dW, da, grad_h).
"""

import numpy as np
import pytest

import paper_2311_14898_b200 as H
from oracle import hongtu_oracle as O

pytestmark = pytest.mark.gpu

V, DEG, DIMS, SEED = 2_400_000, 26.8, [100, 256, 256, 47], 0


@pytest.fixture(scope="module")
def full():
    ds = H.synth_dataset(H.SynthSpec(num_vertices=V, avg_degree=DEG, seed=SEED), DIMS[0], DIMS[-1])
    a = H.partition_vertices(ds.graph, 1, seed=SEED)
    p = H.split_chunks(ds.graph, a, 1)
    plan = H.plan_for_partition(p, device=0)
    return ds, p, plan


def _epoch(full, placement):
    ds, p, plan = full
    model = H.init_model("gcn", DIMS, seed=SEED, lr=0.1, dtype=np.float32)
    w0 = [w.copy() for w in model.weights]
    host = H.HostStore(V, DIMS, dtype=np.float32, placement=placement)
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, precision="tf32")
    res = H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    return res, model, w0, host, fleet


def test_fullsize_epoch_properties(full):
    ds, p, plan = full
    g = ds.graph
    res, model, w0, host, fleet = _epoch(full, "device")
    L = len(DIMS) - 1
    rng = np.random.default_rng(7)
    rows = np.sort(rng.choice(V, 2000, replace=False))
    h = [np.asarray(x) for x in host.h]
    agg = [np.asarray(host.agg[l]) for l in range(L)]
    w32 = np.asarray(g.edge_weights, dtype=np.float32)
    for l in range(L):
        for v in rows[:300]:  # bitwise sequential aggregation
            acc = np.zeros(DIMS[l], np.float32)
            for e in range(g.csc_offsets[v], g.csc_offsets[v + 1]):
                acc = acc + w32[e] * h[l][g.csc_sources[e]]
            np.testing.assert_array_equal(agg[l][v], acc, err_msg=f"layer {l} row {v}")
        z = agg[l][rows].astype(np.float64) @ w0[l].astype(np.float64)
        ref = np.maximum(z, 0)
        err = np.abs(h[l + 1][rows] - ref).max() / np.abs(ref).max()
        assert err < 1e-5, (l, err)
    # loss gradient rows
    hl = h[L][rows].astype(np.float64)
    pr = np.exp(hl - hl.max(1, keepdims=True))
    pr /= pr.sum(1, keepdims=True)
    count = int(np.asarray(ds.mask).sum())
    gref = (pr - np.eye(DIMS[L])[np.asarray(ds.labels)[rows]]) / count
    gref[~np.asarray(ds.mask)[rows]] = 0
    gl = np.asarray(host.grad_h[L])[rows]
    assert np.abs(gl - gref).max() <= 1e-6 * np.abs(gref).max() + 1e-12
    # last layer's weight gradient over every row, against float64
    gz = np.asarray(host.grad_h[L]).astype(np.float64) * (h[L] > 0)
    dW = agg[L - 1].astype(np.float64).T @ gz
    err = np.abs(res.grads[L - 1] - dW).max() / np.abs(dW).max()
    assert err < 1e-3, err
    # SGD step, bitwise (separate roundings, src/engine.py:342)
    for l in range(L):
        np.testing.assert_array_equal(model.weights[l],
                                      w0[l] - np.float32(0.1) * res.grads[l])
    fleet.close()


def test_fullsize_host_store_equals_hbm_store(full):
    r_d, m_d, _, host_d, f_d = _epoch(full, "device")
    hd = [np.asarray(x) for x in host_d.h[1:]]
    f_d.close()
    del host_d
    r_h, m_h, _, host_h, f_h = _epoch(full, "host")
    assert f_h.cache_active
    assert r_d.loss == r_h.loss
    for a, b in zip(m_d.weights, m_h.weights):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(hd, host_h.h[1:]):
        np.testing.assert_array_equal(a, b)
    f_h.close()


def _graph_dict(g):
    return {"num_vertices": g.num_vertices, "csc_offsets": g.csc_offsets,
            "csc_sources": g.csc_sources, "edge_weights": g.edge_weights}


def _check_rows(l, got, ref, rows, hubs, what):
    err = O.rel_err(got[rows], ref[rows])
    assert err < 1e-3, (what, l, "sampled rows", err)
    err = O.rel_err(got[hubs], ref[hubs])
    assert err < 1e-3, (what, l, "hub rows", err)


def _loss_check(res, h_last, g_last, labels, mask):
    loss_ref, grad_ref = O.masked_xent_fp64(h_last, labels, mask)
    assert abs(res.loss - loss_ref) <= 1e-5 * abs(loss_ref), (res.loss, loss_ref)
    assert O.rel_err(g_last, grad_ref) < 1e-5


def test_fullsize_gcn_layerwise_vs_fp64_oracle(full):
    ds, p, plan = full
    g = ds.graph
    res, model, w0, host, fleet = _epoch(full, "device")
    L = len(DIMS) - 1
    h = [np.asarray(x) for x in host.h]
    gh = [np.asarray(x) for x in host.grad_h]
    fleet.close()
    _loss_check(res, h[L], gh[L], ds.labels, ds.mask)
    hubs = np.argsort(np.diff(g.csr_offsets), kind="stable")[-20:]
    assert np.diff(g.csr_offsets)[hubs].min() > 1024  # they run through the pieces path
    rows = np.random.default_rng(11).choice(V, 2000, replace=False)
    A = O.adjacency_fp64(_graph_dict(g))
    for l in reversed(range(L)):
        r = O.gcn_layer_fp64(A, h[l], w0[l], gh[l + 1])
        err = O.rel_err(h[l + 1], r["h_out"])
        assert err < 1e-3, ("h", l + 1, err)
        err = O.rel_err(res.grads[l], r["grad_W"])
        assert err < 1e-3, ("dW", l, err)
        _check_rows(l, gh[l], r["grad_h"], rows, hubs, "grad_h")
        del r


GAT_DIMS = [256, 128, 128, 64]  # bench.py's GAT line (config 5's widths)


def test_fullsize_gat_layerwise_vs_fp64_oracle(full):
    ds, p, plan = full
    g = ds.graph
    X = np.random.default_rng(SEED).standard_normal((V, GAT_DIMS[0]), dtype=np.float32)
    y = (np.asarray(ds.labels) % GAT_DIMS[-1]).astype(np.int64)
    model = H.init_model("gat", GAT_DIMS, seed=SEED, lr=0.1, dtype=np.float32)
    w0 = [w.copy() for w in model.weights]
    a0 = [a.copy() for a in model.attn]
    host = H.HostStore(V, GAT_DIMS, dtype=np.float32, placement="device")
    host.set_features(X)
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, precision="tf32")
    res = H.train_epoch(p, fleet, model, host, y, ds.mask)
    L = len(GAT_DIMS) - 1
    h = [np.asarray(x) for x in host.h]
    gh = [np.asarray(x) for x in host.grad_h]
    fleet.close()
    _loss_check(res, h[L], gh[L], y, ds.mask)
    hubs = np.argsort(np.diff(g.csr_offsets), kind="stable")[-20:]
    rows = np.random.default_rng(12).choice(V, 2000, replace=False)
    gd = _graph_dict(g)
    for l in reversed(range(L)):
        r = O.gat_layer_fp64(gd, h[l], w0[l], a0[l], slope=model.leaky_slope, grad_out=gh[l + 1])
        err = O.rel_err(h[l + 1], r["h_out"])
        assert err < 1e-3, ("h", l + 1, err)
        err = O.rel_err(res.grads[l], r["grad_W"])
        assert err < 1e-3, ("dW", l, err)
        err = O.rel_err(res.attn_grads[l], r["grad_a"])
        assert err < 1e-3, ("da", l, err)
        _check_rows(l, gh[l], r["grad_h"], rows, hubs, "grad_h")
        del r
