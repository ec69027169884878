"""Edge cases the reference's own tests pin (tests/test_engine.py:69-75,
145-163, 351-356, 482-490, 500-507), run through the GPU path: no edges,
sources without out-edges, empty training mask, zero learning rate, the
activation tracker - for GCN and GAT, with and without the owner cache."""

import warnings

import numpy as np
import pytest

import paper_2311_14898_b200 as H
from oracle import hongtu_oracle as O

pytestmark = pytest.mark.gpu


def _setup(g, X, labels, mask, m, n, kind, dims, cache="auto", lr=0.1, seed=1):
    a = H.partition_vertices(g, m, seed=seed)
    p = H.split_chunks(g, a, n)
    plan = H.plan_for_partition(p)
    model = H.init_model(kind, dims, seed=seed, lr=lr, dtype=np.float32)
    host = H.HostStore(g.num_vertices, dims, dtype=np.float32)
    host.set_features(X)
    fleet = H.DeviceFleet(plan, dtype=np.float32, precision="fp32", cache=cache)
    return a, p, model, host, fleet


@pytest.mark.parametrize("kind", ["gcn", "gat"])
@pytest.mark.parametrize("cache", ["auto", "off"])
def test_graph_without_edges(kind, cache):
    """No edges: every aggregate is zero, so h^1.. = 0 and the loss is ln K
    on the masked rows; nothing is flushed but the epoch completes."""
    V, K = 64, 4
    g = H.from_edges(np.zeros(0, np.int64), np.zeros(0, np.int64), V)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((V, 8))
    labels = rng.integers(0, K, V)
    mask = np.ones(V, bool)
    a, p, model, host, fleet = _setup(g, X, labels, mask, 2, 2, kind, [8, 8, K], cache)
    res = H.train_epoch(p, fleet, model, host, labels, mask)
    assert res.loss == pytest.approx(np.log(K), rel=1e-6)
    assert not np.any(np.asarray(host.h[1]))
    for gw in res.grads:
        assert not np.any(gw)


@pytest.mark.parametrize("kind", ["gcn", "gat"])
def test_sources_without_out_edges_and_isolated_vertices(kind):
    """A star into vertex 0 plus isolated vertices: sources without
    out-edges get exactly-zero gradients, against the oracle."""
    V = 40
    src = np.arange(1, 21, dtype=np.int64)
    dst = np.zeros(20, np.int64)
    src = np.concatenate([src, [3, 4, 5]])
    dst = np.concatenate([dst, [7, 7, 8]])
    g = H.from_edges(src, dst, V)
    rng = np.random.default_rng(2)
    X = rng.standard_normal((V, 8))
    labels = rng.integers(0, 4, V)
    mask = rng.random(V) < 0.7
    a, p, model, host, fleet = _setup(g, X, labels, mask, 2, 1, kind, [8, 8, 4])
    w0 = [w.copy() for w in model.weights]
    a0 = [x.copy() for x in model.attn] if kind == "gat" else None
    res = H.train_epoch(p, fleet, model, host, labels, mask)
    grid = [[vars(c) for c in row] for row in p.chunks]
    ref = O.partitioned_epoch(grid, O.plan_of_grid(grid, a.owner), w0, X, labels, mask,
                              dtype=np.float32, kind=kind, attn=a0)
    assert abs(res.loss - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    gh0 = np.asarray(host.grad_h[0])
    assert not np.any(gh0[21:][~np.isin(np.arange(21, V), [3, 4, 5])])  # no out-edges
    assert O.rel_err(gh0, ref["grad_h"][0]) < 1e-5
    for l in range(2):
        assert O.rel_err(res.grads[l], ref["grads"][l]) < 1e-5


@pytest.mark.parametrize("kind", ["gcn", "gat"])
def test_empty_mask_warns_zero_loss_and_no_update(kind):
    ds = H.synth_dataset(H.SynthSpec(num_vertices=900, avg_degree=6.0, seed=3), 8, 4)
    mask = np.zeros(900, bool)
    a, p, model, host, fleet = _setup(ds.graph, ds.features, ds.labels, mask, 2, 2, kind,
                                      [8, 8, 4])
    w0 = [w.copy() for w in model.weights]
    with pytest.warns(UserWarning, match="mask is empty"):
        res = H.train_epoch(p, fleet, model, host, ds.labels, mask)
    assert res.loss == 0.0
    for w, w_ in zip(model.weights, w0):
        np.testing.assert_array_equal(w, w_)
    assert not np.any(np.asarray(host.grad_h[2]))


@pytest.mark.parametrize("kind", ["gcn", "gat"])
def test_zero_learning_rate_is_flat_and_tracker_balanced(kind):
    ds = H.synth_dataset(H.SynthSpec(num_vertices=1200, avg_degree=7.0, seed=4), 8, 4)
    a, p, model, host, fleet = _setup(ds.graph, ds.features, ds.labels, ds.mask, 3, 2, kind,
                                      [8, 8, 4], lr=0.0)
    w0 = [w.copy() for w in model.weights]
    tracker = H.ActivationTracker()
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        r1 = H.train_epoch(p, fleet, model, host, ds.labels, ds.mask, tracker=tracker)
        r2 = H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    assert r1.loss == r2.loss
    for w, w_ in zip(model.weights, w0):
        np.testing.assert_array_equal(w, w_)
    assert tracker.live_count == 0
    assert 1 <= tracker.peak <= p.m
    fwd, bwd = H.comm_passes_per_epoch(model)
    assert fleet.transfer_report(2 * fwd, 2 * bwd)["planner_consistent"]
