"""HBM owner cache: with the cache the layer drivers
read owned rows from HBM mirrors instead of the host store and write every
produced row through.  The arithmetic is unchanged, so an epoch with the
cache must equal the cache-off epoch bitwise - host arrays (h, agg,
grad_h), weights, attention vectors, loss and meters - for GCN and GAT,
single and multiple devices and batches (re-flushes)."""

import numpy as np
import pytest

import paper_2311_14898_b200 as H

pytestmark = pytest.mark.gpu


def _epochs(p, ds, dims, kind, cache, mode="full", precision="tf32", epochs=2):
    plan = H.plan_for_partition(p)
    model = H.init_model(kind, dims, seed=3, lr=0.1, dtype=np.float32)
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, mode=mode, dtype=np.float32, precision=precision, cache=cache)
    out = []
    for _ in range(epochs):
        r = H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
        snap = {"loss": r.loss, "W": [w.copy() for w in model.weights],
                "h": [np.array(x) for x in host.h], "gh": [np.array(x) for x in host.grad_h],
                "agg": {k: np.array(v) for k, v in host.agg.items()}}
        if kind == "gat":
            snap["A"] = [a.copy() for a in model.attn]
        out.append(snap)
    rep = fleet.transfer_report(*H.comm_passes_per_epoch(model))
    return out, rep, fleet.cache_active


@pytest.mark.parametrize("kind", ["gcn", "gat"])
@pytest.mark.parametrize("m,n,mode", [(1, 1, "full"), (1, 3, "full"), (3, 2, "full"),
                                      (2, 3, "p2p")])
def test_cache_bitwise_equals_host_path(kind, m, n, mode, monkeypatch):
    # the narrow-side backward reassociates (A^T gz) W^T; it needs gz built
    # from the HBM-resident output, which only the cache path has - compare
    # like with like here (the narrow path is checked against the oracle)
    monkeypatch.setenv("HT_NO_NARROW_BWD", "1")
    # likewise the one-device GAT path sums dW / da over all rows (rows
    # without out-edges add zeros: a different association of the same sums)
    monkeypatch.setenv("HT_NO_GAT_DIRECT", "1")
    monkeypatch.setenv("HT_NO_PROJECT_FIRST", "1")  # (needs HBM checkpoints; reassociates)
    # the split GAT backward needs h^{l+1} in HBM (cache on) and reassociates gq
    monkeypatch.setenv("HT_NO_GAT_SPLIT", "1")
    ds = H.synth_dataset(H.SynthSpec(num_vertices=2500, avg_degree=8.0, seed=4), 16, 8)
    a = H.partition_vertices(ds.graph, m, seed=4)
    p = H.split_chunks(ds.graph, a, n)
    if n > 1:
        p = H.reorganize(p).partition
    dims = [16, 24, 8]
    off, rep_off, act_off = _epochs(p, ds, dims, kind, "off", mode)
    on, rep_on, act_on = _epochs(p, ds, dims, kind, "on", mode)
    assert not act_off and act_on
    assert rep_on["totals"] == rep_off["totals"]
    for a_, b_ in zip(off, on):
        assert a_["loss"] == b_["loss"]
        for key in ("W", "h", "gh") + (("A",) if kind == "gat" else ()):
            for x, y in zip(a_[key], b_[key]):
                np.testing.assert_array_equal(x, y, err_msg=key)
        for l in a_["agg"]:
            np.testing.assert_array_equal(a_["agg"][l], b_["agg"][l])


def test_cache_refused_in_baseline_mode():
    ds = H.synth_dataset(H.SynthSpec(num_vertices=800, avg_degree=6.0, seed=1), 8, 4)
    p = H.split_chunks(ds.graph, H.partition_vertices(ds.graph, 2, seed=1), 2)
    with pytest.raises(H.ChunktrainError, match="cache"):
        _epochs(p, ds, [8, 8, 4], "gcn", "on", mode="baseline", epochs=1)
    _, _, active = _epochs(p, ds, [8, 8, 4], "gcn", "auto", mode="baseline", epochs=1)
    assert not active


def test_compact_host_store_single_device():
    """A compact store holding all rows (m = 1) is the full store; the
    compact path (contiguous host copies) must give bitwise the same epoch."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=2000, avg_degree=8.0, seed=6), 16, 8)
    a = H.partition_vertices(ds.graph, 1, seed=6)
    p = H.split_chunks(ds.graph, a, 2)
    dims = [16, 24, 8]
    plan = H.plan_for_partition(p)
    outs = []
    for rows in (None, np.arange(ds.graph.num_vertices)):
        model = H.init_model("gcn", dims, seed=3, lr=0.1, dtype=np.float32)
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32, rows=rows)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, dtype=np.float32)
        r = H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
        outs.append((r.loss, [w.copy() for w in model.weights], np.array(host.grad_h[0]),
                     np.array(host.h[2]), np.array(host.agg[1])))
    a_, b_ = outs
    assert a_[0] == b_[0]
    for x, y in zip(a_[1:], b_[1:]):
        np.testing.assert_array_equal(x if not isinstance(x, list) else np.concatenate(
            [w.ravel() for w in x]), y if not isinstance(y, list) else np.concatenate(
            [w.ravel() for w in y]))


def test_compact_host_store_rejected_for_multi_device_fleet():
    ds = H.synth_dataset(H.SynthSpec(num_vertices=1000, avg_degree=6.0, seed=2), 8, 4)
    a = H.partition_vertices(ds.graph, 2, seed=2)
    p = H.split_chunks(ds.graph, a, 1)
    plan = H.plan_for_partition(p)
    model = H.init_model("gcn", [8, 8, 4], seed=1, dtype=np.float32)
    host = H.HostStore(ds.graph.num_vertices, [8, 8, 4], dtype=np.float32,
                       rows=np.flatnonzero(a.owner == 0))
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, dtype=np.float32)
    with pytest.raises(H.ChunktrainError, match="one local device"):
        H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)


@pytest.mark.parametrize("kind", ["gcn", "gat"])
def test_lean_epoch_same_parameters(kind):
    """Lean epochs skip grad_h^0 and the host copies of
    h^L / grad_h^L; weights, attention vectors, loss and the remaining host
    arrays are bitwise those of the full epoch."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=2500, avg_degree=8.0, seed=8), 16, 8)
    a = H.partition_vertices(ds.graph, 2, seed=8)
    p = H.split_chunks(ds.graph, a, 2)
    dims = [16, 24, 8]
    plan = H.plan_for_partition(p)
    outs = []
    for lean in (False, True):
        model = H.init_model(kind, dims, seed=3, lr=0.1, dtype=np.float32)
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, dtype=np.float32, lean=lean)
        losses = [H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss for _ in range(2)]
        outs.append((losses, [w.copy() for w in model.weights],
                     [x.copy() for x in model.attn] if kind == "gat" else [],
                     np.array(host.h[1]), np.array(host.grad_h[1]), np.array(host.grad_h[0])))
    full, lean = outs
    assert full[0] == lean[0]
    for x, y in zip(full[1] + full[2], lean[1] + lean[2]):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(full[3], lean[3])
    np.testing.assert_array_equal(full[4], lean[4])
    assert np.any(full[5] != 0) and not np.any(lean[5])  # grad_h^0 not produced


@pytest.mark.parametrize("kind", ["gcn", "gat"])
def test_hbm_store_in_place_equals_host_store(kind):
    """An HBM-resident store (placement="device", one device) is used in place
    as the owner-cache mirror: same epoch, bitwise, as the pinned host store."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=2500, avg_degree=8.0, seed=5), 16, 8)
    a = H.partition_vertices(ds.graph, 1, seed=5)
    p = H.split_chunks(ds.graph, a, 2)
    dims = [16, 24, 8]
    plan = H.plan_for_partition(p)
    outs = []
    for placement in ("host", "device"):
        model = H.init_model(kind, dims, seed=3, lr=0.1, dtype=np.float32)
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32, placement=placement)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, dtype=np.float32)
        losses = [H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss for _ in range(2)]
        assert fleet.cache_active
        snap = [np.array(x) for x in host.h] + [np.array(x) for x in host.grad_h]
        if kind == "gcn":
            snap += [np.array(host.agg[l]) for l in range(2)]
        outs.append((losses, [w.copy() for w in model.weights], snap))
    assert outs[0][0] == outs[1][0]
    for x, y in zip(outs[0][1] + outs[0][2], outs[1][1] + outs[1][2]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("m,n", [(1, 1), (1, 3), (3, 2)])
def test_hbm_checkpoints_equal_host_checkpoints(m, n, monkeypatch):
    """Checkpoint tier: with the owner cache the GCN agg checkpoints stay in
    HBM (checkpoints="auto") instead of being written through ("host").
    The epochs must be bitwise equal, and host.agg - filled from HBM on first
    read, here after two epochs and after the fleet is closed - must equal
    the written-through arrays."""
    monkeypatch.setenv("HT_NO_PROJECT_FIRST", "1")  # same arithmetic on both sides
    ds = H.synth_dataset(H.SynthSpec(num_vertices=2500, avg_degree=8.0, seed=5), 16, 8)
    a = H.partition_vertices(ds.graph, m, seed=5)
    p = H.split_chunks(ds.graph, a, n)
    if n > 1:
        p = H.reorganize(p).partition
    dims = [16, 24, 8]
    plan = H.plan_for_partition(p)
    res = {}
    for ck in ("host", "auto"):
        model = H.init_model("gcn", dims, seed=3, lr=0.1, dtype=np.float32)
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, cache="on", checkpoints=ck)
        losses = [H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss for _ in range(2)]
        held = dict(host.agg.pending)
        assert bool(held) == (ck == "auto")
        fleet.close()  # HBM-held checkpoints are materialized before the buffers go
        assert not host.agg.pending
        res[ck] = (losses, [w.copy() for w in model.weights], [np.array(g) for g in host.grad_h],
                   {l: np.array(host.agg[l]) for l in range(len(dims) - 1)})
    assert res["host"][0] == res["auto"][0]
    for x, y in zip(res["host"][1] + res["host"][2], res["auto"][1] + res["auto"][2]):
        np.testing.assert_array_equal(x, y)
    for l in res["host"][3]:
        np.testing.assert_array_equal(res["host"][3][l], res["auto"][3][l])
        assert np.abs(res["auto"][3][l]).sum() > 0


def test_project_first_layers(monkeypatch):
    """One device, one batch, HBM checkpoints: layers with d_out < d_in run
    z = A.(h.W) (narrow gather) and dW = h^T (A^T gz).  Against the
    (A.h).W path: parameters and outputs within FP32 reassociation error,
    and the deferred checkpoints - aggregated when host.agg is read - bitwise
    equal where their inputs are (agg^0)."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=3000, avg_degree=9.0, seed=8), 32, 8)
    p = H.split_chunks(ds.graph, H.partition_vertices(ds.graph, 1, seed=8), 1)
    plan = H.plan_for_partition(p)
    dims = [32, 16, 8]  # both layers narrow
    out = {}
    for flag in ("1", None):
        if flag:
            monkeypatch.setenv("HT_NO_PROJECT_FIRST", flag)
        else:
            monkeypatch.delenv("HT_NO_PROJECT_FIRST", raising=False)
        model = H.init_model("gcn", dims, seed=3, lr=0.1, dtype=np.float32)
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, cache="on")
        losses = [H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss for _ in range(2)]
        out[flag] = (losses, [w.copy() for w in model.weights],
                     [np.array(x) for x in host.h[1:]], [np.array(g) for g in host.grad_h],
                     {l: np.array(host.agg[l]) for l in range(2)})
        fleet.close()
    a, b = out["1"], out[None]
    np.testing.assert_allclose(a[0], b[0], rtol=1e-5)
    for x, y in zip(a[1] + a[2] + a[3], b[1] + b[2] + b[3]):
        assert np.abs(x - y).max() <= 1e-4 * max(np.abs(x).max(), 1e-30)
    # lean epochs (no grad_h^0) on the project-first path: layer 0's dW
    # still comes from the A^T gz rows - parameters bitwise the same
    model = H.init_model("gcn", dims, seed=3, lr=0.1, dtype=np.float32)
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, cache="on", lean=True)
    lean_losses = [H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss for _ in range(2)]
    fleet.close()
    assert lean_losses == b[0]
    for x, y in zip(model.weights, b[1]):
        np.testing.assert_array_equal(x, y)
    # agg^0 = A.h^0 reads the same features: bitwise; agg^1 aggregates h^1,
    # which the two paths produce with different roundings
    np.testing.assert_array_equal(a[4][0], b[4][0])
    assert np.abs(a[4][1] - b[4][1]).max() <= 1e-4 * np.abs(b[4][1]).max()


@pytest.mark.parametrize("wider", [False, True])
def test_checkpoints_of_two_stores_on_one_fleet(wider):
    """Store A trains, then store B (other features, possibly a wider model)
    trains on the same fleet: A's HBM-held checkpoints are copied out before
    B's epoch overwrites the mirrors, so A.agg reads A's own epoch (the
    reference keeps agg per store, devices.py:391-404) - checked against A
    run alone with the checkpoints written through."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=2000, avg_degree=8.0, seed=6), 16, 8)
    p = H.split_chunks(ds.graph, H.partition_vertices(ds.graph, 1, seed=6), 1)
    plan = H.plan_for_partition(p)
    dims_a = [16, 24, 8]
    dims_b = [16, 40, 8] if wider else dims_a

    def store(dims, X):
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
        host.set_features(X)
        return host

    # A alone, written-through checkpoints
    ref = store(dims_a, ds.features)
    f0 = H.DeviceFleet(plan, mode="full", dtype=np.float32, cache="on", checkpoints="host")
    H.train_epoch(p, f0, H.init_model("gcn", dims_a, seed=3, dtype=np.float32), ref,
                  ds.labels, ds.mask)
    want = [np.array(ref.agg[l]) for l in range(2)]
    f0.close()
    # A then B on one fleet with HBM-held checkpoints
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, cache="on")
    host_a = store(dims_a, ds.features)
    H.train_epoch(p, fleet, H.init_model("gcn", dims_a, seed=3, dtype=np.float32), host_a,
                  ds.labels, ds.mask)
    assert host_a.agg.pending
    host_b = store(dims_b, np.asarray(ds.features) * 2.0 + 1.0)
    H.train_epoch(p, fleet, H.init_model("gcn", dims_b, seed=4, dtype=np.float32), host_b,
                  ds.labels, ds.mask)
    assert not host_a.agg.pending
    for l in range(2):
        np.testing.assert_array_equal(np.array(host_a.agg[l]), want[l])
    fleet.close()


def test_loss_label_and_mask_validation():
    """Labels / mask follow the reference's numpy indexing (engine.py:308-315):
    wrong lengths and masked labels outside [-d, d) raise IndexError;
    negative labels index from the end."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=1500, avg_degree=6.0, seed=2), 16, 4)
    p = H.split_chunks(ds.graph, H.partition_vertices(ds.graph, 1, seed=2), 1)
    plan = H.plan_for_partition(p)
    dims = [16, 12, 4]
    V = ds.graph.num_vertices

    def run(labels, mask):
        host = H.HostStore(V, dims, dtype=np.float32)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32)
        try:
            return H.train_epoch(p, fleet, H.init_model("gcn", dims, seed=1, dtype=np.float32),
                                 host, labels, mask).loss
        finally:
            fleet.close()

    y = np.asarray(ds.labels).copy()
    mask = np.asarray(ds.mask)
    with pytest.raises(IndexError):
        run(y[:-1], mask)
    with pytest.raises(IndexError):
        run(y, mask[:-1])
    bad = y.copy()
    bad[np.flatnonzero(mask)[0]] = dims[-1]
    with pytest.raises(IndexError):
        run(bad, mask)
    bad[np.flatnonzero(mask)[0]] = -dims[-1] - 1
    with pytest.raises(IndexError):
        run(bad, mask)
    ok = y.copy()
    ok[~mask] = 99  # unmasked labels are never read
    neg = y - dims[-1]  # every label as its negative alias
    assert run(ok, mask) == run(y, mask) == run(neg, mask)


@pytest.mark.parametrize("n", [1, 3])
@pytest.mark.parametrize("ck", ["auto", "host"])
def test_recompute_hybrid_under_budget(n, ck, monkeypatch):
    """Recompute-cache hybrid: under an HBM budget that
    holds the h / grad mirrors but not every agg mirror, the agg^l that do
    not fit are re-aggregated in the backward from the h^l mirror.  The
    forward gather is deterministic, so the epochs equal the all-cached
    epoch and the cache-off (host staging) epoch bitwise - weights, loss,
    every host array including host.agg (re-aggregated when read)."""
    monkeypatch.setenv("HT_NO_NARROW_BWD", "1")     # compare like with like with
    monkeypatch.setenv("HT_NO_PROJECT_FIRST", "1")  # the host-staging path
    V = 3000
    ds = H.synth_dataset(H.SynthSpec(num_vertices=V, avg_degree=8.0, seed=9), 64, 8)
    p = H.split_chunks(ds.graph, H.partition_vertices(ds.graph, 1, seed=9), n)
    dims = [64, 32, 128, 8]
    mirrors = 4 * V * (sum(dims[:-1]) + sum(dims))  # h + grad mirrors
    if n == 1:
        mirrors += 2 * 4 * V * 32  # the project-first buffers are reserved for one batch
    slack = 64 * 1024  # < 4 V (the next width step) bytes
    budgets = {"all": None,
               "one": (mirrors + 4 * V * (32 + 128) + slack) / 2 ** 30,  # keep agg^1, scratch 128
               "none": (mirrors + 4 * V * 128 + slack) / 2 ** 30,        # scratch only
               "off": None}
    res = {}
    for key, b in budgets.items():
        res[key] = _epochs_budget(p, ds, dims, "off" if key == "off" else "on", b, ck)
    assert res["all"][3] == [] and res["off"][2] is False
    assert res["one"][3] == [0, 2], res["one"][3]
    assert res["none"][3] == [0, 1, 2], res["none"][3]
    for key in ("all", "one", "none"):
        a, b = res["off"][0], res[key][0]
        assert a["loss"] == b["loss"], key
        for name in ("W", "h", "gh"):
            for x, y in zip(a[name], b[name]):
                np.testing.assert_array_equal(x, y, err_msg=f"{key} {name}")
        for l in a["agg"]:
            np.testing.assert_array_equal(a["agg"][l], b["agg"][l], err_msg=f"{key} agg{l}")


def _epochs_budget(p, ds, dims, cache, budget, ck, epochs=2):
    plan = H.plan_for_partition(p)
    model = H.init_model("gcn", dims, seed=3, lr=0.1, dtype=np.float32)
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, cache=cache, hbm_budget_gb=budget,
                          checkpoints=ck)
    for _ in range(epochs):
        r = H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    snap = {"loss": r.loss, "W": [w.copy() for w in model.weights],
            "h": [np.array(x) for x in host.h], "gh": [np.array(x) for x in host.grad_h],
            "agg": {l: np.array(host.agg[l]) for l in range(len(dims) - 1)}}
    out = (snap, fleet.recompute_layers, fleet.cache_active, list(fleet.recompute_layers))
    fleet.close()
    return out


def test_budget_too_small_for_the_mirrors():
    """A budget below the h / grad mirrors: "auto" falls back to host
    staging, "on" refuses."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=2000, avg_degree=8.0, seed=9), 16, 8)
    p = H.split_chunks(ds.graph, H.partition_vertices(ds.graph, 1, seed=9), 1)
    plan = H.plan_for_partition(p)
    dims = [16, 24, 8]
    for cache in ("auto", "on"):
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, dtype=np.float32, cache=cache, hbm_budget_gb=1e-6)
        model = H.init_model("gcn", dims, seed=3, dtype=np.float32)
        if cache == "auto":
            H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
            assert not fleet.cache_active and fleet.recompute_layers == []
        else:
            with pytest.raises(H.ChunktrainError, match="recompute"):
                H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
        fleet.close()


@pytest.mark.parametrize("placement,cache", [("host", "on"), ("device", "off")])
def test_mask_fold_bitwise(placement, cache, monkeypatch):
    """The ReLU'-mask folded into the backward's gz . W^T GEMM (g and h tiles
    by TMA, gz written from the masked stage; ht_gcn.cu) against the separate
    masking pass (HT_NO_MASK_FOLD=1): the same TF32-rounded gz feeds both
    GEMMs, so two epochs are bitwise equal - loss, weights, h, grad_h.  Both
    layouts of h^{l+1} in HBM: the owner-cache mirror and an HBM store."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=3000, avg_degree=9.0, seed=9), 16, 8)
    p = H.split_chunks(ds.graph, H.partition_vertices(ds.graph, 1, seed=9), 1)
    plan = H.plan_for_partition(p)
    dims = [16, 32, 32, 8]  # layers 0 / 1 run gz . W^T; layer 2 is narrow
    out = {}
    for flag in ("1", None):
        if flag:
            monkeypatch.setenv("HT_NO_MASK_FOLD", flag)
        else:
            monkeypatch.delenv("HT_NO_MASK_FOLD", raising=False)
        model = H.init_model("gcn", dims, seed=5, lr=0.1, dtype=np.float32)
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32, placement=placement)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, cache=cache)
        losses = [H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss for _ in range(2)]
        out[flag] = (losses, [w.copy() for w in model.weights],
                     [np.array(x) for x in host.h[1:]], [np.array(g) for g in host.grad_h])
        fleet.close()
    a, b = out["1"], out[None]
    assert a[0] == b[0]
    for x, y in zip(a[1] + a[2] + a[3], b[1] + b[2] + b[3]):
        np.testing.assert_array_equal(x, y)
