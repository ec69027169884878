"""Full GCN epochs on the GPU through the C ABI, against the reference's
golden vectors and the CPU oracle (FP32 validation mode: 1e-5 relative,
max-normalised as in the reference's tests/test_engine.py:122-124)."""

import numpy as np
import pytest

import paper_2311_14898_b200 as H
from conftest import load_json
from oracle import hongtu_oracle as O

pytestmark = pytest.mark.gpu
TOL = {"fp32": 1e-5, "tf32": 1e-3}


def _small(golden_small):
    meta, arr = golden_small
    s = meta["synth"]
    ds = H.synth_dataset(H.SynthSpec(num_vertices=s["num_vertices"], avg_degree=s["avg_degree"],
                                     seed=s["seed"]), s["feature_dim"], s["num_classes"])
    a = H.PartitionAssignment(owner=arr["owner_m3"].astype(np.int64), m=3)
    p = H.reorganize(H.split_chunks(ds.graph, a, 4)).partition
    return meta, arr, ds, p


def _run(p, ds, dims, mode="full", precision="fp32", epochs=2, seed=5, flush="on_eviction"):
    plan = H.plan_for_partition(p)
    model = H.init_model("gcn", dims, seed=seed, lr=0.1, dtype=np.float32)
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, mode=mode, dtype=np.float32, precision=precision, flush_policy=flush)
    losses, snaps = [], []
    for _ in range(epochs):
        res = H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
        losses.append(res.loss)
        snaps.append({"agg0": np.array(host.agg[0]), "hL": np.array(host.h[-1]),
                      "gh0": np.array(host.grad_h[0]), "gh1": np.array(host.grad_h[1]),
                      "W": [w.copy() for w in model.weights], "grads": res.grads})
    return losses, snaps, fleet, model


@pytest.mark.parametrize("mode", ["baseline", "p2p", "full"])
def test_small_epochs_match_reference(golden_small, mode):
    meta, arr, ds, p = _small(golden_small)
    losses, snaps, fleet, model = _run(p, ds, meta["dims"], mode=mode)
    run = meta["runs"][f"f32_{mode}"]
    np.testing.assert_allclose(losses, run["losses"], rtol=1e-5)
    # the golden ran two epochs: two communication sweeps per layer
    rep = fleet.transfer_report(*(2 * x for x in H.comm_passes_per_epoch(model)))
    assert rep["totals"] == run["totals"]
    assert rep["peak_live_slots"] == run["peaks"]
    assert rep["planner_consistent"]
    if mode == "full":
        # forward aggregation is sequential multiply-then-add: bitwise
        np.testing.assert_array_equal(snaps[0]["agg0"], arr["f32_agg0_e0"])
        assert O.rel_err(snaps[0]["hL"], arr["f32_hL_e0"]) < 1e-5
        assert O.rel_err(snaps[0]["gh0"], arr["f32_gh0_e0"]) < 1e-5
        assert O.rel_err(snaps[0]["gh1"], arr["f32_gh1_e0"]) < 1e-5
        for l in range(2):
            assert O.rel_err(snaps[0]["W"][l], arr[f"f32_W{l}_after1"]) < 1e-5
            assert O.rel_err(snaps[1]["W"][l], arr[f"f32_W{l}_after2"]) < 1e-5


@pytest.mark.parametrize("m,n", [(1, 1), (2, 3), (4, 2)])
def test_epoch_matches_oracle_grads(m, n):
    ds = H.synth_dataset(H.SynthSpec(num_vertices=3000, avg_degree=7.0, seed=11), 20, 5)
    a = H.partition_vertices(ds.graph, m, seed=11)
    p = H.split_chunks(ds.graph, a, n)
    dims = [20, 32, 5]
    w0 = H.init_model("gcn", dims, seed=2, dtype=np.float32).weights
    losses, snaps, _, _ = _run(p, ds, dims, epochs=1, seed=2)
    grid = [[vars(c) for c in row] for row in p.chunks]
    ref = O.partitioned_epoch(grid, O.plan_of_grid(grid, a.owner), [w.copy() for w in w0],
                              ds.features, ds.labels, ds.mask, dtype=np.float32)
    assert abs(losses[0] - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    for l in range(2):
        assert O.rel_err(snaps[0]["grads"][l], ref["grads"][l]) < 1e-5
        assert O.rel_err(snaps[0]["W"][l], ref["weights"][l]) < 1e-5
    assert O.rel_err(snaps[0]["gh0"], ref["grad_h"][0]) < 1e-5
    np.testing.assert_array_equal(snaps[0]["agg0"], ref["agg"][0])


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_long_segments_split_path(precision):
    """A hub source and a hub destination with thousands of edges (> the 1024-edge piece length)
    in-edges exercise the piece + fixup kernels in both directions (one device, one batch:
    the expanded CSR; in TF32 the narrow last layer also runs project-first)."""
    rng = np.random.default_rng(9)
    V = 12000
    src = np.concatenate([np.zeros(9000, np.int64), rng.integers(0, V, 30000),
                          rng.integers(0, V, 6000)])
    dst = np.concatenate([rng.integers(0, V, 9000), rng.integers(0, V, 30000),
                          np.full(6000, 5, np.int64)])
    g = H.from_edges(src, dst, V)
    X = rng.standard_normal((V, 12))
    labels = rng.integers(0, 3, V)
    mask = rng.random(V) < 0.5
    a = H.PartitionAssignment(owner=np.zeros(V, np.int64), m=1)
    p = H.split_chunks(g, a, 1)
    ds = H.SynthDataset(graph=g, features=X, labels=labels, mask=mask)
    dims = [12, 16, 3]
    w0 = H.init_model("gcn", dims, seed=4, dtype=np.float32).weights
    losses, snaps, _, _ = _run(p, ds, dims, epochs=1, seed=4, precision=precision)
    grid = [[vars(c) for c in row] for row in p.chunks]
    tol = TOL[precision]
    ref = O.partitioned_epoch(grid, O.plan_of_grid(grid, a.owner),
                              [w.astype(np.float64) for w in w0], X, labels, mask,
                              dtype=np.float32 if precision == "fp32" else np.float64)
    assert abs(losses[0] - ref["loss"]) <= tol * abs(ref["loss"])
    assert O.rel_err(snaps[0]["agg0"], ref["agg"][0]) < 1e-5  # hub pieces reassociate
    assert O.rel_err(snaps[0]["gh0"], ref["grad_h"][0]) < tol
    for l in range(2):
        assert O.rel_err(snaps[0]["grads"][l], ref["grads"][l]) < tol


def test_train_epoch_errors(golden_small):
    meta, arr, ds, p = _small(golden_small)
    dims = meta["dims"]
    plan = H.plan_for_partition(p)
    model = H.init_model("gcn", dims, seed=5, dtype=np.float32)
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
    fleet = H.DeviceFleet(plan, dtype=np.float32)
    with pytest.raises(H.SimulationError, match="features"):
        H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    host.set_features(ds.features)
    with pytest.warns(UserWarning, match="empty"):
        res = H.train_epoch(p, fleet, model, host, ds.labels, np.zeros_like(ds.mask))
    assert res.loss == 0.0


@pytest.mark.slow
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_cfg1_two_epochs_match_reference(precision):
    """BASELINE config 1 (100K V / 1.87M E, 64-128-16, m=4, n=4, reorganized):
    loss and weights after each of two epochs within the north-star
    tolerance of the precision mode (FP32 1e-5, TF32 1e-3)."""
    gold = load_json("cfg1.json")
    arr = dict(np.load(__import__("os").path.join(__import__("conftest").GOLDEN, "cfg1.npz")))
    ds = H.synth_dataset(H.SynthSpec(num_vertices=100_000, avg_degree=20.0, seed=0), 64, 16)
    a = H.partition_vertices(ds.graph, 4, seed=0)
    p = H.reorganize(H.split_chunks(ds.graph, a, 4)).partition
    losses, snaps, fleet, model = _run(p, ds, [64, 128, 16], epochs=2, seed=0, precision=precision)
    tol = TOL[precision]
    np.testing.assert_allclose(losses, gold["losses_f32"], rtol=tol)
    for l in range(2):
        assert O.rel_err(snaps[0]["W"][l], arr[f"W{l}_after1"]) < tol
        assert O.rel_err(snaps[1]["W"][l], arr[f"W{l}_after2"]) < tol
    assert fleet.transfer_report()["totals"] == gold["totals_f32"]


@pytest.mark.parametrize("m,n", [(1, 1), (3, 2)])
def test_tf32_epoch_within_north_star_tolerance(m, n):
    """TF32 mode (tcgen05; 3xTF32 for z = agg.W): logits, loss and weight
    gradients within 1e-3 of the fp64 oracle (north star tolerance)."""
    ds = H.synth_dataset(H.SynthSpec(num_vertices=4000, avg_degree=9.0, seed=21), 64, 7)
    a = H.partition_vertices(ds.graph, m, seed=21)
    p = H.split_chunks(ds.graph, a, n)
    dims = [64, 96, 7]
    w0 = H.init_model("gcn", dims, seed=8, dtype=np.float32).weights
    losses, snaps, _, _ = _run(p, ds, dims, epochs=1, seed=8, precision="tf32")
    grid = [[vars(c) for c in row] for row in p.chunks]
    ref = O.partitioned_epoch(grid, O.plan_of_grid(grid, a.owner), [w.astype(np.float64) for w in w0],
                              ds.features, ds.labels, ds.mask, dtype=np.float64)
    assert abs(losses[0] - ref["loss"]) <= 1e-3 * abs(ref["loss"])
    assert O.rel_err(snaps[0]["hL"], ref["h"][-1]) < 1e-3
    for l in range(2):
        assert O.rel_err(snaps[0]["grads"][l], ref["grads"][l]) < 1e-3


def test_hbm_resident_store_matches_host_store(golden_small):
    """The HongTu-IM variant (vertex store in HBM, bench.py's `value`) runs
    the same kernels on device memory: identical results to the pinned
    host store, bitwise."""
    meta, arr, ds, p = _small(golden_small)
    dims = meta["dims"]
    plan = H.plan_for_partition(p)
    out = {}
    for placement in ("host", "device"):
        model = H.init_model("gcn", dims, seed=5, lr=0.1, dtype=np.float32)
        host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32, placement=placement)
        host.set_features(ds.features)
        fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32)
        losses = [H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss for _ in range(2)]
        out[placement] = (losses, [w.copy() for w in model.weights], np.asarray(host.grad_h[0]),
                          np.asarray(host.agg[1]))
    assert out["host"][0] == out["device"][0]
    for a, b in zip(out["host"][1], out["device"][1]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(out["host"][2], out["device"][2])
    np.testing.assert_array_equal(out["host"][3], out["device"][3])
