"""Pin the CPU oracle to the reference: every golden vector written by
tests/golden/make_golden.py (which ran the unmodified reference package)
must be reproduced by oracle/hongtu_oracle.py."""

import numpy as np
import pytest

from conftest import TOY_EDGES, TOY_OWNER, TOY_RANGES, random_set_instances
from digest import chunk_digest, plan_digest
from oracle import hongtu_oracle as O


def _toy_graph():
    src = np.array([e[0] for e in TOY_EDGES])
    dst = np.array([e[1] for e in TOY_EDGES])
    return O.build_graph(src, dst, 8)


def _toy_grid(g):
    grid = []
    for i, row in enumerate(TOY_RANGES):
        mine = np.flatnonzero(TOY_OWNER == i)
        grid.append([O.chunk_of(g, mine[a:b], i, j) for j, (a, b) in enumerate(row)])
    return grid


def _digest(pl):
    return plan_digest(pl["m"], pl["n"], pl["N"], pl["U"], pl["T"], pl["carry"],
                       pl["load"], pl["fetch"], pl["nbr_carry"], pl["live"],
                       pl["slots"], pl["caps"], pl["volumes"])


def test_toy_graph_arrays(golden_toy):
    g = _toy_graph()
    for k, v in golden_toy["graph"].items():
        np.testing.assert_array_equal(g[k], v)
    np.testing.assert_array_equal(g["edge_weights"], golden_toy["weights"])
    assert O.graph_hash(g) == golden_toy["hash"]


def test_toy_plan_sets_slots_volumes(golden_toy):
    g = _toy_graph()
    grid = _toy_grid(g)
    pl = O.plan_of_grid(grid, TOY_OWNER)
    gt = golden_toy
    for key in ("N", "T", "carry", "load", "nbr_carry", "live", "slots"):
        for i in range(3):
            for j in range(2):
                np.testing.assert_array_equal(pl[key][i][j], gt[key][i][j], err_msg=key)
    for j in range(2):
        np.testing.assert_array_equal(pl["U"][j], gt["U"][j])
    for i in range(3):
        for j in range(2):
            assert {str(k): list(v) for k, v in pl["fetch"][i][j].items()} == gt["fetch"][i][j]
    assert pl["caps"] == gt["caps"] == [4, 4, 3]
    assert list(pl["volumes"]) == gt["volumes"] == [19, 11, 8]
    assert O.transfer_cost(pl["volumes"]) == pytest.approx(gt["cost"], abs=0, rel=0)
    assert _digest(pl) == gt["digest"]
    assert chunk_digest(grid) == gt["chunk_digest"]
    for mode, pred in gt["predicted"].items():
        assert O.expected_rows(pl, mode) == pred
        # the reference's own meters equal its predictions for one sweep
        sw = gt["sweeps"][mode]
        assert sw["consistent"]
        assert sw["totals"]["h2d_rows"] == pred["fwd_h2d_rows"]
        assert sw["totals"]["d2h_rows"] == pred["bwd_d2h_rows"]
    assert gt["sweep_every_batch"]["totals"]["d2h_rows"] == 11


def test_toy_reorganize(golden_toy):
    g = _toy_graph()
    _, orders, batch = O.reorganize_grid(_toy_grid(g))
    assert orders == golden_toy["reorg"]["chunk_orders"]
    assert batch == golden_toy["reorg"]["batch_order"]


def _small_graph(arr, shuffle_seed=None):
    off = arr["g_csc_offsets"].astype(np.int64)
    src = arr["g_csc_sources"].astype(np.int64)
    dst = np.repeat(np.arange(off.size - 1), np.diff(off))
    if shuffle_seed is not None:
        p = np.random.default_rng(shuffle_seed).permutation(src.size)
        src, dst = src[p], dst[p]
    return O.build_graph(src, dst, off.size - 1)


def test_small_graph_rebuilt_from_shuffled_edges(golden_small):
    meta, arr = golden_small
    g = _small_graph(arr, shuffle_seed=1)
    assert O.graph_hash(g) == meta["hash"]
    for k in ("csc_offsets", "csc_sources", "csr_offsets", "csr_targets"):
        np.testing.assert_array_equal(g[k], arr["g_" + k])
    np.testing.assert_array_equal(g["edge_weights"], arr["g_weights"])


def test_small_ldg_partition_bit_exact(golden_small):
    meta, arr = golden_small
    g = _small_graph(arr)
    for m in (1, 2, 3, 4):
        own = O.ldg_partition(g, m, eps=0.1, seed=7)
        np.testing.assert_array_equal(own, arr[f"owner_m{m}"], err_msg=f"m={m}")


def _small_grid(meta, arr):
    g = _small_graph(arr)
    owner = arr["owner_m3"].astype(np.int64)
    return g, owner, O.chunk_grid(g, owner, 3, 4)


def test_small_chunks_plan_reorg(golden_small):
    meta, arr = golden_small
    g, owner, grid = _small_grid(meta, arr)
    indeg = np.diff(g["csc_offsets"])
    for i in range(3):
        cuts = O.balanced_cuts(indeg[np.flatnonzero(owner == i)], 4)
        assert [list(c) for c in cuts] == meta["ranges_m3n4"][i]
    assert chunk_digest(grid) == meta["chunk_digest_m3n4"]
    pl = O.plan_of_grid(grid, owner)
    assert _digest(pl) == meta["plan_digest_identity"]
    assert list(pl["volumes"]) == meta["volumes_identity"]
    new_grid, orders, batch = O.reorganize_grid(grid)
    assert orders == meta["reorg"]["chunk_orders"]
    assert batch == meta["reorg"]["batch_order"]
    _, orders2, batch2 = O.reorganize_grid(grid, move_all_rows=False)
    assert orders2 == meta["reorg_fixed_row0"]["chunk_orders"]
    assert batch2 == meta["reorg_fixed_row0"]["batch_order"]
    pr = O.plan_of_grid(new_grid, owner)
    assert _digest(pr) == meta["plan_digest_reorg"]
    assert pr["caps"] == meta["caps_reorg"]
    for mode, pred in meta["predicted_reorg"].items():
        assert O.expected_rows(pr, mode) == pred


@pytest.mark.parametrize("tag,dtype", [("f64", np.float64), ("f32", np.float32)])
@pytest.mark.parametrize("mode", ["baseline", "p2p", "full"])
def test_small_partitioned_epochs(golden_small, tag, dtype, mode):
    meta, arr = golden_small
    g, owner, grid = _small_grid(meta, arr)
    grid, _, _ = O.reorganize_grid(grid)
    pl = O.plan_of_grid(grid, owner)
    W = O.glorot_weights(meta["dims"], 5, dtype=dtype)
    run = meta["runs"][f"{tag}_{mode}"]
    tot = None
    losses = []
    for e in range(2):
        res = O.partitioned_epoch(grid, pl, W, arr["X"], arr["labels"], arr["mask"],
                                  mode=mode, dtype=dtype)
        W = res["weights"]
        losses.append(res["loss"])
        tot = res["meters"] if tot is None else [
            {k: a[k] + b[k] for k in a} for a, b in zip(tot, res["meters"])]
        if e == 0 and mode == "full":
            # forward is bitwise: same sequential aggregation, same BLAS
            np.testing.assert_array_equal(res["agg"][0], arr[f"{tag}_agg0_e0"])
            np.testing.assert_array_equal(res["h"][-1], arr[f"{tag}_hL_e0"])
            tol = 1e-12 if dtype == np.float64 else 2e-6
            assert O.rel_err(res["grad_h"][0], arr[f"{tag}_gh0_e0"]) < tol
            assert O.rel_err(res["grad_h"][1], arr[f"{tag}_gh1_e0"]) < tol
            for l in range(2):
                assert O.rel_err(W[l], arr[f"{tag}_W{l}_after1"]) < tol
    tol = 1e-12 if dtype == np.float64 else 1e-6
    np.testing.assert_allclose(losses, run["losses"], rtol=tol)
    totals = {k: sum(d[k] for d in tot) for k in O.METER_KEYS}
    assert totals == run["totals"]
    assert res["peaks"] == run["peaks"]


def test_small_monolithic_oracle(golden_small):
    meta, arr = golden_small
    g = _small_graph(arr)
    W = O.glorot_weights(meta["dims"], 5)
    losses = []
    for _ in range(2):
        loss, W, _ = O.monolithic_epoch(g, W, arr["X"], arr["labels"], arr["mask"])
        losses.append(loss)
    np.testing.assert_allclose(losses, meta["mono_losses"], rtol=1e-12)
    for l in range(2):
        assert O.rel_err(W[l], arr[f"mono_W{l}_after2"]) < 1e-12


def test_set_instances_plan_digests(golden_sets):
    inst = random_set_instances()
    assert len(inst) == len(golden_sets)
    for (nbrs, owner), gold in zip(inst, golden_sets):
        pl = O.dedup_plan(nbrs, owner)
        assert _digest(pl) == gold["digest"]
        for mode, pred in gold["predicted"].items():
            assert O.expected_rows(pl, mode) == pred


# ---------------------------------------------------------------------------
# GAT: kernel vectors and 2-epoch runs of the reference
# ---------------------------------------------------------------------------


def _gat_grid(golden_small):
    meta, arr = golden_small
    g, owner, grid = _small_grid(meta, arr)
    grid, _, _ = O.reorganize_grid(grid)
    return arr, owner, grid


def test_gat_chunk_kernels(golden_small, golden_gat):
    meta, ga = golden_gat
    arr, owner, grid = _gat_grid(golden_small)
    i, j = meta["kernel_chunk"]
    ch = grid[i][j]
    h, st = O.gat_chunk_forward(ch, ga["k_h_nbr"], ga["k_h_dst"], ga["k_W"], ga["k_a"])
    # the reference's softmax denominator uses reduceat (numpy-internal
    # association): tolerance, not bitwise
    assert O.rel_err(h, ga["k_h"]) < 1e-13
    assert O.rel_err(st["alpha"], ga["k_alpha"]) < 1e-13
    np.testing.assert_array_equal(st["t"], ga["k_t"])
    out = O.gat_chunk_backward(ch, ga["k_h_nbr"], ga["k_h_dst"], ga["k_R"], ga["k_W"], ga["k_a"])
    for k, v in zip(("g_nbr", "g_dst", "g_W", "g_a"), out):
        assert O.rel_err(v, ga["k_" + k]) < 1e-12, k


def test_gat_single_edge_and_empty_destination():
    """Known answers of the reference's tests (tests/test_engine.py:181-222):
    one in-edge => alpha 1, h = ReLU(h_nbr W), zero attention gradient; a
    destination without in-edges gets a zero row and finite gradients."""
    rng = np.random.default_rng(3)
    ch = {"csc_offsets": np.array([0, 1]), "csc_local_src": np.array([0])}
    hn, hd = rng.standard_normal((1, 3)), rng.standard_normal((1, 3))
    W, a = rng.standard_normal((3, 2)), rng.standard_normal(4)
    h, st = O.gat_chunk_forward(ch, hn, hd, W, a)
    np.testing.assert_array_equal(st["alpha"], [1.0])
    np.testing.assert_array_equal(h, np.maximum(hn @ W, 0.0))
    _, _, _, g_a = O.gat_chunk_backward(ch, hn, hd, rng.standard_normal((1, 2)), W, a)
    np.testing.assert_array_equal(g_a, np.zeros(4))
    ch = {"csc_offsets": np.array([0, 1, 1, 2]), "csc_local_src": np.array([0, 1])}
    hn, hd = rng.standard_normal((2, 4)), rng.standard_normal((3, 4))
    W, a = rng.standard_normal((4, 2)), rng.standard_normal(4)
    h, _ = O.gat_chunk_forward(ch, hn, hd, W, a)
    np.testing.assert_array_equal(h[1], 0.0)
    out = O.gat_chunk_backward(ch, hn, hd, rng.standard_normal(h.shape), W, a)
    assert all(np.isfinite(x).all() for x in out)


@pytest.mark.parametrize("tag,dtype", [("f64", np.float64), ("f32", np.float32)])
@pytest.mark.parametrize("mode", ["baseline", "p2p", "full"])
def test_gat_partitioned_epochs(golden_small, golden_gat, tag, dtype, mode):
    meta, ga = golden_gat
    arr, owner, grid = _gat_grid(golden_small)
    pl = O.plan_of_grid(grid, owner)
    assert _digest(pl) == meta["plan_digest_reorg"]
    W, A = O.glorot_weights(meta["dims"], 5, dtype=dtype, gat=True)
    run = meta["runs"][f"{tag}_{mode}"]
    tot, losses = None, []
    tol = 1e-12 if dtype == np.float64 else 2e-6
    for e in range(2):
        res = O.partitioned_epoch(grid, pl, W, arr["X"], arr["labels"], arr["mask"], mode=mode,
                                  dtype=dtype, kind="gat", attn=A)
        W, A = res["weights"], res["attn"]
        losses.append(res["loss"])
        tot = res["meters"] if tot is None else [
            {k: a[k] + b[k] for k in a} for a, b in zip(tot, res["meters"])]
        if e == 0 and mode == "full":
            assert O.rel_err(res["h"][-1], ga[f"{tag}_hL_e0"]) < tol
            assert O.rel_err(res["grad_h"][0], ga[f"{tag}_gh0_e0"]) < tol
            assert O.rel_err(res["grad_h"][1], ga[f"{tag}_gh1_e0"]) < tol
            for l in range(2):
                assert O.rel_err(W[l], ga[f"{tag}_W{l}_after1"]) < tol
                assert O.rel_err(A[l], ga[f"{tag}_a{l}_after1"]) < tol
    np.testing.assert_allclose(losses, run["losses"], rtol=1e-12 if dtype == np.float64 else 1e-6)
    totals = {k: sum(d[k] for d in tot) for k in O.METER_KEYS}
    assert totals == run["totals"]
    assert res["peaks"] == run["peaks"]
    if mode == "full":
        for l in range(2):
            assert O.rel_err(W[l], ga[f"{tag}_W{l}_after2"]) < tol
            assert O.rel_err(A[l], ga[f"{tag}_a{l}_after2"]) < tol


def test_gat_partitioned_matches_monolithic_reference(golden_small, golden_gat):
    """The reference's own acceptance bar (tests/test_acceptance.py:154-156):
    the partitioned fp64 GAT epoch equals the monolithic trainer."""
    meta, ga = golden_gat
    arr, owner, grid = _gat_grid(golden_small)
    pl = O.plan_of_grid(grid, owner)
    W, A = O.glorot_weights(meta["dims"], 5, dtype=np.float64, gat=True)
    losses = []
    for _ in range(2):
        res = O.partitioned_epoch(grid, pl, W, arr["X"], arr["labels"], arr["mask"],
                                  dtype=np.float64, kind="gat", attn=A)
        W, A = res["weights"], res["attn"]
        losses.append(res["loss"])
    np.testing.assert_allclose(losses, meta["mono_losses"], rtol=1e-10)
    for l in range(2):
        assert O.rel_err(W[l], ga[f"mono_W{l}_after2"]) < 1e-8
        assert O.rel_err(A[l], ga[f"mono_a{l}_after2"]) < 1e-8
