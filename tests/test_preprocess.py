"""Integer preprocessing of the package (native, CPU) is bit-exact with the
reference: graph arrays, synthetic inputs, LDG owners, chunks, plan sets
and slots, volumes, predictions and reorganization (golden vectors from
tests/golden/make_golden.py).  Runs without a GPU."""

import numpy as np
import pytest

import paper_2311_14898_b200 as H
from conftest import TOY_EDGES, TOY_OWNER, TOY_RANGES, load_json, random_set_instances
from digest import chunk_digest, plan_digest


def _digest(plan):
    return plan_digest(plan.m, plan.n, plan.neighbor_sets, plan.union_sets, plan.owned_sets,
                       plan.carry_sets, plan.load_sets, plan.fetch_sets, plan.nbr_carry_sets,
                       plan.layout.live_sets, plan.layout.slots, plan.layout.capacities,
                       (plan.volumes.v_ori, plan.volumes.v_p2p, plan.volumes.v_ru))


def _toy():
    src = np.array([e[0] for e in TOY_EDGES])
    dst = np.array([e[1] for e in TOY_EDGES])
    g = H.from_edges(src, dst, num_vertices=8)
    a = H.PartitionAssignment(owner=TOY_OWNER.copy(), m=3)
    return g, H.two_level_from_ranges(g, a, TOY_RANGES)


def test_toy_graph_plan(golden_toy):
    g, p = _toy()
    for k, v in golden_toy["graph"].items():
        np.testing.assert_array_equal(getattr(g, k), v)
    np.testing.assert_array_equal(g.edge_weights, golden_toy["weights"])
    np.testing.assert_array_equal(H.gcn_edge_weights(g), golden_toy["weights"])
    assert g.content_hash() == golden_toy["hash"]
    assert chunk_digest(p.chunks) == golden_toy["chunk_digest"]
    plan = H.plan_for_partition(p)
    assert _digest(plan) == golden_toy["digest"]
    assert plan.layout.capacities == [4, 4, 3]
    assert (plan.volumes.v_ori, plan.volumes.v_p2p, plan.volumes.v_ru) == (19, 11, 8)
    assert H.comm_cost(plan.volumes, H.CostParams()) == golden_toy["cost"]
    assert H.replication_factor(p) == golden_toy["alpha"] == 2.375
    for mode, pred in golden_toy["predicted"].items():
        assert H.predicted_transfers(plan, mode) == pred
    # slot maps as dicts (reference BufferLayout.slot_maps)
    for i in range(3):
        for j in range(2):
            sm = plan.layout.slot_maps[i][j]
            assert [sm[v] for v in golden_toy["live"][i][j]] == golden_toy["slots"][i][j]
    r = H.reorganize(p)
    assert r.chunk_orders == golden_toy["reorg"]["chunk_orders"]
    assert r.batch_order == golden_toy["reorg"]["batch_order"]


def test_small_synth_graph_and_node_data(golden_small):
    meta, arr = golden_small
    s = meta["synth"]
    ds = H.synth_dataset(H.SynthSpec(num_vertices=s["num_vertices"], avg_degree=s["avg_degree"],
                                     seed=s["seed"]), s["feature_dim"], s["num_classes"])
    assert ds.graph.content_hash() == meta["hash"]
    for k in ("csc_offsets", "csc_sources", "csr_offsets", "csr_targets", "csr_edge_perm"):
        np.testing.assert_array_equal(getattr(ds.graph, k), arr["g_" + k])
    np.testing.assert_array_equal(ds.graph.edge_weights, arr["g_weights"])
    np.testing.assert_array_equal(ds.features, arr["X"])
    np.testing.assert_array_equal(ds.labels, arr["labels"])
    np.testing.assert_array_equal(ds.mask, arr["mask"])


def _small_graph(arr, shuffle=None):
    off = arr["g_csc_offsets"].astype(np.int64)
    src = arr["g_csc_sources"].astype(np.int64)
    dst = np.repeat(np.arange(off.size - 1), np.diff(off))
    if shuffle is not None:
        p = np.random.default_rng(shuffle).permutation(src.size)
        src, dst = src[p], dst[p]
    return H.from_edges(src, dst, num_vertices=off.size - 1)


def test_graph_from_shuffled_edges(golden_small):
    meta, arr = golden_small
    g = _small_graph(arr, shuffle=4)
    assert g.content_hash() == meta["hash"]
    np.testing.assert_array_equal(g.csr_edge_perm, arr["g_csr_edge_perm"])


def test_duplicate_edges_keep_reference_order():
    # parallel edges and self loops are kept; stable order on ties
    src = np.array([3, 1, 3, 0, 3, 2, 2])
    dst = np.array([0, 0, 0, 2, 2, 2, 2])
    g = H.from_edges(src, dst, 4)
    np.testing.assert_array_equal(g.csc_sources, [1, 3, 3, 0, 2, 2, 3])
    order = np.lexsort((src, dst))
    np.testing.assert_array_equal(g.csc_sources, src[order])
    order_csr = np.lexsort((dst, src))
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    np.testing.assert_array_equal(g.csr_edge_perm, inv[order_csr])


def test_ldg_partition_bit_exact(golden_small):
    meta, arr = golden_small
    g = _small_graph(arr)
    for m in (1, 2, 3, 4):
        a = H.partition_vertices(g, m, epsilon=0.1, seed=7)
        np.testing.assert_array_equal(a.owner, arr[f"owner_m{m}"], err_msg=f"m={m}")
    assert H.edge_cut(g, H.PartitionAssignment(owner=arr["owner_m3"].astype(np.int64), m=3)) == \
        meta["edge_cut_m3"]


def test_chunks_plan_reorganize(golden_small):
    meta, arr = golden_small
    g = _small_graph(arr)
    a = H.PartitionAssignment(owner=arr["owner_m3"].astype(np.int64), m=3)
    p = H.split_chunks(g, a, 4)
    assert chunk_digest(p.chunks) == meta["chunk_digest_m3n4"]
    plan = H.plan_for_partition(p)
    assert _digest(plan) == meta["plan_digest_identity"]
    r = H.reorganize(p)
    assert r.chunk_orders == meta["reorg"]["chunk_orders"]
    assert r.batch_order == meta["reorg"]["batch_order"]
    r2 = H.reorganize(p, move_all_rows=False)
    assert r2.chunk_orders == meta["reorg_fixed_row0"]["chunk_orders"]
    assert r2.batch_order == meta["reorg_fixed_row0"]["batch_order"]
    plan_r = H.plan_for_partition(r.partition)
    assert _digest(plan_r) == meta["plan_digest_reorg"]
    assert plan_r.layout.capacities == meta["caps_reorg"]
    for mode, pred in meta["predicted_reorg"].items():
        assert H.predicted_transfers(plan_r, mode) == pred


def test_random_set_instances(golden_sets):
    for (nbrs, owner), gold in zip(random_set_instances(), golden_sets):
        plan = H.build_plan(nbrs, owner)
        assert _digest(plan) == gold["digest"]
        for mode, pred in gold["predicted"].items():
            assert H.predicted_transfers(plan, mode) == pred


def test_errors_match_reference_contract():
    with pytest.raises(H.GraphParseError):
        H.from_edges(np.array([0, 1]), np.array([1]))
    with pytest.raises(H.GraphParseError):
        H.from_edges(np.array([0, 5]), np.array([1, 1]), num_vertices=3)
    g, p = _toy()
    with pytest.raises(H.PartitionError):
        H.partition_vertices(g, 0)
    with pytest.raises(H.PartitionError):
        H.split_chunks(g, p.assignment, 5)
    with pytest.raises(H.PlanError):
        H.build_plan([[np.array([9])]], np.zeros(3, dtype=np.int64))
    with pytest.raises(H.PlanError, match="positive"):
        H.comm_cost(H.Volumes(1, 1, 1), H.CostParams(t_hd=0.0))
    with pytest.raises(H.PlanError, match="unknown mode"):
        H.predicted_transfers(H.plan_for_partition(p), "warp")


def test_graph_cache_round_trip(tmp_path, golden_small):
    meta, arr = golden_small
    g = _small_graph(arr)
    path = str(tmp_path / "g.htg")
    H.save_graph_cache(g, path)
    g2 = H.load_graph_cache(path)
    assert g2.content_hash() == g.content_hash()
    np.testing.assert_array_equal(g2.csr_edge_perm, g.csr_edge_perm)
    np.testing.assert_array_equal(g2.edge_weights, g.edge_weights)
    with open(path, "ab") as fh:
        fh.write(b"x")
    with pytest.raises(H.GraphFormatError):
        H.load_graph_cache(path)


@pytest.mark.slow
def test_cfg1_preprocessing_matches_reference():
    """BASELINE config 1: graph hash, LDG owner hash, chunks, reorganized plan."""
    gold = load_json("cfg1.json")
    ds = H.synth_dataset(H.SynthSpec(num_vertices=100_000, avg_degree=20.0, seed=0), 64, 16)
    g = ds.graph
    assert g.content_hash() == gold["hash"]
    a = H.partition_vertices(g, 4, seed=0)
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(a.owner).tobytes()).hexdigest() == gold["owner_sha"]
    p = H.split_chunks(g, a, 4)
    assert chunk_digest(p.chunks) == gold["chunk_digest"]
    r = H.reorganize(p)
    assert r.batch_order == gold["batch_order"]
    assert r.chunk_orders == gold["chunk_orders"]
    plan = H.plan_for_partition(r.partition)
    assert _digest(plan) == gold["plan_digest_reorg"]
    assert plan.layout.capacities == gold["caps"]


def test_graph_cache_mmap_and_duplicate_edges(tmp_path):
    """HTG1 memory-mapped load with the native CSR permutation equals the
    lexsort of the reference (graph.py:262-264) - incl. duplicate edges and
    self loops, where tie order matters - and the private-copy load."""
    rng = np.random.default_rng(4)
    V = 500
    src = rng.integers(0, V, 4000)
    dst = rng.integers(0, V, 4000)
    src = np.concatenate([src, src[:300], np.arange(20)])   # duplicates + self loops
    dst = np.concatenate([dst, dst[:300], np.arange(20)])
    g = H.from_edges(src, dst, V)
    path = str(tmp_path / "g.htg")
    H.save_graph_cache(g, path)
    for mm in (True, False):
        g2 = H.load_graph_cache(path, mmap=mm)
        assert g2.content_hash() == g.content_hash()
        np.testing.assert_array_equal(g2.csr_edge_perm, g.csr_edge_perm)
        dstc = np.repeat(np.arange(V), np.diff(g.csc_offsets))
        np.testing.assert_array_equal(g2.csr_edge_perm, np.lexsort((dstc, g.csc_sources)))


def test_feature_matrix_mmap_into_host_store(tmp_path):
    rng = np.random.default_rng(5)
    X = rng.standard_normal((3000, 24))
    path = str(tmp_path / "x.htf")
    H.save_matrix(X, path)
    Xm = H.load_matrix(path, mmap=True)
    np.testing.assert_array_equal(np.asarray(Xm), X)


@pytest.mark.gpu  # pinned host memory needs the driver
def test_feature_matrix_mmap_into_pinned_host_store(tmp_path):
    rng = np.random.default_rng(5)
    X = rng.standard_normal((3000, 24))
    path = str(tmp_path / "x.htf")
    H.save_matrix(X, path)
    Xm = H.load_matrix(path, mmap=True)
    host = H.HostStore(3000, [24, 8], dtype=np.float32)
    host.set_features(Xm)
    np.testing.assert_array_equal(host.h[0], X.astype(np.float32))
    big = rng.standard_normal((200_000, 24))  # the threaded row-block cast
    hb = H.HostStore(200_000, [24, 8], dtype=np.float32)
    hb.set_features(big)
    np.testing.assert_array_equal(hb.h[0], big.astype(np.float32))


def test_bench_dedup_report_matches_reference_numbers():
    """bench.py's host-bytes accounting on config 1 against the reference's
    own measurements: m=8, n=1 volumes (263217, 99968,
    99968) and 422,350,848 host bytes per epoch through the 'full' plan
    (plus the loss-gradient rows and the label/mask upload this path adds)."""
    import bench
    c = bench.CONFIGS["cfg1"]
    ds = H.synth_dataset(H.SynthSpec(num_vertices=c["V"], avg_degree=c["avg_degree"], seed=0),
                         c["dims"][0], c["dims"][-1])
    r = bench.dedup_at_scale(ds, c["dims"], m=8, n=1)
    assert (r["volumes"]["v_ori"], r["volumes"]["v_p2p"], r["volumes"]["v_ru"]) == (263217, 99968, 99968)
    V, dL = c["V"], c["dims"][-1]
    assert round(r["host_gb_full"] * 1e9) == 422_350_848 + 4 * V * dL + 9 * V
    assert r["reduction"] > 0.25  # the north star's >= 25 % host-byte reduction


def test_bench_dedup_report_m4n4_matches_reference_numbers():
    """Config 1 at m=4, n=4 (reorganized): 466,520,064 host bytes through the
    'full' plan, 903,375,360 through the non-deduplicated one (SURVEY App. A
    epoch meters), plus the loss-gradient rows and label/mask upload."""
    import bench
    r = bench.dedup_report()
    extra = 4 * 100_000 * 16 + 9 * 100_000
    assert round(r["host_gb_full"] * 1e9) == 466_520_064 + extra
    assert round(r["host_gb_baseline"] * 1e9) == 903_375_360 + extra
    assert (r["volumes"]["v_ori"], r["volumes"]["v_p2p"], r["volumes"]["v_ru"]) == (413135, 319160, 128724)
