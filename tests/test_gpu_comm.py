"""Deduplicated transfer machinery on the GPU (K1/K2/K9/K10 + dest/checkpoint
rows), mirroring the reference's device tests (tests/test_devices.py):
bitwise forward views, exact scatter-add gradients, meters equal to the
planner, sequencing errors.  Runs through the C ABI on cuda:0."""

import numpy as np
import pytest

import paper_2311_14898_b200 as H
from conftest import TOY_EDGES, TOY_OWNER, TOY_RANGES, random_graph, random_set_instances, random_two_level

pytestmark = pytest.mark.gpu
DIM = 3


@pytest.fixture
def toy_plan():
    src = np.array([e[0] for e in TOY_EDGES])
    dst = np.array([e[1] for e in TOY_EDGES])
    g = H.from_edges(src, dst, num_vertices=8)
    p = H.two_level_from_ranges(g, H.PartitionAssignment(owner=TOY_OWNER.copy(), m=3), TOY_RANGES)
    return H.plan_for_partition(p)


def _host_rows(rng, V, dim=DIM, dtype=np.float64):
    return rng.standard_normal((V, dim)).astype(dtype)


def _fwd(fleet, host):
    fleet.begin_forward_layer(host.shape[1])
    return [fleet.dedup_comm_fwd(host, j) for j in range(fleet.n)]


def _bwd(fleet, rng, host_grad, dtype=np.float64):
    fleet.begin_backward_layer(host_grad.shape[1])
    fed = []
    for j in range(fleet.n):
        views = [rng.standard_normal((fleet.plan.neighbor_sets[i][j].size, host_grad.shape[1])).astype(dtype)
                 for i in range(fleet.m)]
        fed.append(views)
        fleet.dedup_comm_bwd(views, host_grad, j)
    return fed


def _scatter_oracle(plan, fed, V, dim):
    out = np.zeros((V, dim))
    for j in range(plan.n):
        for i in range(plan.m):
            nb = plan.neighbor_sets[i][j]
            if nb.size:
                out[nb] += fed[j][i]
    return out


def _random_plan(rng, with_dests=False):
    if with_dests:
        g = random_graph(rng, num_vertices=int(rng.integers(12, 40)))
        m, n = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        return H.plan_for_partition(random_two_level(g, rng, m, n)), g.num_vertices
    nbrs, owner = random_set_instances(1, seed=int(rng.integers(0, 2**31)))[0]
    return H.build_plan(nbrs, owner), owner.shape[0]


@pytest.mark.parametrize("mode,h2d", [("baseline", 19), ("p2p", 11), ("full", 8)])
def test_toy_forward_views_and_h2d(toy_plan, mode, h2d):
    rng = np.random.default_rng(0)
    host = _host_rows(rng, 8)
    fleet = H.DeviceFleet(toy_plan, mode=mode)
    views = _fwd(fleet, host)
    assert fleet.transfer_report()["totals"]["h2d_rows"] == h2d
    for j in range(fleet.n):
        for i in range(fleet.m):
            np.testing.assert_array_equal(views[j][i], host[toy_plan.neighbor_sets[i][j]])


@pytest.mark.parametrize("mode,d2h", [("baseline", 19), ("p2p", 11), ("full", 8)])
def test_toy_backward_d2h(toy_plan, mode, d2h):
    rng = np.random.default_rng(1)
    fleet = H.DeviceFleet(toy_plan, mode=mode)
    hg = np.zeros((8, DIM))
    fed = _bwd(fleet, rng, hg)
    assert fleet.transfer_report()["totals"]["d2h_rows"] == d2h
    np.testing.assert_allclose(hg, _scatter_oracle(toy_plan, fed, 8, DIM), rtol=1e-12, atol=1e-14)


def test_toy_reuse_peaks_every_batch(toy_plan):
    rng = np.random.default_rng(2)
    fleet = H.DeviceFleet(toy_plan, mode="full")
    _fwd(fleet, _host_rows(rng, 8))
    rep = fleet.transfer_report()
    assert rep["totals"]["reuse_rows"] == 3
    assert rep["peak_live_slots"] == [4, 4, 3]
    fleet = H.DeviceFleet(toy_plan, mode="full", flush_policy="every_batch")
    _bwd(fleet, rng, np.zeros((8, DIM)))
    assert fleet.transfer_report()["totals"]["d2h_rows"] == 11


@pytest.mark.parametrize("mode", H.MODES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_random_views_bitwise_and_scatter(mode, dtype):
    rng = np.random.default_rng(10)
    for _ in range(12):
        plan, V = _random_plan(rng)
        fleet = H.DeviceFleet(plan, mode=mode, dtype=dtype)
        host = _host_rows(rng, V, dtype=dtype)
        views = _fwd(fleet, host)
        for j in range(plan.n):
            for i in range(plan.m):
                np.testing.assert_array_equal(views[j][i], host[plan.neighbor_sets[i][j]])
        hg = np.zeros((V, DIM), dtype=dtype)
        fed = _bwd(fleet, rng, hg, dtype)
        tol = 1e-12 if dtype == np.float64 else 1e-6
        np.testing.assert_allclose(hg, _scatter_oracle(plan, fed, V, DIM), rtol=tol, atol=tol)
        rep = fleet.transfer_report(fwd_passes=1, bwd_passes=1)
        assert rep["planner_consistent"], rep


def _interval_instance(rng, m, n, universe):
    nbrs = [[set() for _ in range(n)] for _ in range(m)]
    for v in range(universe):
        a = int(rng.integers(0, n))
        b = int(rng.integers(a, n))
        cover = int(rng.integers(0, m))
        for j in range(a, b + 1):
            nbrs[cover][j].add(v)
            for i in range(m):
                if rng.random() < 0.3:
                    nbrs[i][j].add(v)
    owner = rng.integers(0, m, size=universe)
    return [[np.array(sorted(s), dtype=np.int64) for s in row] for row in nbrs], owner


def test_baseline_and_full_gradients_bitwise():
    rng = np.random.default_rng(30)
    for _ in range(8):
        m, n, V = int(rng.integers(1, 5)), int(rng.integers(1, 7)), int(rng.integers(8, 40))
        nbrs, owner = _interval_instance(rng, m, n, V)
        plan = H.build_plan(nbrs, owner)
        seed = int(rng.integers(0, 2**31))
        out = {}
        for mode in ("baseline", "full"):
            hg = np.zeros((V, DIM))
            _bwd(H.DeviceFleet(plan, mode=mode), np.random.default_rng(seed), hg)
            out[mode] = hg
        np.testing.assert_array_equal(out["baseline"], out["full"])


def test_watermarks_and_byte_meters():
    rng = np.random.default_rng(50)
    for _ in range(6):
        plan, V = _random_plan(rng)
        for mode in ("p2p", "full"):
            fleet = H.DeviceFleet(plan, mode=mode)
            _fwd(fleet, _host_rows(rng, V))
            _bwd(fleet, rng, np.zeros((V, DIM)))
            assert [d.peak_live_slots for d in fleet.devices] == plan.layout.capacities
            assert [fleet.capacity(i) for i in range(plan.m)] == plan.layout.capacities
    plan, V = _random_plan(rng)
    for dtype, item in ((np.float64, 8), (np.float32, 4)):
        fleet = H.DeviceFleet(plan, mode="full", dtype=dtype)
        _fwd(fleet, _host_rows(rng, V, dtype=dtype))
        t = fleet.transfer_report()["totals"]
        assert t["h2d_bytes"] == t["h2d_rows"] * DIM * item
        assert t["d2d_bytes"] == t["d2d_rows"] * DIM * item
        assert all(d.buffer.dtype == np.dtype(dtype) for d in fleet.devices)


def test_sequencing_errors(toy_plan):
    fleet = H.DeviceFleet(toy_plan, mode="full")
    host = np.zeros((8, DIM))
    with pytest.raises(H.SimulationError, match="out of order"):
        fleet.dedup_comm_fwd(host, 0)
    fleet.begin_forward_layer(DIM)
    with pytest.raises(H.SimulationError, match="out of order"):
        fleet.dedup_comm_fwd(host, 1)
    fleet.dedup_comm_fwd(host, 0)
    with pytest.raises(H.SimulationError, match="out of order"):
        fleet.dedup_comm_fwd(host, 0)
    fleet.begin_backward_layer(DIM)
    grads = [np.zeros((toy_plan.neighbor_sets[i][1].size, DIM)) for i in range(3)]
    with pytest.raises(H.SimulationError, match="out of order"):
        fleet.dedup_comm_bwd(grads, np.zeros((8, DIM)), 1)
    with pytest.raises(H.SimulationError, match="unknown mode"):
        H.DeviceFleet(toy_plan, mode="warp")
    with pytest.raises(H.SimulationError, match="flush policy"):
        H.DeviceFleet(toy_plan, flush_policy="sometimes")
    plan = H.build_plan([[np.array([0, 1])]], np.array([0, 0]))
    with pytest.raises(H.SimulationError, match="destination sets"):
        H.DeviceFleet(plan).load_dest_rows(np.zeros((2, DIM)), 0)


def test_dest_rows_checkpoints(toy_plan):
    rng = np.random.default_rng(70)
    fleet = H.DeviceFleet(toy_plan, mode="full")
    hin = _host_rows(rng, 8)
    hout = np.zeros_like(hin)
    for j in range(fleet.n):
        rows = fleet.load_dest_rows(hin, j)
        for i in range(fleet.m):
            np.testing.assert_array_equal(rows[i], hin[toy_plan.dest_sets[i][j]])
        fleet.store_dest_rows(hout, j, rows)
    np.testing.assert_array_equal(hout, hin)
    t = fleet.transfer_report()["totals"]
    assert t["dest_h2d_rows"] == 8 and t["dest_d2h_rows"] == 8
    hg = np.ones((8, DIM))
    fleet.add_dest_grads(hg, 0, [np.full((toy_plan.dest_sets[i][0].size, DIM), 2.0) for i in range(3)])
    b0 = np.concatenate([toy_plan.dest_sets[i][0] for i in range(3)])
    np.testing.assert_array_equal(hg[b0], 3.0)
    host = H.HostStore(8, [DIM, 2])
    agg = [rng.standard_normal((toy_plan.dest_sets[i][0].size, DIM)) for i in range(3)]
    fleet.store_checkpoint(host, 0, 0, agg)
    back = fleet.load_recomp_chkpt(host, "gcn", 0, 0)
    for i in range(3):
        np.testing.assert_array_equal(back[i], agg[i])
    with pytest.raises(H.CheckpointMissingError) as exc:
        fleet.load_recomp_chkpt(host, "gcn", 0, 1)
    assert exc.value.layer == 0 and exc.value.chunk == 1
    with pytest.raises(H.SimulationError, match="unknown model kind"):
        fleet.load_recomp_chkpt(host, "sage", 0, 0)
    host.set_features(rng.standard_normal((8, DIM)))
    fleet.begin_backward_layer(DIM)
    h_nbr, h_dst = fleet.load_recomp_chkpt(host, "gat", 0, 0)
    for i in range(3):
        np.testing.assert_array_equal(h_nbr[i], host.h[0][toy_plan.neighbor_sets[i][0]])
        np.testing.assert_array_equal(h_dst[i], host.h[0][toy_plan.dest_sets[i][0]])


def test_host_store_contract():
    host = H.HostStore(5, [4, 3, 2])
    assert [h.shape for h in host.h] == [(5, 4), (5, 3), (5, 2)]
    with pytest.raises(H.SimulationError, match="shape"):
        host.set_features(np.zeros((5, 3)))
    host.set_features(np.ones((5, 4)))
    host.grad_h[1][:] = 7
    host.h_valid[1] = True
    host.reset_epoch()
    assert host.h_valid == [True, False, False]
    assert all((g == 0).all() for g in host.grad_h)
