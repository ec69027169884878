"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    python tests/golden/make_golden.py [--skip-cfg1]

It imports ``chunktrain`` read-only from ``/root/reference/pkg/src`` and
writes small fixtures next to this file:

* ``toy.json``       - the reference's 8-vertex / 19-edge 3x2 toy grid
                        (tests/conftest.py:44-78): every plan set, slots,
                        volumes, cost, predicted transfers, metered sweeps.
* ``small.npz`` / ``small.json`` - a 2,000-vertex synthetic graph: graph
                        arrays, LDG owners for m=1..4, chunk/plan digests,
                        reorganization, and 2-epoch GCN runs (fp64 + fp32,
                        three modes) plus the monolithic fp64 oracle.
* ``sets.json``      - plan digests + predicted transfers for 200 random
                        set instances (the reference's random_set_instance
                        recipe, tests/conftest.py:101-111).
* ``gat.json`` / ``gat.npz`` - GAT (config 5's model) on the small graph:
                        2-epoch runs (fp64 + fp32, three modes), the
                        monolithic fp64 trainer, single-chunk kernel vectors.
* ``cfg1.json`` / ``cfg1.npz`` - BASELINE config 1 (100K V, 64-128-16,
                        m=4, n=4, reorganized): hashes, volumes, caps,
                        predicted transfers, fp32 losses and weights.
"""

import argparse
import json
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from chunktrain import devices, engine, graph, partition, planner, reference, synth  # noqa: E402
from digest import chunk_digest, plan_digest  # noqa: E402

TOY_EDGES = [
    (1, 0), (2, 0), (0, 1), (3, 1), (4, 2), (3, 2), (2, 3), (5, 3),
    (0, 4), (1, 4), (4, 4), (2, 5), (4, 5), (5, 5), (6, 5), (3, 6),
    (4, 6), (7, 6), (3, 7),
]
TOY_OWNER = [0, 0, 0, 0, 1, 1, 2, 2]
TOY_RANGES = [[(0, 2), (2, 4)], [(0, 1), (1, 2)], [(0, 1), (1, 2)]]


def _l(a):
    return [int(x) for x in np.asarray(a).ravel()]


def ref_plan_digest(plan):
    live = plan.layout.live_sets
    slots = [[np.array([plan.layout.slot_maps[i][j][int(v)] for v in live[i][j]],
                       dtype=np.int64) for j in range(plan.n)] for i in range(plan.m)]
    return plan_digest(plan.m, plan.n, plan.neighbor_sets, plan.union_sets,
                       plan.owned_sets, plan.carry_sets, plan.load_sets,
                       plan.fetch_sets, plan.nbr_carry_sets, live, slots,
                       plan.layout.capacities,
                       (plan.volumes.v_ori, plan.volumes.v_p2p, plan.volumes.v_ru))


def sweep_meters(plan, mode, V, dim, seed, flush_policy="on_eviction"):
    """Deterministic forward+backward comm sweep; returns totals, peaks and
    the host gradient checksum."""
    rng = np.random.default_rng(seed)
    fleet = devices.DeviceFleet(plan, mode=mode, flush_policy=flush_policy)
    host = rng.standard_normal((V, dim))
    fleet.begin_forward_layer(dim)
    for j in range(plan.n):
        fleet.dedup_comm_fwd(host, j)
    host_grad = np.zeros((V, dim))
    fleet.begin_backward_layer(dim)
    for j in range(plan.n):
        views = [rng.standard_normal((plan.neighbor_sets[i][j].size, dim))
                 for i in range(plan.m)]
        fleet.dedup_comm_bwd(views, host_grad, j)
    rep = fleet.transfer_report(fwd_passes=1, bwd_passes=1)
    return {"totals": rep["totals"], "peaks": rep["peak_live_slots"],
            "consistent": bool(rep["planner_consistent"]),
            "grad_sum": float(host_grad.sum())}


def toy():
    src = np.array([e[0] for e in TOY_EDGES])
    dst = np.array([e[1] for e in TOY_EDGES])
    g = graph.from_edges(src, dst, num_vertices=8)
    a = partition.PartitionAssignment(owner=np.array(TOY_OWNER, dtype=np.int64), m=3)
    p = partition.two_level_from_ranges(g, a, TOY_RANGES)
    plan = planner.plan_for_partition(p)
    m, n = plan.m, plan.n
    out = {
        "graph": {k: _l(getattr(g, k)) for k in ("csc_offsets", "csc_sources", "csr_offsets",
                                                   "csr_targets", "csr_edge_perm")},
        "weights": [float(x) for x in g.edge_weights],
        "hash": g.content_hash(),
        "N": [[_l(s) for s in row] for row in plan.neighbor_sets],
        "U": [_l(u) for u in plan.union_sets],
        "T": [[_l(s) for s in row] for row in plan.owned_sets],
        "carry": [[_l(s) for s in row] for row in plan.carry_sets],
        "load": [[_l(s) for s in row] for row in plan.load_sets],
        "fetch": [[{str(k): _l(v) for k, v in d.items()} for d in row] for row in plan.fetch_sets],
        "nbr_carry": [[_l(s) for s in row] for row in plan.nbr_carry_sets],
        "live": [[_l(s) for s in row] for row in plan.layout.live_sets],
        "slots": [[[int(plan.layout.slot_maps[i][j][int(v)]) for v in plan.layout.live_sets[i][j]]
                   for j in range(n)] for i in range(m)],
        "caps": _l(plan.layout.capacities),
        "volumes": [plan.volumes.v_ori, plan.volumes.v_p2p, plan.volumes.v_ru],
        "cost": planner.comm_cost(plan.volumes, planner.CostParams()),
        "alpha": partition.replication_factor(p),
        "predicted": {md: planner.predicted_transfers(plan, md) for md in planner.MODES},
        "digest": ref_plan_digest(plan),
        "chunk_digest": chunk_digest(p.chunks),
        "sweeps": {md: sweep_meters(plan, md, 8, 3, 11) for md in planner.MODES},
        "sweep_every_batch": sweep_meters(plan, "full", 8, 3, 11, "every_batch"),
    }
    r = planner.reorganize(p)
    out["reorg"] = {"chunk_orders": r.chunk_orders, "batch_order": r.batch_order}
    return out


def _epochs(g, p, plan, ds, dims, mode, dtype, epochs=2, seed=5, kind="gcn"):
    model = engine.init_model(kind, dims, seed=seed, lr=0.1, dtype=dtype)
    host = devices.HostStore(g.num_vertices, dims, dtype=dtype)
    host.set_features(ds.features)
    fleet = devices.DeviceFleet(plan, mode=mode, dtype=dtype)
    losses, snaps = [], {}
    for e in range(epochs):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = engine.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
        losses.append(float(res.loss))
        if e == 0:
            snaps["hL"] = host.h[len(dims) - 1].copy()
            snaps["gh0"] = host.grad_h[0].copy()
            snaps["gh1"] = host.grad_h[1].copy()
            if kind == "gcn":
                snaps["agg0"] = host.agg[0].copy()
            snaps["w_e0"] = [w.copy() for w in model.weights]
            if kind == "gat":
                snaps["a_e0"] = [a.copy() for a in model.attn]
    rep = fleet.transfer_report(*engine.comm_passes_per_epoch(model))
    if kind == "gat":
        snaps["a_after"] = [a.copy() for a in model.attn]
    return losses, [w.copy() for w in model.weights], snaps, rep


def small(arrays, meta):
    spec = synth.SynthSpec(num_vertices=2000, avg_degree=8.0, seed=7)
    ds = synth.synth_dataset(spec, 8, 4)
    g = ds.graph
    meta["synth"] = {"num_vertices": 2000, "avg_degree": 8.0, "seed": 7,
                     "feature_dim": 8, "num_classes": 4}
    meta["hash"] = g.content_hash()
    meta["num_edges"] = g.num_edges
    for k in ("csc_offsets", "csc_sources", "csr_offsets", "csr_targets", "csr_edge_perm"):
        arrays["g_" + k] = getattr(g, k).astype(np.int32)
    arrays["g_weights"] = g.edge_weights
    arrays["X"] = ds.features
    arrays["labels"] = ds.labels.astype(np.int8)
    arrays["mask"] = ds.mask
    arrays["cluster_of"] = ds.cluster_of.astype(np.int8)
    owners = {}
    for m in (1, 2, 3, 4):
        a = partition.partition_vertices(g, m, epsilon=0.1, seed=7)
        arrays[f"owner_m{m}"] = a.owner.astype(np.int8)
        owners[m] = a
    meta["edge_cut_m3"] = partition.edge_cut(g, owners[3])
    a3 = owners[3]
    p = partition.split_chunks(g, a3, 4)
    meta["ranges_m3n4"] = [[list(map(int, r)) for r in partition.split_ranges(
        g.in_degrees()[np.flatnonzero(a3.owner == i)], 4)] for i in range(3)]
    meta["chunk_digest_m3n4"] = chunk_digest(p.chunks)
    plan_id = planner.plan_for_partition(p)
    meta["plan_digest_identity"] = ref_plan_digest(plan_id)
    meta["volumes_identity"] = [plan_id.volumes.v_ori, plan_id.volumes.v_p2p, plan_id.volumes.v_ru]
    r = planner.reorganize(p)
    meta["reorg"] = {"chunk_orders": r.chunk_orders, "batch_order": r.batch_order}
    r2 = planner.reorganize(p, move_all_rows=False)
    meta["reorg_fixed_row0"] = {"chunk_orders": r2.chunk_orders, "batch_order": r2.batch_order}
    pr = r.partition
    plan = planner.plan_for_partition(pr)
    meta["plan_digest_reorg"] = ref_plan_digest(plan)
    meta["volumes_reorg"] = [plan.volumes.v_ori, plan.volumes.v_p2p, plan.volumes.v_ru]
    meta["caps_reorg"] = _l(plan.layout.capacities)
    meta["predicted_reorg"] = {md: planner.predicted_transfers(plan, md) for md in planner.MODES}
    meta["alpha_m3n4"] = partition.replication_factor(p)
    dims = [8, 12, 4]
    meta["dims"] = dims
    runs = {}
    for dtype, tag in ((np.float64, "f64"), (np.float32, "f32")):
        for mode in planner.MODES:
            losses, weights, snaps, rep = _epochs(g, pr, plan, ds, dims, mode, dtype)
            runs[f"{tag}_{mode}"] = {"losses": losses, "totals": rep["totals"],
                                     "peaks": rep["peak_live_slots"],
                                     "consistent": bool(rep["planner_consistent"])}
            if mode == "full":
                for l, w in enumerate(weights):
                    arrays[f"{tag}_W{l}_after2"] = w
                for l, w in enumerate(snaps["w_e0"]):
                    arrays[f"{tag}_W{l}_after1"] = w
                arrays[f"{tag}_hL_e0"] = snaps["hL"]
                arrays[f"{tag}_gh0_e0"] = snaps["gh0"]
                arrays[f"{tag}_gh1_e0"] = snaps["gh1"]
                arrays[f"{tag}_agg0_e0"] = snaps["agg0"]
    meta["runs"] = runs
    model = engine.init_model("gcn", dims, seed=5, lr=0.1)
    mono = reference.reference_train(g, model, ds.features, ds.labels, ds.mask, epochs=2)
    meta["mono_losses"] = [float(x) for x in mono]
    for l, w in enumerate(model.weights):
        arrays[f"mono_W{l}_after2"] = w


def gat(arrays, meta):
    """GAT on the 2,000-vertex graph of small(): m=3,
    n=4 reorganized, dims 8-12-4, two epochs per dtype and mode through the
    reference's train_epoch; the fp64 monolithic trainer; and single-chunk
    kernel vectors (gat_layer_forward / gat_layer_backward_recompute)."""
    spec = synth.SynthSpec(num_vertices=2000, avg_degree=8.0, seed=7)
    ds = synth.synth_dataset(spec, 8, 4)
    g = ds.graph
    meta["hash"] = g.content_hash()
    a3 = partition.partition_vertices(g, 3, epsilon=0.1, seed=7)
    pr = planner.reorganize(partition.split_chunks(g, a3, 4)).partition
    plan = planner.plan_for_partition(pr)
    meta["plan_digest_reorg"] = ref_plan_digest(plan)
    dims = [8, 12, 4]
    meta["dims"] = dims
    runs = {}
    for dtype, tag in ((np.float64, "f64"), (np.float32, "f32")):
        for mode in planner.MODES:
            losses, weights, snaps, rep = _epochs(g, pr, plan, ds, dims, mode, dtype, kind="gat")
            runs[f"{tag}_{mode}"] = {"losses": losses, "totals": rep["totals"],
                                     "peaks": rep["peak_live_slots"],
                                     "consistent": bool(rep["planner_consistent"])}
            if mode == "full":
                for l, w in enumerate(weights):
                    arrays[f"{tag}_W{l}_after2"] = w
                for l, w in enumerate(snaps["w_e0"]):
                    arrays[f"{tag}_W{l}_after1"] = w
                for l, a in enumerate(snaps["a_e0"]):
                    arrays[f"{tag}_a{l}_after1"] = a
                for l, a in enumerate(snaps["a_after"]):
                    arrays[f"{tag}_a{l}_after2"] = a
                arrays[f"{tag}_hL_e0"] = snaps["hL"]
                arrays[f"{tag}_gh0_e0"] = snaps["gh0"]
                arrays[f"{tag}_gh1_e0"] = snaps["gh1"]
    meta["runs"] = runs
    model = engine.init_model("gat", dims, seed=5, lr=0.1)
    mono = reference.reference_train(g, model, ds.features, ds.labels, ds.mask, epochs=2)
    meta["mono_losses"] = [float(x) for x in mono]
    for l, (w, a) in enumerate(zip(model.weights, model.attn)):
        arrays[f"mono_W{l}_after2"] = w
        arrays[f"mono_a{l}_after2"] = a
    # single-chunk kernel vectors: chunk (1, 2) of the reorganized grid
    ch = pr.chunks[1][2]
    rng = np.random.default_rng(21)
    d_in, d_out = 8, 12
    h_nbr = rng.standard_normal((ch.sources.size, d_in))
    h_dst = rng.standard_normal((ch.num_vertices, d_in))
    W = rng.standard_normal((d_in, d_out)) * 0.5
    av = rng.standard_normal(2 * d_out) * 0.5
    R = rng.standard_normal((ch.num_vertices, d_out))
    h, st = engine.gat_layer_forward(ch, h_nbr, h_dst, W, av)
    gn, gd, gW, ga = engine.gat_layer_backward_recompute(ch, h_nbr, h_dst, R, W, av)
    for k, v in (("h_nbr", h_nbr), ("h_dst", h_dst), ("W", W), ("a", av), ("R", R), ("h", h),
                 ("alpha", st.alpha), ("t", st.t), ("s", st.s), ("g_nbr", gn), ("g_dst", gd),
                 ("g_W", gW), ("g_a", ga)):
        arrays["k_" + k] = v
    meta["kernel_chunk"] = [1, 2]


def set_instances(count=200, seed=123):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(rng.integers(1, 5))
        n = int(rng.integers(1, 7))
        universe = int(rng.integers(8, 40))
        owner = rng.integers(0, m, size=universe)
        nbrs = []
        for _i in range(m):
            row = []
            for _j in range(n):
                k = int(rng.integers(0, max(2, universe // 2)))
                row.append(np.unique(rng.integers(0, universe, size=k)))
            nbrs.append(row)
        plan = planner.build_plan(nbrs, owner)
        out.append({"digest": ref_plan_digest(plan),
                    "predicted": {md: planner.predicted_transfers(plan, md) for md in planner.MODES}})
    return out


def cfg1(arrays, meta):
    t0 = time.time()
    spec = synth.SynthSpec(num_vertices=100_000, avg_degree=20.0, seed=0)
    ds = synth.synth_dataset(spec, 64, 16)
    g = ds.graph
    meta["hash"] = g.content_hash()
    meta["num_edges"] = g.num_edges
    a = partition.partition_vertices(g, 4, seed=0)
    import hashlib
    meta["owner_sha16"] = hashlib.sha256(np.ascontiguousarray(a.owner).tobytes()).hexdigest()[:16]
    meta["owner_sha"] = hashlib.sha256(np.ascontiguousarray(a.owner).tobytes()).hexdigest()
    p = partition.split_chunks(g, a, 4)
    meta["chunk_digest"] = chunk_digest(p.chunks)
    plan_id = planner.plan_for_partition(p)
    meta["volumes_identity"] = [plan_id.volumes.v_ori, plan_id.volumes.v_p2p, plan_id.volumes.v_ru]
    r = planner.reorganize(p)
    meta["batch_order"] = r.batch_order
    meta["chunk_orders"] = r.chunk_orders
    plan = planner.plan_for_partition(r.partition)
    meta["plan_digest_reorg"] = ref_plan_digest(plan)
    meta["volumes_reorg"] = [plan.volumes.v_ori, plan.volumes.v_p2p, plan.volumes.v_ru]
    meta["caps"] = _l(plan.layout.capacities)
    meta["predicted"] = {md: planner.predicted_transfers(plan, md) for md in planner.MODES}
    dims = [64, 128, 16]
    losses, weights, snaps, rep = _epochs(g, r.partition, plan, ds, dims, "full", np.float32,
                                          epochs=2, seed=0)
    meta["losses_f32"] = losses
    meta["totals_f32"] = rep["totals"]
    for l, w in enumerate(weights):
        arrays[f"W{l}_after2"] = w
    for l, w in enumerate(snaps["w_e0"]):
        arrays[f"W{l}_after1"] = w
    meta["seconds"] = time.time() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-cfg1", action="store_true")
    ap.add_argument("--only-gat", action="store_true")
    args = ap.parse_args()
    arrays, meta = {}, {}
    gat(arrays, meta)
    np.savez_compressed(os.path.join(HERE, "gat.npz"), **arrays)
    with open(os.path.join(HERE, "gat.json"), "w") as fh:
        json.dump(meta, fh, indent=0, sort_keys=True)
    if args.only_gat:
        print("GAT golden vectors written to", HERE)
        return
    with open(os.path.join(HERE, "toy.json"), "w") as fh:
        json.dump(toy(), fh, indent=0, sort_keys=True)
    arrays, meta = {}, {}
    small(arrays, meta)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)
    with open(os.path.join(HERE, "small.json"), "w") as fh:
        json.dump(meta, fh, indent=0, sort_keys=True)
    with open(os.path.join(HERE, "sets.json"), "w") as fh:
        json.dump(set_instances(), fh, indent=0, sort_keys=True)
    if not args.skip_cfg1:
        arrays, meta = {}, {}
        cfg1(arrays, meta)
        np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **arrays)
        with open(os.path.join(HERE, "cfg1.json"), "w") as fh:
            json.dump(meta, fh, indent=0, sort_keys=True)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
