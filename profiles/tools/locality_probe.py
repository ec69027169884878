"""Experiment: how much would a locality-aware destination order buy?  The
cfg2 graph relabelled cluster-major (same graph, vertex ids permuted so each
cluster's id segments are adjacent) vs the original labels: per-phase device
times of value epochs."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2311_14898_b200 as H
from paper_2311_14898_b200 import _native as N
from paper_2311_14898_b200.synth import synth_graph_with_clusters

cfg = bench.CONFIGS["cfg2"]
dims = cfg["dims"]
spec = H.SynthSpec(num_vertices=cfg["V"], avg_degree=cfg["avg_degree"], seed=cfg["seed"])
ds = H.synth_dataset(spec, dims[0], dims[-1])
g0 = ds.graph
_, cl = synth_graph_with_clusters(spec)

def run(tag, g, X, y, mask):
    a = H.partition_vertices(g, 1, seed=0)
    p = H.split_chunks(g, a, 1)
    plan = H.plan_for_partition(p, device=0)
    host = H.HostStore(g.num_vertices, dims, dtype=np.float32, placement="device")
    host.set_features(X)
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32)
    model = H.init_model("gcn", dims, seed=0, lr=0.1, dtype=np.float32)
    for _ in range(3):
        H.train_epoch(p, fleet, model, host, y, mask)
    fleet.set_timing(True)
    N.call("ht_fleet_mark", fleet._handle, 0)
    for _ in range(5):
        H.train_epoch(p, fleet, model, host, y, mask)
    N.call("ht_fleet_mark", fleet._handle, 1)
    ms = C.c_double(0); N.call("ht_fleet_elapsed", fleet._handle, C.byref(ms))
    st = {w: fleet.kernel_stats(w) for w in range(3)}
    print(f"{tag}: {ms.value/5:.2f} ms/epoch  fwd agg {st[0][1]/5:.2f}  bwd agg {st[1][1]/5:.2f}  gemm {st[2][1]/5:.2f}", flush=True)
    fleet.close()

run("original", g0, ds.features, ds.labels, ds.mask)
# cluster-major relabel: new id of old vertex v = rank of v in (cluster, v) order
order = np.lexsort((np.arange(g0.num_vertices), cl))
new_of = np.empty_like(order); new_of[order] = np.arange(order.size)
dst = np.repeat(np.arange(g0.num_vertices), np.diff(g0.csc_offsets))
src = g0.csc_sources
g1 = H.from_edges(new_of[src], new_of[dst], num_vertices=g0.num_vertices)
run("cluster-major", g1, np.asarray(ds.features)[order], np.asarray(ds.labels)[order], np.asarray(ds.mask)[order])
# random relabel (no locality at all)
rp = np.random.default_rng(1).permutation(g0.num_vertices)
new_of = np.empty_like(rp); new_of[rp] = np.arange(rp.size)
g2 = H.from_edges(new_of[src], new_of[dst], num_vertices=g0.num_vertices)
run("random", g2, np.asarray(ds.features)[rp], np.asarray(ds.labels)[rp], np.asarray(ds.mask)[rp])
