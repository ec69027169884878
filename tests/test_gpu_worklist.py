"""The one-launch work-list aggregation (k_seg_work_*: pieces of long
segments and short segments from one device counter, the last piece of a
segment summing the partials in piece order) against r1's three-launch
sequence (segment kernel, pieces kernel, fixup; HT_SEG_SPLIT_LAUNCH=1):
the same sums in the same order, so whole epochs must agree bitwise - loss,
weights, every host array.  The graph has hub sources and destinations of
several thousand edges, so both the CSC forward and the CSR backward run
pieces; widths cover the narrow sub-warp kernel (<= 64 floats) and the
1-4 float4-per-lane kernels, one and several devices/batches."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2311_14898_b200 as H
from paper_2311_14898_b200 import synth as S
m, n, out, prec = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[6]
dims = [int(x) for x in sys.argv[5].split(",")]
spec = S.SynthSpec(num_vertices=60000, avg_degree=24.0, hub_fraction=0.001, hub_prob=0.7, seed=5)
src, dst, cl = S.synth_edges(spec)
rng = np.random.default_rng(9)  # + destination hubs: in-degrees of several thousand
hs = np.concatenate([rng.choice(spec.num_vertices, 3000 + 1500 * k, replace=False)
                     for k in range(3)])
hd = np.repeat(np.array([11, 30011, 59999]), [3000, 4500, 6000])
src, dst = np.concatenate([src, hs]), np.concatenate([dst, hd])
from paper_2311_14898_b200.graph import dedup_edges
keep = dedup_edges(src, dst, spec.num_vertices)
g = H.from_edges(src[keep], dst[keep], num_vertices=spec.num_vertices)
X, y, mask = S.synth_node_data(spec.num_vertices, dims[0], dims[-1], 5, cluster_of=cl)
deg_in = np.diff(g.csc_offsets).max(); deg_out = np.diff(g.csr_offsets).max()
assert deg_in > 2048 and deg_out > 2048, (deg_in, deg_out)
class DS: pass
ds = DS(); ds.graph, ds.features, ds.labels, ds.mask = g, X, y, mask
a = H.partition_vertices(ds.graph, m, seed=5)
p = H.split_chunks(ds.graph, a, n)
plan = H.plan_for_partition(p)
model = H.init_model("gcn", dims, seed=5, lr=0.1, dtype=np.float32)
host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32,
                   placement="device" if m == 1 and n == 1 else "host")
host.set_features(ds.features)
fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, precision=prec)
snap = {}
for e in range(2):
    r = H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    snap[f"loss{e}"] = np.array([r.loss])
for l, w in enumerate(model.weights):
    snap[f"W{l}"] = w
for l, x in enumerate(host.h):
    snap[f"h{l}"] = np.array(x)
for l, x in enumerate(host.grad_h):
    snap[f"g{l}"] = np.array(x)
for l in range(len(dims) - 1):
    snap[f"a{l}"] = np.array(host.agg[l])
fleet.close()
np.savez(out, **snap)
"""


def _run(tmp_path, tag, env_extra, m, n, dims, prec):
    out = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(m), str(n), out,
                        ",".join(map(str, dims)), prec], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("m,n,dims,prec", [(1, 1, [100, 256, 48, 47], "tf32"),
                                           (1, 1, [32, 128, 20], "tf32"),
                                           (2, 2, [64, 192, 40], "tf32"),
                                           (1, 1, [64, 384, 500, 40], "fp32")])
def test_worklist_equals_split_launch(tmp_path, m, n, dims, prec):
    a = _run(tmp_path, "work", {}, m, n, dims, prec)
    b = _run(tmp_path, "split", {"HT_SEG_SPLIT_LAUNCH": "1"}, m, n, dims, prec)
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_forward_hub_pieces_reassociate_only_hub_rows():
    """Forward CSC aggregation rows are the sequential multiply-then-add of
    np.add.at (src/engine.py:139) bitwise - except destinations with more
    than 1024 in-edges, whose pieces are summed separately and then added in
    piece order: deterministic, within FP32 reassociation error of the
    sequential sum (the oracle's association)."""
    import paper_2311_14898_b200 as H
    from paper_2311_14898_b200 import synth as S
    from paper_2311_14898_b200.graph import dedup_edges
    spec = S.SynthSpec(num_vertices=20000, avg_degree=12.0, seed=6)
    src, dst, cl = S.synth_edges(spec)
    rng = np.random.default_rng(3)
    hubs = np.array([5, 777, 19999])
    hs = np.concatenate([rng.choice(spec.num_vertices, 2500 * (k + 1), replace=False) for k in range(3)])
    hd = np.repeat(hubs, [2500, 5000, 7500])
    src, dst = np.concatenate([src, hs]), np.concatenate([dst, hd])
    keep = dedup_edges(src, dst, spec.num_vertices)
    g = H.from_edges(src[keep], dst[keep], num_vertices=spec.num_vertices)
    X, y, mask = S.synth_node_data(spec.num_vertices, 32, 8, 6, cluster_of=cl)
    p = H.split_chunks(g, H.partition_vertices(g, 1, seed=6), 1)
    dims = [32, 16, 8]
    host = H.HostStore(g.num_vertices, dims, dtype=np.float32, placement="device")
    host.set_features(X)
    fleet = H.DeviceFleet(H.plan_for_partition(p), dtype=np.float32)
    H.train_epoch(p, fleet, H.init_model("gcn", dims, seed=2, dtype=np.float32), host, y, mask)
    agg0 = np.array(host.agg[0])
    fleet.close()
    x32 = np.asarray(host.h[0])
    w32 = np.asarray(g.edge_weights, dtype=np.float32)
    off, srcs = g.csc_offsets, g.csc_sources
    deg = np.diff(off)
    assert (deg[hubs] > 1024).all() and np.sort(deg)[-4] <= 1024
    sample = np.concatenate([hubs, rng.choice(g.num_vertices, 200, replace=False)])
    for v in sample:
        acc = np.zeros(dims[0], np.float32)
        for e in range(off[v], off[v + 1]):
            acc = acc + w32[e] * x32[srcs[e]]
        if deg[v] > 1024:
            assert np.abs(agg0[v] - acc).max() <= 1e-5 * max(np.abs(acc).max(), 1e-30), v
        else:
            np.testing.assert_array_equal(agg0[v], acc, err_msg=f"row {v}")
