"""Small epochs for compute-sanitizer (memcheck / racecheck / synccheck):
GCN and GAT through every layer-driver path - m x n in {1x1 (HBM store in
place: direct reads/backward, project-first, work-list hub pieces),
1x1 host store (owner cache + HBM checkpoints), 2x2 host store cache off
(slot loads, peer fetches, owner push / flush), 2x2 cache on}, plus the
recompute-cache hybrid under a budget - and, with --rank R --world W, one
rank of the rank-mode path (CUDA IPC + the device barrier).

    compute-sanitizer --tool memcheck python profiles/tools/sanitize_epoch.py
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2311_14898_b200 as H  # noqa: E402


def dataset(V=3000):
    from paper_2311_14898_b200 import synth as S
    from paper_2311_14898_b200.graph import dedup_edges
    spec = S.SynthSpec(num_vertices=V, avg_degree=10.0, seed=3)
    src, dst, cl = S.synth_edges(spec)
    # a destination and a source with > 1024 edges: hub pieces in both passes
    rng = np.random.default_rng(1)
    hs, hd = rng.choice(V, 1500, replace=False), rng.choice(V, 1500, replace=False)
    src = np.concatenate([src, hs, np.full(1500, 11)])
    dst = np.concatenate([dst, np.full(1500, 7), hd])
    keep = dedup_edges(src, dst, V)
    g = H.from_edges(src[keep], dst[keep], num_vertices=V)
    X, y, mask = S.synth_node_data(V, 16, 8, 3, cluster_of=cl)
    return g, X, y, mask


def run(g, X, y, mask, kind, m, n, placement, cache, budget=None, rank=None, dims=None):
    a = H.partition_vertices(g, m, seed=3)
    p = H.split_chunks(g, a, n)
    plan = H.plan_for_partition(p)
    if dims is None:
        dims = [16, 24, 8] if kind == "gcn" else [16, 12, 8]
    model = H.init_model(kind, dims, seed=3, dtype=np.float32)
    host = H.HostStore(g.num_vertices, dims, dtype=np.float32, placement=placement)
    host.set_features(X)
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, precision="tf32", cache=cache,
                          hbm_budget_gb=budget, rank=rank, devices=[0] if rank is not None else None)
    loss = H.train_epoch(p, fleet, model, host, y, mask).loss
    if kind == "gcn" and rank is None:
        _ = [np.asarray(host.agg[l]) for l in range(len(dims) - 1)]  # checkpoint reads
    fleet.close()
    print(f"{kind} {dims} m={m} n={n} {placement} cache={cache} budget={budget} rank={rank}: "
          f"loss {loss:.6f}", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=None)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--port", type=int, default=29512)
    args = ap.parse_args()
    g, X, y, mask = dataset()
    if args.rank is not None:
        import torch.distributed as tdist
        tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{args.port}",
                                 rank=args.rank, world_size=args.world)
        for kind in ("gcn", "gat"):
            run(g, X, y, mask, kind, args.world, 2, "host", "auto", rank=args.rank)
        tdist.destroy_process_group()
        sys.exit(0)
    for kind in ("gcn", "gat"):
        run(g, X, y, mask, kind, 1, 1, "device", "auto")
        run(g, X, y, mask, kind, 1, 1, "host", "auto")
        run(g, X, y, mask, kind, 2, 2, "host", "off")
        run(g, X, y, mask, kind, 2, 2, "host", "on")
    # a 144-wide layer: the 3xTF32 forward GEMM on CTA pairs (N > 128) and the
    # masked-A backward GEMM (gz formed from the g and h tiles) of session 3
    run(g, X, y, mask, "gcn", 1, 1, "device", "auto", dims=[16, 144, 144, 8])
    run(g, X, y, mask, "gcn", 1, 1, "host", "auto", dims=[16, 144, 144, 8])
    V = g.num_vertices
    # h + grad mirrors, project-first buffers, one 24-wide scratch: both agg^l recomputed
    run(g, X, y, mask, "gcn", 1, 1, "host", "on",
        budget=(4 * V * ((16 + 24) + (16 + 24 + 8) + 2 * 8 + 24) + 4096) / 2 ** 30)
