"""Host-side logic of the one-process-per-GPU (rank) mode, world size 2 over
gloo on the CPU: handle exchange, loss-partial reduction, and the ownership
invariant that lets every rank keep its own host store (in p2p/full mode a
device reads and writes only host rows it owns)."""

import json
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as tdist
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                             world_size=world)
    from paper_2311_14898_b200 import dist
    import paper_2311_14898_b200 as H
    from oracle import hongtu_oracle as O

    res = {}
    # 1. IPC-handle exchange: every rank sees every blob, in rank order
    blobs = dist.exchange(bytes([rank + 1]) * dist.HT_IPC_BYTES)
    res["blobs"] = [b[0] for b in blobs]
    res["lens"] = [len(b) for b in blobs]
    # 2. the same seeded inputs and plan on every rank
    ds = H.synth_dataset(H.SynthSpec(num_vertices=3000, avg_degree=7.0, seed=5), 12, 4)
    a = H.partition_vertices(ds.graph, world, seed=5)
    p = H.reorganize(H.split_chunks(ds.graph, a, 3)).partition
    plan = H.plan_for_partition(p)
    res["owns_full"] = dist.owns_all_touched(plan, rank, "full")
    res["owns_p2p"] = dist.owns_all_touched(plan, rank, "p2p")
    # 3. loss: each rank's partial over its own destination rows (the rows
    # its loss kernel covers) sums to the global masked-mean loss
    grid = [[vars(c) for c in row] for row in p.chunks]
    W = O.glorot_weights([12, 16, 4], 1, dtype=np.float64)
    ref = O.partitioned_epoch(grid, O.plan_of_grid(grid, a.owner), W, ds.features, ds.labels,
                              ds.mask, dtype=np.float64)
    hL = ref["h"][-1]
    mine = np.concatenate([c["vertices"] for c in grid[rank]])
    sel = mine[ds.mask[mine]]
    z = hL[sel] - hL[sel].max(axis=1, keepdims=True)
    lp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    partial = float(-lp[np.arange(sel.size), ds.labels[sel]].sum() / ds.mask.sum())
    res["loss"] = dist.allreduce_sum(partial)
    res["ref_loss"] = ref["loss"]
    res["max"] = dist.allreduce_max(float(rank))
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as fh:
        json.dump(res, fh)
    tdist.destroy_process_group()


def test_rank_mode_host_logic_gloo(tmp_path):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    out = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    for r in range(world):
        assert out[r]["blobs"] == [1, 2]
        assert out[r]["lens"] == [256, 256]
        assert out[r]["owns_full"] and out[r]["owns_p2p"]
        assert out[r]["loss"] == pytest.approx(out[r]["ref_loss"], rel=1e-12)
        assert out[r]["max"] == 1.0
    assert out[0]["loss"] == out[1]["loss"]
