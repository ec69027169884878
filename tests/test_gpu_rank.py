"""One process per device (rank mode) on the GPU: two processes share one
B200 here (the box has one GPU), exchanging slot buffers, gradient views and
weight-gradient accumulators through CUDA IPC and synchronizing with the
device-side cross-process barrier.  Both ranks must reproduce the oracle's
two-epoch trajectory and agree with each other bitwise."""

import json
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, mode, kind, cache, compact=False):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as tdist
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                             world_size=world)
    import paper_2311_14898_b200 as H
    ds = H.synth_dataset(H.SynthSpec(num_vertices=4000, avg_degree=8.0, seed=9), 16, 8)
    a = H.partition_vertices(ds.graph, world, seed=9)
    p = H.reorganize(H.split_chunks(ds.graph, a, 3)).partition
    plan = H.plan_for_partition(p)
    dims = [16, 24, 8]
    model = H.init_model(kind, dims, seed=3, lr=0.1, dtype=np.float32)
    own = np.flatnonzero(a.owner == rank) if compact else None
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32, rows=own)
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, mode=mode, dtype=np.float32, precision="fp32", rank=rank,
                          devices=[0], cache=cache)
    losses = []
    for _ in range(2):
        losses.append(H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss)
    mine = np.concatenate(plan.dest_sets[rank])
    gh0 = np.asarray(host.grad_h[0])
    gh0 = gh0[np.searchsorted(own, mine)] if compact else gh0[mine]
    res = {"losses": losses, "W": [w.tolist() for w in model.weights],
           "A": [x.tolist() for x in model.attn] if kind == "gat" else None,
           "cache": fleet.cache_active,
           "gh0_rows": mine.tolist(), "gh0": gh0.tolist(),
           "report": fleet.transfer_report(
               *(2 * x for x in H.comm_passes_per_epoch(model)))["planner_consistent"]}
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as fh:
        json.dump(res, fh)
    tdist.destroy_process_group()


@pytest.mark.parametrize("kind,mode,cache,compact", [
    ("gcn", "full", "auto", False), ("gcn", "p2p", "auto", False), ("gcn", "full", "off", False),
    ("gcn", "full", "auto", True), ("gat", "full", "auto", False), ("gat", "p2p", "off", False),
    ("gat", "full", "auto", True)])
def test_two_ranks_share_one_gpu(tmp_path, kind, mode, cache, compact):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2311_14898_b200 as H
    from oracle import hongtu_oracle as O
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path), mode, kind, cache,
                                                    compact))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    out = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    assert out[0]["losses"] == out[1]["losses"]
    assert out[0]["W"] == out[1]["W"]
    assert out[0]["A"] == out[1]["A"]
    assert out[0]["cache"] == out[1]["cache"] == (cache == "auto" or compact)
    assert out[0]["report"] and out[1]["report"]
    # oracle: the same partitioned epochs in one process
    ds = H.synth_dataset(H.SynthSpec(num_vertices=4000, avg_degree=8.0, seed=9), 16, 8)
    a = H.partition_vertices(ds.graph, world, seed=9)
    p = H.reorganize(H.split_chunks(ds.graph, a, 3)).partition
    grid = [[vars(c) for c in row] for row in p.chunks]
    plan = O.plan_of_grid(grid, a.owner)
    m0 = H.init_model(kind, [16, 24, 8], seed=3, dtype=np.float32)
    W = [w.copy() for w in m0.weights]
    A = [x.copy() for x in m0.attn] if kind == "gat" else None
    losses = []
    for e in range(2):
        ref = O.partitioned_epoch(grid, plan, W, ds.features, ds.labels, ds.mask, mode=mode,
                                  dtype=np.float32, kind=kind, attn=A)
        W = ref["weights"]
        A = ref.get("attn")
        losses.append(ref["loss"])
        if e == 1:
            for r in range(world):
                rows = np.asarray(out[r]["gh0_rows"])
                assert O.rel_err(np.asarray(out[r]["gh0"]), ref["grad_h"][0][rows]) < 1e-5
    np.testing.assert_allclose(out[0]["losses"], losses, rtol=1e-5)
    for l in range(2):
        assert O.rel_err(np.asarray(out[0]["W"][l]), W[l]) < 1e-5
        if kind == "gat":
            assert O.rel_err(np.asarray(out[0]["A"][l]), A[l]) < 1e-5
