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


def _worker(rank, world, port, out_dir, mode):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as tdist
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                             world_size=world)
    import paper_2311_14898_b200 as H
    ds = H.synth_dataset(H.SynthSpec(num_vertices=4000, avg_degree=8.0, seed=9), 16, 5)
    a = H.partition_vertices(ds.graph, world, seed=9)
    p = H.reorganize(H.split_chunks(ds.graph, a, 3)).partition
    plan = H.plan_for_partition(p)
    dims = [16, 24, 5]
    model = H.init_model("gcn", dims, seed=3, lr=0.1, dtype=np.float32)
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32)
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, mode=mode, dtype=np.float32, precision="fp32", rank=rank,
                          devices=[0])
    losses = []
    for _ in range(2):
        losses.append(H.train_epoch(p, fleet, model, host, ds.labels, ds.mask).loss)
    mine = np.concatenate(plan.dest_sets[rank])
    res = {"losses": losses, "W": [w.tolist() for w in model.weights],
           "gh0_rows": mine.tolist(), "gh0": np.asarray(host.grad_h[0])[mine].tolist(),
           "report": fleet.transfer_report(4, 4)["planner_consistent"]}
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as fh:
        json.dump(res, fh)
    tdist.destroy_process_group()


@pytest.mark.parametrize("mode", ["full", "p2p"])
def test_two_ranks_share_one_gpu(tmp_path, mode):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2311_14898_b200 as H
    from oracle import hongtu_oracle as O
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path), mode))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    out = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    assert out[0]["losses"] == out[1]["losses"]
    assert out[0]["W"] == out[1]["W"]
    assert out[0]["report"] and out[1]["report"]
    # oracle: the same partitioned epochs in one process
    ds = H.synth_dataset(H.SynthSpec(num_vertices=4000, avg_degree=8.0, seed=9), 16, 5)
    a = H.partition_vertices(ds.graph, world, seed=9)
    p = H.reorganize(H.split_chunks(ds.graph, a, 3)).partition
    grid = [[vars(c) for c in row] for row in p.chunks]
    plan = O.plan_of_grid(grid, a.owner)
    W = [w.copy() for w in H.init_model("gcn", [16, 24, 5], seed=3, dtype=np.float32).weights]
    losses = []
    for e in range(2):
        ref = O.partitioned_epoch(grid, plan, W, ds.features, ds.labels, ds.mask, mode=mode,
                                  dtype=np.float32)
        W = ref["weights"]
        losses.append(ref["loss"])
        if e == 1:
            for r in range(world):
                rows = np.asarray(out[r]["gh0_rows"])
                assert O.rel_err(np.asarray(out[r]["gh0"]), ref["grad_h"][0][rows]) < 1e-5
    np.testing.assert_allclose(out[0]["losses"], losses, rtol=1e-5)
    for l in range(2):
        assert O.rel_err(np.asarray(out[0]["W"][l]), W[l]) < 1e-5
