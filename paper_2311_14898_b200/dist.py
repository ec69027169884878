"""Host-side logic of the one-process-per-GPU (rank) mode.

In rank mode (``DeviceFleet(plan, rank=r)``) process r drives virtual device
r of the plan on its own GPU.  The data path needs no collective: peers'
slot buffers, neighbour-gradient views and weight-gradient accumulators are
mapped with CUDA IPC, and the Alg. 2/3 barriers are device-side counter
waits (``k_xbarrier``).  What remains for the host is small and lives here:

* exchanging the IPC handles once (``exchange``),
* summing the per-rank loss partials (``allreduce_sum``), and
* the invariant that makes per-process host stores valid: in p2p/full mode a
  device only ever reads or writes host rows it owns (``touched_rows``).

All of it runs over ``torch.distributed`` (gloo or NCCL) and is covered by
the world-size-2 gloo tests in tests/test_dist_host.py.
"""

from __future__ import annotations

import numpy as np

HT_IPC_BYTES = 256


def _dist():
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("rank mode needs torch.distributed to be initialised")
    return dist


def world() -> tuple[int, int]:
    dist = _dist()
    return dist.get_rank(), dist.get_world_size()


def exchange(blob: bytes) -> list:
    """All-gather one byte string per rank, returned in rank order."""
    dist = _dist()
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, bytes(blob))
    return out


def allreduce_sum(x: float) -> float:
    """Sum a float over ranks (float64 on the wire)."""
    import torch
    dist = _dist()
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return float(t.item())


def allreduce_max(x: float) -> float:
    import torch
    dist = _dist()
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    _dist().barrier()


def touched_rows(plan, i: int, mode: str = "full") -> np.ndarray:
    """Every host row device i reads or writes during an epoch: host loads
    (load/owned sets), destination and checkpoint rows, and flushes."""
    parts = []
    for j in range(plan.n):
        parts.append(plan.load_sets[i][j] if mode == "full" else plan.owned_sets[i][j])
        parts.append(plan.owned_sets[i][j])  # flush rows are a subset
        if plan.dest_sets is not None:
            parts.append(plan.dest_sets[i][j])
    return np.unique(np.concatenate(parts + [np.empty(0, np.int64)]))


def owns_all_touched(plan, i: int, mode: str = "full") -> bool:
    rows = touched_rows(plan, i, mode)
    return bool((plan.owner[rows] == i).all()) if rows.size else True
