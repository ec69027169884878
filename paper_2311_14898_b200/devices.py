"""Host-resident vertex store and the B200 device fleet.

Drop-in for ``chunktrain/devices.py``.  Where the reference simulates m
devices with numpy buffers, this fleet runs them for real:

* ``HostStore`` arrays live in pinned, portable, mapped host memory (or in
  HBM for the HongTu-IM variant, ``placement="device"``); GPUs read and
  write their rows directly (zero-copy over PCIe);
* each virtual device owns a slot buffer in HBM laid out by the plan;
  peer fetches are loads from the peer's buffer (NVLink P2P when the
  virtual devices sit on different GPUs, HBM when they share one);
* the forward/backward communication steps, barriers and flushes of
  Alg. 2/3 are executed by the native library (``ht_comm_fwd`` /
  ``ht_comm_bwd`` / ``ht_forward_layer`` / ``ht_backward_layer``).

Meters count rows and bytes exactly like the reference (devices.py:83-121)
and are derived from the same plan sets the kernels execute.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import CheckpointMissingError, DeviceError, SimulationError
from .planner import DedupPlan, _intersect, _isect_count, comm_cost, predicted_transfers

_MODES = ("baseline", "p2p", "full")
_FLUSH_POLICIES = ("on_eviction", "every_batch")
_MODE_ID = {"baseline": 0, "p2p": 1, "full": 2}
PRECISIONS = {"fp32": 0, "tf32": 1}


# ---------------------------------------------------------------------------
# HBM-resident arrays (placement="device")
# ---------------------------------------------------------------------------


class DeviceArray:
    """A (rows, cols) array in HBM, readable as numpy through __array__."""

    def __init__(self, shape, dtype, device: int = 0):
        self.shape = tuple(int(s) for s in shape)
        self.dtype = np.dtype(dtype)
        self.device = device
        self.nbytes = int(np.prod(self.shape, dtype=np.int64)) * self.dtype.itemsize
        p = C.c_void_p()
        N.call("ht_dev_alloc", device, max(self.nbytes, 16), C.byref(p), kind=DeviceError)
        self.device_ptr = int(p.value)
        weakref.finalize(self, N.lib().ht_dev_free, device, self.device_ptr)
        self.zero()

    def zero(self):
        N.call("ht_memset", self.device_ptr, 0, self.nbytes, kind=DeviceError)

    def __array__(self, dtype=None, copy=None):
        out = np.empty(self.shape, self.dtype)
        N.call("ht_memcpy", N.ptr(out), self.device_ptr, self.nbytes, kind=DeviceError)
        return out if dtype is None else out.astype(dtype)

    def __getitem__(self, idx):
        return np.asarray(self)[idx]

    def __setitem__(self, idx, value):
        if idx != slice(None) and idx is not Ellipsis:
            raise SimulationError("device-resident arrays support whole-array assignment only")
        src = np.ascontiguousarray(np.broadcast_to(np.asarray(value, self.dtype), self.shape))
        N.call("ht_memcpy", self.device_ptr, N.ptr(src), self.nbytes, kind=DeviceError)

    def copy(self):
        return np.asarray(self)

    @property
    def ndim(self):
        return len(self.shape)


# ---------------------------------------------------------------------------
# host store
# ---------------------------------------------------------------------------


def _zero_rows(a, rows):
    if isinstance(a, DeviceArray):
        if rows is None:
            a.zero()
        elif len(rows):
            host = np.asarray(a)
            host[rows] = 0
            a[:] = host
        return
    if rows is None:
        _parallel_zero(a)
    elif len(rows):
        a[rows] = 0


def _parallel_zero(a: np.ndarray, threads: int = 8):
    """Zero a large pinned array with several threads (numpy releases the GIL)."""
    flat = a.reshape(-1)
    if flat.size < (1 << 22):
        flat[:] = 0
        return
    step = (flat.size + threads - 1) // threads

    def work(t):
        flat[t * step:(t + 1) * step] = 0

    ts = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def _parallel_rows(dst: np.ndarray, src, threads: int = 8):
    """dst[:] = src (with dtype conversion) in row blocks on several threads:
    no full-size temporary, and memory-mapped sources stream in."""
    n = dst.shape[0]
    if n * dst.shape[1] < (1 << 22):
        dst[:] = src
        return
    step = (n + threads - 1) // threads

    def work(t):
        dst[t * step:(t + 1) * step] = src[t * step:(t + 1) * step]

    ts = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


class _Checkpoints(dict):
    """``HostStore.agg``: layer -> (V, d_l) checkpoint array.  When a fleet
    keeps an epoch's checkpoints in its HBM mirrors (``checkpoints="hbm"``),
    the host array is filled on first access, so readers see exactly the
    reference's contents (devices.py:391-404) without the epoch paying the
    device-to-host copy."""

    def __init__(self):
        super().__init__()
        self.pending = {}  # layer -> fleet holding that layer's checkpoints

    def _materialize(self, layer):
        fleet = self.pending.pop(layer, None)
        if fleet is not None:
            dst = dict.__getitem__(self, layer)
            # the fleet's mirrors must still hold this store's epoch: a fleet
            # materializes every other store's pending checkpoints before it
            # starts a new epoch (DeviceFleet.flush_checkpoints)
            if fleet._ckpt_shapes.get((id(self), layer)) != tuple(dst.shape):
                raise SimulationError(f"checkpoint of layer {layer} does not match the "
                                      f"fleet's mirrors")
            N.call("ht_fleet_checkpoint_read", fleet._handle, int(layer), N.ptr(dst),
                   kind=DeviceError)

    def materialize_all(self):
        for layer in list(self.pending):
            self._materialize(layer)

    def __getitem__(self, layer):
        self._materialize(layer)
        return dict.__getitem__(self, layer)

    def get(self, layer, default=None):
        return self[layer] if layer in self else default

    def values(self):
        self.materialize_all()
        return dict.values(self)

    def items(self):
        self.materialize_all()
        return dict.items(self)


class HostStore:
    """Per-layer representations h^l, gradients and aggregation checkpoints
    (devices.py:44-75).  Arrays are pinned host memory (``placement="host"``,
    the HongTu setting) or HBM (``placement="device"``, HongTu-IM)."""

    def __init__(self, num_vertices: int, dims: list, dtype=np.float64, placement: str = "host",
                 device: int = 0, rows=None):
        if placement not in ("host", "device"):
            raise SimulationError(f"unknown placement {placement!r}")
        self.num_vertices = int(num_vertices)
        self.dims = list(dims)
        self.dtype = np.dtype(dtype)
        self.placement = placement
        self.device = device
        # compact store (rank mode): only these vertices' rows, ascending -
        # row k of every array is vertex rows[k] (new; the reference keeps
        # all V rows in one process)
        self.rows = None
        if rows is not None:
            r = np.ascontiguousarray(rows, dtype=np.int64)
            if r.ndim != 1 or (r.size > 1 and np.any(r[1:] <= r[:-1])) or \
                    (r.size and (r[0] < 0 or r[-1] >= self.num_vertices)):
                raise SimulationError("HostStore rows must be ascending unique vertex ids")
            self.rows = r
        self.h = [self._alloc(d) for d in self.dims]
        self.grad_h = [self._alloc(d) for d in self.dims]
        self.h_valid = [False] * len(self.dims)
        self.agg = _Checkpoints()
        self.agg_written = set()

    def _alloc(self, d):
        shape = (self.num_vertices if self.rows is None else self.rows.size, d)
        if self.placement == "device":
            return DeviceArray(shape, self.dtype, self.device)
        return N.pinned_zeros(shape, self.dtype)

    def agg_array(self, layer: int):
        """The checkpoint array of `layer` (allocated on first use), without
        materializing HBM-held checkpoints."""
        if layer not in self.agg:
            self.agg[layer] = self._alloc(self.dims[layer])
        return dict.__getitem__(self.agg, layer)

    def set_features(self, features) -> None:
        X = features if isinstance(features, np.ndarray) else np.asarray(features)
        if self.rows is not None and X.ndim == 2 and X.shape[0] == self.num_vertices:
            X = X[self.rows]  # a compact store takes its rows of the full matrix
        if X.shape != tuple(self.h[0].shape):
            raise SimulationError(f"feature matrix shape {X.shape} does not match "
                                  f"(num_vertices, d0) = {tuple(self.h[0].shape)}")
        if isinstance(self.h[0], DeviceArray):
            self.h[0][:] = np.asarray(X, dtype=self.dtype)
        else:  # cast straight into the pinned rows, in parallel row blocks
            _parallel_rows(self.h[0], X)
        self.h_valid[0] = True

    def reset_epoch(self) -> None:
        """Invalidate h^{>=1}, zero every gradient, forget checkpoints."""
        for l in range(1, len(self.h)):
            self.h_valid[l] = False
        for g in self.grad_h:
            _zero_rows(g, None)
        self.agg_written.clear()
        self.agg.pending.clear()


# ---------------------------------------------------------------------------
# device fleet
# ---------------------------------------------------------------------------


@dataclass(eq=False)
class DeviceState:
    """Per-device transfer meters (devices.py:83-121)."""

    device_id: int
    h2d_rows: int = 0
    d2h_rows: int = 0
    d2d_rows: int = 0
    reuse_rows: int = 0
    dest_h2d_rows: int = 0
    dest_d2h_rows: int = 0
    chkpt_h2d_rows: int = 0
    chkpt_d2h_rows: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    d2d_bytes: int = 0
    dest_bytes: int = 0
    chkpt_bytes: int = 0
    peak_live_slots: int = 0
    buffer: object = None
    grad_buffer: object = None

    def counter_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "h2d_rows", "d2h_rows", "d2d_rows", "reuse_rows", "dest_h2d_rows", "dest_d2h_rows",
            "chkpt_h2d_rows", "chkpt_d2h_rows", "h2d_bytes", "d2h_bytes", "d2d_bytes",
            "dest_bytes", "chkpt_bytes", "peak_live_slots")}


class BufferInfo:
    """Shape/dtype descriptor of a device-resident slot buffer."""

    def __init__(self, shape, dtype):
        self.shape = tuple(shape)
        self.dtype = np.dtype(dtype)


# HBM owner cache: each device keeps HBM mirrors of the
# host rows it owns (layer inputs, checkpoints, gradients) and reads those
# instead of the host; every row produced is still written through to the
# HostStore.  "auto" enables it for host-resident stores in p2p/full mode
# when the mirrors fit in free HBM.
_CACHE_MODES = {"off": 0, "on": 1, "auto": 2}
_CKPT_MODES = ("auto", "host")


class DeviceFleet:
    """Executes a DedupPlan over m virtual devices on the GPU(s)
    (devices.py:129-488).  ``devices[i]`` maps virtual device i to a CUDA
    ordinal (default: round-robin over the visible GPUs)."""

    def __init__(self, plan: DedupPlan, mode: str = "full", flush_policy: str = "on_eviction",
                 dtype=np.float64, devices=None, precision: str = "tf32", rank: int | None = None,
                 cache: str = "auto", lean: bool = False, checkpoints: str = "auto",
                 hbm_budget_gb: float | None = None):
        if mode not in _MODES:
            raise SimulationError(f"unknown mode {mode!r}")
        if flush_policy not in _FLUSH_POLICIES:
            raise SimulationError(f"unknown flush policy {flush_policy!r}")
        if precision not in PRECISIONS:
            raise SimulationError(f"unknown precision {precision!r}, expected one of {list(PRECISIONS)}")
        if cache not in _CACHE_MODES:
            raise SimulationError(f"unknown cache mode {cache!r}, expected one of {list(_CACHE_MODES)}")
        if checkpoints not in _CKPT_MODES:
            raise SimulationError(f"unknown checkpoint placement {checkpoints!r}, expected one "
                                  f"of {list(_CKPT_MODES)}")
        self.plan = plan
        self.mode = mode
        self.cache = cache
        # GCN agg checkpoints: "auto" keeps them in the owner cache's HBM
        # mirrors when it is active (host.agg filled on first read), "host"
        # always writes them through (devices.py:391-404)
        self.checkpoints = checkpoints
        # recompute-cache hybrid: cap on the owner cache's
        # HBM per device; agg^l mirrors that do not fit are recomputed in the
        # backward (one device) - see recompute_layers
        if hbm_budget_gb is not None and not hbm_budget_gb > 0:
            raise SimulationError(f"hbm_budget_gb must be positive, got {hbm_budget_gb!r}")
        self.hbm_budget_gb = hbm_budget_gb
        self.recompute_layers: list = []  # set per epoch by train_epoch
        self._ckpt_hosts = weakref.WeakSet()
        self._ckpt_shapes = {}  # (id(host.agg), layer) -> shape the mirrors hold
        # lean epochs (opt-in): no grad_h^0, and no host copies of h^L /
        # grad_h^L with the owner cache; the transfer
        # meters stay the reference's
        self.lean = bool(lean)
        self.flush_policy = flush_policy
        self.dtype = np.dtype(dtype)
        self.precision = precision
        self.m, self.n = plan.m, plan.n
        self.devices = [DeviceState(i) for i in range(self.m)]
        ngpu = N.device_count()
        if ngpu < 1:
            raise DeviceError("no CUDA device visible; the fleet runs on B200 GPUs only")
        # rank mode: this process drives virtual device `rank` only (one
        # process per GPU); peers are other processes (see dist.py)
        self.rank = rank
        if rank is not None:
            if not 0 <= rank < self.m:
                raise SimulationError(f"rank {rank} outside the plan's {self.m} devices")
            if mode == "baseline":
                raise SimulationError("rank mode needs mode 'p2p' or 'full'")
            import os
            local = int(os.environ.get("LOCAL_RANK", rank))
            self.ordinals = [list(devices)[0] if devices is not None else local % ngpu]
        else:
            self.ordinals = list(devices) if devices is not None else [i % ngpu for i in range(self.m)]
        self._ipc_ready = rank is None or self.m == 1
        self.cache_active = False  # set per epoch by train_epoch
        self._handle = None
        self._create_native()
        self._precompute_meters()
        self._dim = None
        self._fwd_next = None
        self._bwd_next = None
        self._attached = None

    # -- native state ---------------------------------------------------------
    def _create_native(self):
        plan = self.plan
        h = C.c_void_p()
        flush = 0 if self.flush_policy == "on_eviction" else 1
        if self.rank is not None:
            N.call("ht_fleet_create_rank", self.m, self.n, self.rank, self.ordinals[0],
                   _MODE_ID[self.mode], flush, C.byref(h))
        else:
            ords = (C.c_int * self.m)(*self.ordinals)
            N.call("ht_fleet_create", self.m, self.n, ords, _MODE_ID[self.mode], flush, C.byref(h))
        self._handle = h.value
        self._finalizer = weakref.finalize(self, N.lib().ht_fleet_destroy, self._handle)
        keep = []

        def arr(a):
            a = np.ascontiguousarray(a, dtype=np.int64)
            keep.append(a)
            return a

        for i in range(self.m):
            for j in range(self.n):
                nb = arr(plan.neighbor_sets[i][j])
                ow = arr(plan.owned_sets[i][j])
                ld = arr(plan.load_sets[i][j])
                nc = arr(plan.nbr_carry_sets[i][j])
                lv = arr(plan.layout.live_sets[i][j])
                sl = arr(plan.layout.slots[i][j])
                if plan.dest_sets is not None:
                    de = arr(plan.dest_sets[i][j])
                    dp, dn = N.ptr(de), de.size
                else:
                    dp, dn = None, -1
                N.call("ht_fleet_set_sets", self._handle, i, j, N.ptr(nb), nb.size, N.ptr(ow),
                       ow.size, N.ptr(ld), ld.size, N.ptr(nc), nc.size, N.ptr(lv), N.ptr(sl),
                       lv.size, dp, dn)
                for k, rows in plan.fetch_sets[i][j].items():
                    r = arr(rows)
                    N.call("ht_fleet_set_fetch", self._handle, i, j, int(k), N.ptr(r), r.size)
        N.call("ht_fleet_finalize", self._handle)
        keep.clear()

    def _precompute_meters(self):
        plan, m, n = self.plan, self.m, self.n
        z = lambda: [[0] * n for _ in range(m)]  # noqa: E731
        self._m_h2d, self._m_reuse, self._m_fd2d = z(), z(), z()
        self._m_bd2d, self._m_d2h, self._m_live = z(), z(), z()
        for i in range(m):
            for j in range(n):
                nn = int(plan.neighbor_sets[i][j].size)
                if self.mode == "baseline":
                    self._m_h2d[i][j] = nn
                    self._m_d2h[i][j] = nn
                    self._m_live[i][j] = nn
                    continue
                self._m_live[i][j] = int(plan.live_set(i, j).size)
                fetch = plan.fetch_sets[i][j]
                self._m_bd2d[i][j] = sum(int(f.size) for f in fetch.values())
                if self.mode == "full":
                    self._m_h2d[i][j] = int(plan.load_sets[i][j].size)
                    self._m_reuse[i][j] = int(plan.carry_sets[i][j].size)
                    nc = plan.nbr_carry_sets[i][j]
                    self._m_fd2d[i][j] = sum(int(f.size) - _isect_count(f, nc) for f in fetch.values())
                else:
                    self._m_h2d[i][j] = int(plan.owned_sets[i][j].size)
                    self._m_fd2d[i][j] = self._m_bd2d[i][j]
                owned = plan.owned_sets[i][j]
                if self.mode == "p2p" or self.flush_policy == "every_batch" or j + 1 == n:
                    self._m_d2h[i][j] = int(owned.size)
                else:
                    self._m_d2h[i][j] = int(owned.size) - _isect_count(owned, plan.owned_sets[i][j + 1])

    def capacity(self, i: int) -> int:
        c = C.c_int64(0)
        N.call("ht_fleet_capacity", self._handle, i, C.byref(c))
        return int(c.value)

    def flush_checkpoints(self, keep=None) -> None:
        """Copy every HBM-held checkpoint this fleet owes a host store into
        that store's agg arrays (all stores but `keep`, whose epoch is about
        to be replaced anyway).  Called before the fleet's mirrors change: at
        the start of every epoch and at close (the reference keeps agg per
        store, so a store's reads must never see another store's epoch)."""
        for host in list(self._ckpt_hosts):
            if host is keep:
                continue
            for layer, fl in list(host.agg.pending.items()):
                if fl is self:
                    host.agg._materialize(layer)
            self._ckpt_hosts.discard(host)

    def close(self) -> None:
        """Release the fleet's device buffers now (otherwise at garbage
        collection)."""
        if self._handle is not None and self._finalizer.alive:
            self.flush_checkpoints()  # HBM-held checkpoints -> host first
            self._finalizer()

    # -- meters ---------------------------------------------------------------
    def _meter_fwd(self, j: int, row_bytes: int):
        for i, dev in enumerate(self.devices):
            h2d = self._m_h2d[i][j]
            dev.h2d_rows += h2d
            dev.h2d_bytes += h2d * row_bytes
            dev.reuse_rows += self._m_reuse[i][j]
            dev.d2d_rows += self._m_fd2d[i][j]
            dev.d2d_bytes += self._m_fd2d[i][j] * row_bytes
            dev.peak_live_slots = max(dev.peak_live_slots, self._m_live[i][j])

    def _meter_bwd(self, j: int, row_bytes: int):
        for i, dev in enumerate(self.devices):
            dev.d2d_rows += self._m_bd2d[i][j]
            dev.d2d_bytes += self._m_bd2d[i][j] * row_bytes
            dev.d2h_rows += self._m_d2h[i][j]
            dev.d2h_bytes += self._m_d2h[i][j] * row_bytes
            dev.peak_live_slots = max(dev.peak_live_slots, self._m_live[i][j])

    def _meter_dest(self, j: int, row_bytes: int, direction: str, klass: str = "dest"):
        for i, dev in enumerate(self.devices):
            nv = int(self.plan.dest_sets[i][j].size)
            setattr(dev, f"{klass}_{direction}_rows", getattr(dev, f"{klass}_{direction}_rows") + nv)
            setattr(dev, f"{klass}_bytes", getattr(dev, f"{klass}_bytes") + nv * row_bytes)

    # -- layer lifecycle --------------------------------------------------------
    def begin_forward_layer(self, dim: int) -> None:
        self._dim = int(dim)
        N.call("ht_begin_layer", self._handle, self._dim, self.dtype.itemsize, 0)
        self._set_buffers(False)
        self._fwd_next = 0

    def begin_backward_layer(self, dim: int) -> None:
        self._dim = int(dim)
        N.call("ht_begin_layer", self._handle, self._dim, self.dtype.itemsize, 1)
        self._set_buffers(self.mode != "baseline")
        self._fwd_next = 0
        self._bwd_next = 0

    def _set_buffers(self, grads: bool):
        for i, dev in enumerate(self.devices):
            cap = self.capacity(i)
            dev.buffer = BufferInfo((cap, self._dim), self.dtype)
            if grads:
                dev.grad_buffer = BufferInfo((cap, self._dim), self.dtype)

    def _check_seq(self, kind: str, batch: int) -> None:
        expected = self._fwd_next if kind == "fwd" else self._bwd_next
        if expected is None or batch != expected:
            raise SimulationError(
                f"{kind} communication for batch {batch} out of order "
                f"(expected {expected}); batches must run 0..n-1 after a layer begin")

    def _check_dim(self, a):
        if a.ndim != 2 or a.shape[1] != self._dim:
            raise SimulationError(f"rows of width {a.shape[1] if a.ndim == 2 else '?'} do not "
                                  f"match the layer width {self._dim}")

    # -- communication (Alg. 2 / Alg. 3) ---------------------------------------
    def dedup_comm_fwd(self, host_rows, batch: int) -> list:
        """Stage batch rows on the devices; returns each device's N_ij view
        (copies, bitwise equal to host_rows[N_ij])."""
        self._check_seq("fwd", batch)
        self._check_dim(host_rows)
        self._fwd_next = batch + 1 if batch + 1 < self.n else None
        j = batch
        src = N.staged(host_rows, self.dtype)
        sizes = [int(self.plan.neighbor_sets[i][j].size) for i in range(self.m)]
        out = N.pinned_empty((sum(sizes), self._dim), self.dtype)
        N.call("ht_comm_fwd", self._handle, j, N.ptr(src), N.ptr(out))
        row_bytes = host_rows.shape[1] * np.dtype(host_rows.dtype).itemsize
        self._meter_fwd(j, row_bytes)
        views, o = [], 0
        for s in sizes:
            views.append(np.array(out[o:o + s]))
            o += s
        return views

    def dedup_comm_bwd(self, grad_views: list, host_grad, batch: int) -> None:
        """Push neighbour gradients to owners (ascending source device), then
        flush completed rows into host_grad (devices.py:284-341)."""
        self._check_seq("bwd", batch)
        self._check_dim(host_grad)
        self._bwd_next = batch + 1 if batch + 1 < self.n else None
        j = batch
        views = N.staged(np.concatenate([np.asarray(v, self.dtype).reshape(-1, self._dim)
                                         for v in grad_views]), self.dtype)
        tgt = N.staged(host_grad, self.dtype)
        N.call("ht_comm_bwd", self._handle, j, N.ptr(views), N.ptr(tgt))
        if tgt is not host_grad:
            host_grad[...] = tgt
        row_bytes = host_grad.shape[1] * np.dtype(host_grad.dtype).itemsize
        self._meter_bwd(j, row_bytes)

    # -- destination rows and checkpoints --------------------------------------
    def _dest(self, i: int, j: int):
        if self.plan.dest_sets is None:
            raise SimulationError("plan carries no destination sets; build it from a "
                                  "partition to run training traffic")
        return self.plan.dest_sets[i][j]

    def _dest_op(self, op, batch, host_rows, rows_cat):
        self._dest(0, batch)
        d = host_rows.shape[1]
        N.call("ht_dest_rows", self._handle, op, batch, d, np.dtype(host_rows.dtype).itemsize,
               N.ptr(host_rows), N.ptr(rows_cat))

    def load_dest_rows(self, host_rows, batch: int) -> list:
        sizes = [int(self._dest(i, batch).size) for i in range(self.m)]
        src = N.staged(host_rows)
        out = N.pinned_empty((sum(sizes), host_rows.shape[1]), src.dtype)
        self._dest_op(0, batch, src, out)
        self._meter_dest(batch, host_rows.shape[1] * src.dtype.itemsize, "h2d")
        res, o = [], 0
        for s in sizes:
            res.append(np.array(out[o:o + s]))
            o += s
        return res

    def _rows_cat(self, rows, dtype, d):
        return N.staged(np.concatenate([np.asarray(r, dtype).reshape(-1, d) for r in rows]), dtype)

    def store_dest_rows(self, host_rows, batch: int, rows: list) -> None:
        self._dest(0, batch)
        tgt = N.staged(host_rows)
        cat = self._rows_cat(rows, tgt.dtype, host_rows.shape[1])
        self._dest_op(1, batch, tgt, cat)
        if tgt is not host_rows:
            host_rows[...] = tgt
        self._meter_dest(batch, host_rows.shape[1] * tgt.dtype.itemsize, "d2h")

    def add_dest_grads(self, host_grad, batch: int, rows: list) -> None:
        self._dest(0, batch)
        tgt = N.staged(host_grad)
        cat = self._rows_cat(rows, tgt.dtype, host_grad.shape[1])
        self._dest_op(2, batch, tgt, cat)
        if tgt is not host_grad:
            host_grad[...] = tgt
        self._meter_dest(batch, host_grad.shape[1] * tgt.dtype.itemsize, "d2h")

    def store_checkpoint(self, host: HostStore, layer: int, batch: int, agg_rows: list) -> None:
        arr = host.agg_array(layer)
        self._dest(0, batch)
        cat = self._rows_cat(agg_rows, host.dtype, host.dims[layer])
        self._dest_op(1, batch, arr, cat)
        for i in range(self.m):
            host.agg_written.add((layer, i, batch))
        self._meter_dest(batch, host.dims[layer] * host.dtype.itemsize, "d2h", "chkpt")

    def load_recomp_chkpt(self, host: HostStore, kind: str, layer: int, batch: int):
        if kind == "gcn":
            for i in range(self.m):
                if (layer, i, batch) not in host.agg_written:
                    raise CheckpointMissingError(layer, i, batch)
            arr = host.agg[layer]
            sizes = [int(self._dest(i, batch).size) for i in range(self.m)]
            out = N.pinned_empty((sum(sizes), host.dims[layer]), host.dtype)
            self._dest_op(0, batch, arr, out)
            self._meter_dest(batch, host.dims[layer] * host.dtype.itemsize, "h2d", "chkpt")
            res, o = [], 0
            for s in sizes:
                res.append(np.array(out[o:o + s]))
                o += s
            return res
        if kind == "gat":
            if not host.h_valid[layer]:
                raise CheckpointMissingError(layer, 0, batch)
            h_nbr = self.dedup_comm_fwd(host.h[layer], batch)
            h_dst = self.load_dest_rows(host.h[layer], batch)
            return h_nbr, h_dst
        raise SimulationError(f"unknown model kind {kind!r}")

    # -- training-path attachment --------------------------------------------------
    def attach_partition(self, p) -> None:
        """Upload the chunk CSC/CSR structure of the partition this plan was
        built from (once per fleet); the layer kernels need it."""
        if self._attached is p:
            return
        if p.m != self.m or p.n != self.n:
            raise SimulationError("partition grid does not match the fleet's plan")
        for i in range(self.m):
            for j in range(self.n):
                c = p.chunks[i][j]
                if not np.array_equal(c.sources, self.plan.neighbor_sets[i][j]):
                    raise SimulationError(f"chunk ({i},{j}) neighbour set differs from the plan")
                if self.plan.dest_sets is None or not np.array_equal(c.vertices, self.plan.dest_sets[i][j]):
                    raise SimulationError("plan carries no destination sets matching the partition")
                arrs = [np.ascontiguousarray(a, dtype=t) for a, t in (
                    (c.csc_offsets, np.int64), (c.csc_local_src, np.int64), (c.edge_weights, np.float64),
                    (c.csr_offsets, np.int64), (c.csr_local_dst, np.int64), (c.csr_edge_perm, np.int64))]
                N.call("ht_fleet_set_chunk", self._handle, i, j, c.num_vertices, int(c.sources.size),
                       c.num_edges, *[N.ptr(a) for a in arrs])
        N.call("ht_fleet_finalize", self._handle)
        self._attached = p
        # rows of the vertex set no chunk reads: their gradients stay zero
        touched = np.zeros(self.plan.owner.shape[0], dtype=bool)
        for u in self.plan.union_sets:
            touched[u] = True
        self._untouched = np.flatnonzero(~touched)

    def connect_peers(self) -> None:
        """Rank mode: exchange CUDA IPC handles of the shared device buffers
        with every peer rank (once; buffers are sized by the first
        ht_epoch_begin and never move afterwards)."""
        if self._ipc_ready:
            return
        from . import dist
        mine = (C.c_byte * dist.HT_IPC_BYTES)()
        N.call("ht_fleet_ipc_export", self._handle, mine)
        blobs = dist.exchange(bytes(mine))
        for k, blob in enumerate(blobs):
            if k != self.rank:
                buf = (C.c_byte * dist.HT_IPC_BYTES).from_buffer_copy(blob)
                N.call("ht_fleet_ipc_import", self._handle, k, buf)
        self._ipc_ready = True

    def set_timing(self, enabled: bool) -> None:
        N.call("ht_set_timing", self._handle, int(bool(enabled)))

    def kernel_stats(self, which: int):
        lc, ms, by = C.c_int64(0), C.c_double(0), C.c_double(0)
        N.call("ht_kernel_stats", self._handle, which, C.byref(lc), C.byref(ms), C.byref(by))
        return int(lc.value), float(ms.value), float(by.value)

    # -- reporting ------------------------------------------------------------------
    def transfer_report(self, fwd_passes: int = 0, bwd_passes: int = 0, cost_params=None) -> dict:
        per_device = [dev.counter_dict() for dev in self.devices]
        totals: dict = {}
        for rec in per_device:
            for k, v in rec.items():
                if k != "peak_live_slots":
                    totals[k] = totals.get(k, 0) + v
        rep = {
            "mode": self.mode, "per_device": per_device, "totals": totals,
            "peak_live_slots": [dev.peak_live_slots for dev in self.devices],
            "volumes": {"v_ori": self.plan.volumes.v_ori, "v_p2p": self.plan.volumes.v_p2p,
                        "v_ru": self.plan.volumes.v_ru},
        }
        if cost_params is not None:
            rep["predicted_cost_per_layer"] = comm_cost(self.plan.volumes, cost_params)
        if fwd_passes or bwd_passes:
            pred = predicted_transfers(self.plan, self.mode)
            expected = {
                "h2d_rows": fwd_passes * pred["fwd_h2d_rows"],
                "d2h_rows": bwd_passes * pred["bwd_d2h_rows"],
                "d2d_rows": fwd_passes * pred["fwd_d2d_rows"] + bwd_passes * pred["bwd_d2d_rows"],
                "reuse_rows": fwd_passes * pred["fwd_reuse_rows"],
            }
            rep["expected"] = expected
            rep["planner_consistent"] = all(totals[k] == v for k, v in expected.items()) and all(
                dev.peak_live_slots == pred["peak_slots"][i] for i, dev in enumerate(self.devices))
        return rep


__all__ = ["DeviceArray", "DeviceFleet", "DeviceState", "HostStore", "PRECISIONS", "_intersect"]
