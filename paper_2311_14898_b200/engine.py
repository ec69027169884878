"""Model configuration and the partitioned full-graph GCN epoch on B200.

Drop-in for the training entry points of ``chunktrain/engine.py``
(``ModelConfig``, ``init_model``, ``train_epoch``, ``EpochResult``,
``ActivationTracker``, ``sync_and_update``, ``comm_passes_per_epoch`` and
the HTF1/HTL1 matrix files).  ``train_epoch`` drives the native layer
kernels through the C ABI: per layer one call runs every batch of the
chunk grid on the GPU(s), so Python only does bookkeeping (meters,
sequencing, tracker) per batch.
"""

from __future__ import annotations

import ctypes as C
import struct
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .devices import PRECISIONS, DeviceArray, DeviceFleet, HostStore, _zero_rows
from .errors import GraphFormatError, SimulationError
from .partition import TwoLevelPartition

KINDS = ("gcn", "gat")


@dataclass(eq=False)
class ModelConfig:
    """Layer widths plus the replicated parameters (engine.py:37-69)."""

    kind: str
    dims: list
    weights: list
    attn: list | None
    leaky_slope: float = 0.2
    lr: float = 0.1
    epochs: int = 1
    seed: int = 0

    @property
    def num_layers(self) -> int:
        return len(self.dims) - 1

    def copy(self) -> "ModelConfig":
        return ModelConfig(kind=self.kind, dims=list(self.dims),
                           weights=[w.copy() for w in self.weights],
                           attn=None if self.attn is None else [a.copy() for a in self.attn],
                           leaky_slope=self.leaky_slope, lr=self.lr, epochs=self.epochs,
                           seed=self.seed)


def init_model(kind: str, dims: list, seed: int, *, lr: float = 0.1, epochs: int = 1,
               leaky_slope: float = 0.2, dtype=np.float64) -> ModelConfig:
    """Seeded Glorot-uniform weights, drawn in float64 in the order W (then
    attention) layer by layer, then cast (engine.py:72-99)."""
    if kind not in KINDS:
        raise SimulationError(f"unknown model kind {kind!r}")
    if len(dims) < 2:
        raise SimulationError("dims needs at least an input and output width")
    dtype = np.dtype(dtype)
    gen = np.random.default_rng(seed)
    weights, attn = [], ([] if kind == "gat" else None)
    for a, b in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(6.0 / (a + b))
        weights.append(gen.uniform(-lim, lim, size=(a, b)).astype(dtype))
        if kind == "gat":
            la = np.sqrt(6.0 / (2 * b + 1))
            attn.append(gen.uniform(-la, la, size=2 * b).astype(dtype))
    return ModelConfig(kind=kind, dims=list(dims), weights=weights, attn=attn,
                       leaky_slope=leaky_slope, lr=lr, epochs=epochs, seed=seed)


class ActivationTracker:
    """Counts live chunk intermediates (engine.py:352-372)."""

    def __init__(self):
        self._live = set()
        self.peak = 0

    def acquire(self, tag) -> None:
        if tag in self._live:
            raise SimulationError(f"intermediate {tag} acquired twice")
        self._live.add(tag)
        self.peak = max(self.peak, len(self._live))

    def release(self, tag) -> None:
        self._live.discard(tag)

    @property
    def live_count(self) -> int:
        return len(self._live)


@dataclass(eq=False)
class EpochResult:
    loss: float
    model: ModelConfig
    tracker: ActivationTracker = field(default_factory=ActivationTracker)
    grads: list | None = None        # summed weight gradients of this epoch (new)
    attn_grads: list | None = None   # GAT: summed attention-vector gradients (new)


def sync_and_update(model: ModelConfig, device_grads: list, lr: float | None = None) -> ModelConfig:
    """Replica-gradient sum in ascending device order + plain SGD
    (engine.py:328-344), for callers holding per-device gradients."""
    lr = model.lr if lr is None else lr
    for l in range(model.num_layers):
        tot = np.zeros_like(model.weights[l])
        for dg in device_grads:
            tot += dg["W"][l]
        model.weights[l] -= lr * tot
        if model.kind == "gat":
            ta = np.zeros_like(model.attn[l])
            for dg in device_grads:
                ta += dg["a"][l]
            model.attn[l] -= lr * ta
    return model


def comm_passes_per_epoch(model: ModelConfig) -> tuple:
    L = model.num_layers
    return (2 * L, L) if model.kind == "gat" else (L, L)


def _epoch_reset(host: HostStore, fleet: DeviceFleet, kind: str = "gcn",
                 cached: bool = False) -> None:
    """reset_epoch with the same observable result but without rewriting
    rows the epoch overwrites anyway: the loss writes every row of
    grad_h[L], and in p2p/full GCN mode the first flush of a row stores it,
    so only rows no chunk ever reads need explicit zeros.  GAT adds
    destination-input gradients into the host rows before the flushes, so
    every flush is a read-modify-write there and all rows are zeroed.  With
    the HBM owner cache every owned row of every gradient array is written
    through from a zeroed mirror, so nothing needs zeroing."""
    L = len(host.dims) - 1
    for l in range(1, len(host.h)):
        host.h_valid[l] = False
    host.agg_written.clear()
    host.agg.pending.clear()
    if cached:
        return
    for l in range(L):
        g = host.grad_h[l]
        if isinstance(g, DeviceArray) or fleet.mode == "baseline" or kind == "gat":
            _zero_rows(g, None)
        else:
            _zero_rows(g, fleet._untouched)


def _loss(h_, host: HostStore, dims: list, labels, mask) -> None:
    """Validate labels/mask the way the reference's indexing does
    (engine.py:308-315: ``h_last[mask]`` and ``p[arange, y]`` raise
    IndexError; negative labels index from the end), then enqueue the
    device loss."""
    mask_b = np.ascontiguousarray(np.asarray(mask, dtype=bool))
    labels_i = np.ascontiguousarray(np.asarray(labels, dtype=np.int64))
    V = int(host.num_vertices)
    L = len(dims) - 1
    if mask_b.ndim != 1 or mask_b.shape[0] != V:
        raise IndexError(f"boolean index did not match: mask has shape {mask_b.shape}, "
                         f"expected ({V},)")
    if labels_i.ndim != 1 or labels_i.shape[0] != V:
        raise IndexError(f"labels have shape {labels_i.shape}, expected ({V},)")
    count = int(mask_b.sum())
    if count == 0:
        warnings.warn("training mask is empty; loss is 0", stacklevel=3)
    else:
        y = labels_i[mask_b]
        lo, hi = int(y.min()), int(y.max())
        if lo < -dims[L] or hi >= dims[L]:
            bad = lo if lo < -dims[L] else hi
            raise IndexError(f"index {bad} is out of bounds for axis 1 with size {dims[L]}")
        if lo < 0:  # numpy fancy indexing wraps negative labels
            labels_i = np.where(labels_i < 0, labels_i + dims[L], labels_i)
    N.call("ht_loss", h_, dims[L], N.ptr(labels_i), N.ptr(mask_b.view(np.uint8)),
           int(host.num_vertices), count, N.ptr(host.grad_h[L]), None)  # value read after SGD


def _f32_params(params: list, shapes: list) -> list:
    out = []
    for k, (x, shp) in enumerate(zip(params, shapes)):
        if x.dtype != np.float32 or not x.flags.c_contiguous or x.shape != shp:
            params[k] = np.ascontiguousarray(x, dtype=np.float32).reshape(shp)
        out.append(params[k])
    return out


def train_epoch(p: TwoLevelPartition, fleet: DeviceFleet, model: ModelConfig, host: HostStore,
                labels: np.ndarray, mask: np.ndarray,
                tracker: ActivationTracker | None = None) -> EpochResult:
    """One full-graph epoch over the chunk grid on the GPU (engine.py:387-480).

    GCN forward: per layer, every batch stages its deduplicated neighbour
    rows (host loads, barrier, peer fetches, barrier), aggregates them,
    applies z = agg.W and ReLU, and writes h^{l+1} and the agg checkpoint
    rows to the host store.  Loss on the last layer.  Backward: checkpoint
    and dest-gradient reload, hybrid recompute, transposed aggregation,
    owner push and flush into grad_h[l].  GAT (engine.py:418-423, 455-470):
    the forward also loads destination inputs and aggregates with edge
    softmax attention; no checkpoints; the backward re-stages the layer
    inputs through the forward machinery, recomputes, adds the
    destination-input gradients to the host and then pushes/flushes the
    neighbour gradients.  Then the ascending-device gradient sum and the
    SGD step (W, and the attention vectors for GAT), in place.
    """
    if tracker is None:
        tracker = ActivationTracker()
    if model.kind not in KINDS:
        raise SimulationError(f"unknown model kind {model.kind!r}")
    if not host.h_valid[0]:
        raise SimulationError("host features not set; call set_features first")
    if host.dtype != np.float32 or fleet.dtype != np.float32:
        raise SimulationError("the B200 path computes in float32; build HostStore and "
                              "DeviceFleet with dtype=np.float32")
    m, n, L = p.m, p.n, model.num_layers
    dims = [int(d) for d in model.dims]
    if list(host.dims) != dims:
        raise SimulationError("host store widths do not match the model")
    gat = model.kind == "gat"
    W = _f32_params(model.weights, [(dims[l], dims[l + 1]) for l in range(L)])
    A = _f32_params(model.attn, [(2 * dims[l + 1],) for l in range(L)]) if gat else None
    prec = PRECISIONS[fleet.precision]
    fleet.attach_partition(p)
    fleet.flush_checkpoints(keep=host)  # other stores' HBM-held checkpoints, before reuse
    h_ = fleet._handle
    item = host.dtype.itemsize
    dims_c = (C.c_int * (L + 1))(*dims)
    # HBM owner cache ("auto": host-resident stores only - an HBM store needs
    # no mirror; the native side refuses plans that do not admit it)
    from .devices import _CACHE_MODES
    want = _CACHE_MODES[fleet.cache]
    if fleet.cache == "auto" and host.placement != "host":
        want = 0
    if host.rows is not None:  # compact store: host row k = owned row k (needs the cache)
        want = 1
        if getattr(fleet, "_compact_for", None) is not host:
            N.call("ht_fleet_set_host_rows", h_, N.ptr(host.rows), int(host.rows.size))
            fleet._compact_for = host
    elif getattr(fleet, "_compact_for", None) is not None:
        N.call("ht_fleet_set_host_rows", h_, None, 0)
        fleet._compact_for = None
    # an HBM store on one device is used in place as the owner-cache mirror
    alias = host.placement == "device" and fleet.m == 1 and fleet.cache != "off" and \
        host.rows is None and fleet.mode != "baseline"
    if alias:
        hp = (C.c_void_p * (L + 1))(*[N.ptr(x) for x in host.h])
        gp_ = (C.c_void_p * (L + 1))(*[N.ptr(x) for x in host.grad_h])
        ap_ = None if gat else (C.c_void_p * L)(*[N.ptr(host.agg_array(l)) for l in range(L)])
        N.call("ht_fleet_alias_store", h_, L, hp, ap_, gp_)
    else:
        N.call("ht_fleet_alias_store", h_, L, None, None, None)
    N.call("ht_fleet_set_cache", h_, want)
    N.call("ht_fleet_set_budget", h_,
           0 if fleet.hbm_budget_gb is None else int(fleet.hbm_budget_gb * (1 << 30)))
    N.call("ht_fleet_set_lean", h_, int(fleet.lean))
    N.call("ht_gat_epoch_begin" if gat else "ht_epoch_begin", h_, L, dims_c)
    on = C.c_int(0)
    N.call("ht_fleet_cache_state", h_, C.byref(on))
    fleet.cache_active = bool(on.value)
    rmask = C.c_int64(0)
    N.call("ht_fleet_recompute_state", h_, C.byref(rmask))
    fleet.recompute_layers = [l for l in range(L) if (rmask.value >> l) & 1]
    # checkpoint tier: with the owner cache the agg checkpoints stay in HBM
    # (the hybrid sized to 180 GB); host.agg is filled from there on read
    ckpt_hbm = fleet.cache_active and fleet.checkpoints == "auto" and not gat
    N.call("ht_fleet_set_checkpoints", h_, int(ckpt_hbm))
    _epoch_reset(host, fleet, model.kind, fleet.cache_active)
    fleet.connect_peers()  # rank mode: IPC handles, once
    slope = C.c_float(model.leaky_slope)

    def chunks(kind_tag, l):
        for j in range(n):
            for i in range(m):
                tag = (kind_tag, l, i, j)
                tracker.acquire(tag)
                tracker.release(tag)

    # ---- forward (Alg. 1 lines 4-9) ----
    for l in range(L):
        fleet._dim = dims[l]
        fleet._fwd_next = None
        if gat:
            N.call("ht_gat_forward_layer", h_, l, dims[l], dims[l + 1], N.ptr(W[l]), N.ptr(A[l]),
                   slope, N.ptr(host.h[l]), N.ptr(host.h[l + 1]), prec)
            for j in range(n):
                fleet._meter_fwd(j, dims[l] * item)
                fleet._meter_dest(j, dims[l] * item, "h2d")
                fleet._meter_dest(j, dims[l + 1] * item, "d2h")
        else:
            agg = host.agg_array(l)
            N.call("ht_forward_layer", h_, l, dims[l], dims[l + 1], N.ptr(W[l]), N.ptr(host.h[l]),
                   N.ptr(host.h[l + 1]), N.ptr(agg), prec)
            if ckpt_hbm:
                host.agg.pending[l] = fleet
                fleet._ckpt_hosts.add(host)
                fleet._ckpt_shapes[(id(host.agg), l)] = tuple(agg.shape)
            for j in range(n):
                fleet._meter_fwd(j, dims[l] * item)
                for i in range(m):
                    host.agg_written.add((l, i, j))
                fleet._meter_dest(j, dims[l + 1] * item, "d2h")
                fleet._meter_dest(j, dims[l] * item, "d2h", "chkpt")
        chunks("fwd", l)
        host.h_valid[l + 1] = True

    # ---- loss ----
    _loss(h_, host, dims, labels, mask)

    # ---- backward (Alg. 1 lines 12-20) ----
    for l in reversed(range(L)):
        fleet._dim = dims[l]
        if gat:
            N.call("ht_gat_backward_layer", h_, l, dims[l], dims[l + 1], N.ptr(W[l]), N.ptr(A[l]),
                   slope, N.ptr(host.h[l]), N.ptr(host.grad_h[l + 1]), N.ptr(host.grad_h[l]),
                   prec)
            for j in range(n):
                fleet._meter_fwd(j, dims[l] * item)          # inputs re-staged
                fleet._meter_dest(j, dims[l] * item, "h2d")  # destination inputs
                fleet._meter_dest(j, dims[l + 1] * item, "h2d")
                fleet._meter_dest(j, dims[l] * item, "d2h")  # add_dest_grads
                fleet._meter_bwd(j, dims[l] * item)
        else:
            N.call("ht_backward_layer", h_, l, dims[l], dims[l + 1], N.ptr(W[l]),
                   N.ptr(host.agg_array(l)), N.ptr(host.grad_h[l + 1]), N.ptr(host.grad_h[l]),
                   prec)
            for j in range(n):
                fleet._meter_dest(j, dims[l] * item, "h2d", "chkpt")
                fleet._meter_dest(j, dims[l + 1] * item, "h2d")
                fleet._meter_bwd(j, dims[l] * item)
        chunks("bwd", l)
    fleet._fwd_next = fleet._bwd_next = None

    # ---- replica gradient sum + SGD (engine.py:479) ----
    grads = [np.empty_like(w) for w in W]
    wp = (C.c_void_p * L)(*[N.ptr(w) for w in W])
    gp = (C.c_void_p * L)(*[N.ptr(g) for g in grads])
    attn_grads = None
    if gat:
        attn_grads = [np.empty_like(a) for a in A]
        ap = (C.c_void_p * L)(*[N.ptr(a) for a in A])
        agp = (C.c_void_p * L)(*[N.ptr(g) for g in attn_grads])
        N.call("ht_sgd2", h_, L, dims_c, wp, ap, C.c_float(model.lr), gp, agp)
    else:
        N.call("ht_sgd", h_, L, dims_c, wp, C.c_float(model.lr), gp)
    loss = C.c_double(0.0)
    N.call("ht_loss_value", h_, C.byref(loss))
    value = float(loss.value)
    if fleet.rank is not None and fleet.m > 1:  # per-rank partials of the mean
        from . import dist
        value = dist.allreduce_sum(value)
    return EpochResult(loss=value, model=model, tracker=tracker, grads=grads,
                       attn_grads=attn_grads)


_MATRIX_MAGIC = b"HTF1"
_LABELS_MAGIC = b"HTL1"


def save_matrix(X: np.ndarray, path: str) -> None:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise GraphFormatError("matrix files hold 2-D arrays")
    with open(path, "wb") as fh:
        fh.write(_MATRIX_MAGIC)
        fh.write(struct.pack("<QQ", X.shape[0], X.shape[1]))
        fh.write(X.astype("<f8").tobytes())


def load_matrix(path: str, mmap: bool = False) -> np.ndarray:
    """HTF1 (engine.py:511-523).  ``mmap=True`` returns a read-only
    memory-mapped view (feature matrices of 10^8 rows stream into
    ``HostStore.set_features`` without a full in-memory copy)."""
    import os
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != _MATRIX_MAGIC:
            raise GraphFormatError(f"{path}: bad magic {magic!r}, expected {_MATRIX_MAGIC!r}")
        rows, cols = struct.unpack("<QQ", fh.read(16))
        if mmap:
            if os.path.getsize(path) < 20 + rows * cols * 8:
                raise GraphFormatError(f"{path}: truncated payload")
            return np.memmap(path, dtype="<f8", mode="r", offset=20, shape=(rows, cols))
        raw = fh.read(rows * cols * 8)
        if len(raw) != rows * cols * 8:
            raise GraphFormatError(f"{path}: truncated payload")
        return np.frombuffer(raw, dtype="<f8").reshape(rows, cols).copy()


def save_labels(y: np.ndarray, path: str) -> None:
    y = np.asarray(y, dtype=np.int64)
    with open(path, "wb") as fh:
        fh.write(_LABELS_MAGIC)
        fh.write(struct.pack("<Q", y.shape[0]))
        fh.write(y.astype("<i8").tobytes())


def load_labels(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != _LABELS_MAGIC:
            raise GraphFormatError(f"{path}: bad magic {magic!r}, expected {_LABELS_MAGIC!r}")
        (count,) = struct.unpack("<Q", fh.read(8))
        raw = fh.read(count * 8)
        if len(raw) != count * 8:
            raise GraphFormatError(f"{path}: truncated payload")
        return np.frombuffer(raw, dtype="<i8").copy()
