"""Probe: community-major processing order + column slices for the
one-device transposed aggregation (value epochs, cfg 2).

    HT_COL_SLICE_BWD=128 python profiles/tools/locality_order_probe.py K

K = LDG parts that define the order (0: ascending order).  Prints per-layer
device time of the backward (CUDA events between the native calls) and a
digest of the weights after two epochs (the order and the slices must not
change any value)."""
import ctypes as C
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2311_14898_b200 as H  # noqa: E402
from paper_2311_14898_b200 import _native as N  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = bench.CONFIGS["cfg2"]
ds, p, plan, _ = bench.build_inputs(cfg, 1)
dims = cfg["dims"]
g = ds.graph
host = H.HostStore(g.num_vertices, dims, dtype=np.float32, placement="device")
host.set_features(ds.features)
fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32)
model = H.init_model("gcn", dims, seed=cfg["seed"], lr=0.1, dtype=np.float32)
H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)  # attaches the chunk structure
if K > 0:
    t0 = time.time()
    parts = H.partition_vertices(g, K, seed=0).owner
    order = np.argsort(parts, kind="stable").astype(np.int32)
    N.call("ht_fleet_set_bwd_order", fleet._handle, N.ptr(order), order.size)
    print(f"LDG {K} parts: {time.time() - t0:.1f} s", flush=True)
model = H.init_model("gcn", dims, seed=cfg["seed"], lr=0.1, dtype=np.float32)
orig = N.call
names = []


def marked(name, *a, **k):
    r = orig(name, *a, **k)
    if name in ("ht_forward_layer", "ht_loss", "ht_backward_layer", "ht_sgd") and len(names) < 15:
        names.append(name + (f"[{a[1]}]" if name.endswith("layer") else ""))
        orig("ht_fleet_mark", fleet._handle, len(names))
    return r


import paper_2311_14898_b200.engine as E  # noqa: E402
for ep in range(6):
    names.clear()
    E.N.call = marked
    orig("ht_fleet_mark", fleet._handle, 0)
    H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    E.N.call = orig
    ms = C.c_double(0)
    parts_ms = []
    for i in range(1, len(names) + 1):
        orig("ht_fleet_elapsed_between", fleet._handle, i - 1, i, C.byref(ms))
        parts_ms.append(f"{names[i - 1]}={ms.value:.2f}")
    orig("ht_fleet_elapsed_between", fleet._handle, 0, len(names), C.byref(ms))
    if ep >= 2:
        print(f"K={K} slice={os.environ.get('HT_COL_SLICE_BWD', '0')} epoch {ep}: {ms.value:.2f} ms  "
              + " ".join(parts_ms), flush=True)
dig = hashlib.sha256(b"".join(np.ascontiguousarray(w).tobytes() for w in model.weights)).hexdigest()[:16]
print(f"weights digest {dig}", flush=True)
fleet.close()
