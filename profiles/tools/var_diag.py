"""Per-phase device time of value epochs (HBM store): which phase carries the
run-to-run variance?  Marks are recorded on the compute stream between the
native calls of train_epoch."""
import collections, ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2311_14898_b200 as H
from paper_2311_14898_b200 import _native as N

cfg = bench.CONFIGS["cfg2"]
ds, p, plan, _ = bench.build_inputs(cfg, 1)
dims = cfg["dims"]
orig = N.call
state = {"h": None, "k": 0, "names": []}
PH = ("ht_forward_layer", "ht_loss", "ht_backward_layer", "ht_sgd")
def timed(name, *a, **k):
    r = orig(name, *a, **k)
    if name in PH and state["h"] is not None and state["k"] < 15:
        state["k"] += 1
        orig("ht_fleet_mark", state["h"], state["k"])
        state["names"].append(name + ("" if name in ("ht_loss", "ht_sgd") else f"[{a[1]}]"))
    return r
import paper_2311_14898_b200.engine as E
E.N.call = timed

def run(tag, clocks, epochs=10):
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32, placement="device")
    host.set_features(ds.features)
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32)
    model = H.init_model("gcn", dims, seed=cfg["seed"], lr=0.1, dtype=np.float32)
    for _ in range(3):
        H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    ctx = bench.Clocks(0) if clocks else None
    if ctx: ctx.__enter__()
    for e in range(epochs):
        state.update(h=fleet._handle, k=0, names=[])
        orig("ht_fleet_mark", fleet._handle, 0)
        H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
        k = state["k"]; state["h"] = None
        ms = C.c_double(0)
        parts = []
        for i in range(1, k + 1):
            orig("ht_fleet_elapsed_between", fleet._handle, i - 1, i, C.byref(ms))
            parts.append(f"{state['names'][i-1]}={ms.value:.1f}")
        orig("ht_fleet_elapsed_between", fleet._handle, 0, k, C.byref(ms))
        print(f"{tag} epoch {e}: total {ms.value:7.2f}  " + " ".join(parts), flush=True)
    if ctx:
        ctx.__exit__(None, None, None)
        print(tag, ctx.summary(), [r[0] for r in ctx.rows][:80])
    fleet.close()

run("noclk", False)
run("clk", True)
