"""GPU diagnostic: wall time per native layer call of a GAT epoch on the
bench graph, with a device sync after each call (finds stalls)."""
import os, sys, time, ctypes as C
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2311_14898_b200 as H
from paper_2311_14898_b200 import _native as N

V = int(os.environ.get("DIAG_V", "2400000")); deg = float(os.environ.get("DIAG_DEG", "26.8"))
kind = os.environ.get("DIAG_KIND", "gat")
dims = [256, 128, 128, 64]
t0 = time.time()
ds = H.synth_dataset(H.SynthSpec(num_vertices=V, avg_degree=deg, seed=0), 16, 8)
a = H.partition_vertices(ds.graph, 1, seed=0)
p = H.split_chunks(ds.graph, a, 1)
plan = H.plan_for_partition(p)
c = p.chunks[0][0]
od = np.diff(c.csr_offsets); idg = np.diff(c.csc_offsets)
print(f"setup {time.time()-t0:.1f}s E={ds.graph.num_edges} max out-deg {od.max()} max in-deg {idg.max()} "
      f"edges in out-segs>4096: {od[od>4096].sum()}", flush=True)
X = np.random.default_rng(0).standard_normal((V, dims[0]), dtype=np.float32)
y = (ds.labels % dims[-1]).astype(np.int64)
host = H.HostStore(V, dims, dtype=np.float32, placement=os.environ.get("DIAG_PLACE", "device"))
host.set_features(X)
fleet = H.DeviceFleet(plan, dtype=np.float32, precision="tf32")
model = H.init_model(kind, dims, seed=0, dtype=np.float32)
orig = N.call
times = {}
def timed(name, *args, **kw):
    t = time.perf_counter()
    r = orig(name, *args, **kw)
    if name.startswith(("ht_gat", "ht_forward", "ht_backward", "ht_loss", "ht_sgd", "ht_epoch")):
        orig("ht_fleet_sync", fleet._handle)
        times.setdefault(name, []).append(time.perf_counter() - t)
    return r
N.call = timed
for e in range(3):
    times.clear()
    t = time.perf_counter()
    r = H.train_epoch(p, fleet, model, host, y, ds.mask)
    print(f"epoch {e}: {time.perf_counter()-t:.3f}s loss {r.loss:.5f}", flush=True)
    for k, v in times.items():
        print(f"   {k:24s} " + " ".join(f"{x*1e3:8.1f}" for x in v), flush=True)
