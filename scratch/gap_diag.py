"""Per-epoch wall vs device time of the value (HBM store) GCN epoch at cfg2,
and a cProfile of the host side of one epoch (finds host gaps)."""
import cProfile, ctypes as C, os, pstats, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2311_14898_b200 as H
from paper_2311_14898_b200 import _native as N
ds = H.synth_dataset(H.SynthSpec(num_vertices=2_400_000, avg_degree=26.8, seed=0), 100, 47)
a = H.partition_vertices(ds.graph, 1, seed=0)
p = H.split_chunks(ds.graph, a, 1)
plan = H.plan_for_partition(p, device=0)
dims = [100, 256, 256, 47]
host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32, placement=os.environ.get("PLACE", "device"))
host.set_features(ds.features)
fleet = H.DeviceFleet(plan, dtype=np.float32)
model = H.init_model("gcn", dims, seed=0, dtype=np.float32)
for e in range(3):
    H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
for e in range(6):
    N.call("ht_fleet_mark", fleet._handle, 0)
    t = time.perf_counter()
    H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    wall = time.perf_counter() - t
    N.call("ht_fleet_mark", fleet._handle, 1)
    ms = C.c_double(0)
    N.call("ht_fleet_elapsed", fleet._handle, C.byref(ms))
    print(f"epoch {e}: wall {wall*1e3:.1f} ms  device {ms.value:.1f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
H.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
