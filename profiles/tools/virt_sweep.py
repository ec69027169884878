"""The reference-faithful host path (8 virtual devices on one GPU, dedup
plan, cache off) at n = 1, 2, 4 batches per partition: epoch time, metered
host bytes and the implied PCIe rate."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
ds, p, plan, _ = bench.build_inputs(cfg, 1)
for n in (1, 2, 4):
    r = bench.virtual_fleet_epochs(ds, cfg["dims"], n=n, steps=2, warmup=1)
    r["host_gbs"] = r["metered_host_gb_per_step"] / (r["ms_per_step"] / 1e3)
    print(json.dumps({"n": n, **r}), flush=True)
