"""Full-size synthetic graphs with the streaming generator (SURVEY 8(f)
rank 3): build, report time / edges / peak RSS, round-trip through the
HTG1 cache (memory-mapped reload) and check the canonical invariants on a
sample of vertices.

    python profiles/tools/synth_scale.py cfg5 [--cache /tmp/g.htg1]
"""
import argparse
import json
import os
import resource
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2311_14898_b200 as H  # noqa: E402
from paper_2311_14898_b200 import synth as S  # noqa: E402

SHAPES = {  # BASELINE.json configs 3-5 (avg degree calibrated for the E after deduplication)
    "cfg3": (65_600_000, 27.6), "cfg4": (111_000_000, 14.6), "cfg5": (41_000_000, 28.3)}

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=sorted(SHAPES))
ap.add_argument("--cache", default=None)
a = ap.parse_args()
V, deg = SHAPES[a.config]
t0 = time.time()
g, cl = S.synth_graph_streaming(S.SynthSpec(num_vertices=V, avg_degree=deg, seed=0))
t1 = time.time()
out = {"config": a.config, "vertices": V, "edges": g.num_edges, "build_s": t1 - t0,
       "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6,
       "bytes_per_edge_peak": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1e3 / g.num_edges}
rng = np.random.default_rng(0)
for v in rng.choice(V, 1000, replace=False):
    s = g.csc_sources[g.csc_offsets[v]:g.csc_offsets[v + 1]]
    assert np.all(np.diff(s) > 0)
if a.cache:
    H.save_graph_cache(g, a.cache)
    t2 = time.time()
    g2 = H.load_graph_cache(a.cache)
    out.update({"cache_write_s": t2 - t1, "cache_load_s": time.time() - t2,
                "cache_gb": os.path.getsize(a.cache) / 1e9,
                "roundtrip_equal": bool(g2.content_hash() == g.content_hash())})
    os.remove(a.cache)
print(json.dumps(out), flush=True)
