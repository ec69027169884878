#!/usr/bin/env python
"""Benchmark of the B200-native HongTu GCN epoch (one step = one full-graph
training epoch: forward over every layer and batch, loss, backward, SGD).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
    python bench.py --impl reference ...     # CPU reference arm (chunktrain from
                                             # baseline/_ref, else the oracle port)

Workload (N=1): BASELINE config 2 - 3-layer GCN 100-256-256-47 on an
ogbn-products-shape synthetic graph (2.4M vertices, ~62M edges), m = N
partitions, n = 1 chunk per partition, mode "full", reorganized when the
Eq. 4 cost is lower (the reference CLI's rule).

Two measurements of the same metric (GTEPS = L*|E| / epoch seconds):
  value  HBM-resident vertex store (HongTu-IM: inputs already in HBM),
  e2e    the reference-facing path: HostStore in pinned host memory, every
         row crossing PCIe inside the timed region (the HongTu setting).
Both are timed with CUDA events recorded on the fleet's own streams
(max over devices), after W warm-up epochs, around exactly K epochs.
Inputs exceed L2 (62M edges, 2.4M x 1 KB rows), so no explicit flush.
"""

from __future__ import annotations

import argparse
import ctypes as C
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(V=100_000, avg_degree=20.0, dims=[64, 128, 16], n=4, seed=0,
                 name="2-layer GCN 64-128-16, synthetic power-law 100K V / ~1.87M E"),
    "cfg2": dict(V=2_400_000, avg_degree=26.8, dims=[100, 256, 256, 47], n=1, seed=0,
                 name="3-layer GCN 100-256-256-47, ogbn-products-shape synthetic 2.4M V / ~62M E"),
    # one GPU's share of BASELINE config 3 (friendster-shape 65.6M V / 1.8B E
    # over 8 GPUs): 8.2M V / ~227M E, 256-128-128-64, vertex data host-resident
    "cfg3s": dict(V=8_200_000, avg_degree=28.5, dims=[256, 128, 128, 64], n=1, seed=0,
                  name="3-layer GCN 256-128-128-64, per-GPU share of the friendster-shape config 3 "
                       "(8.2M V / ~227M E synthetic)"),
    # one GPU's share of BASELINE config 4 (ogbn-papers100M-shape 111M V /
    # 1.6B E over 8 GPUs): 13.9M V / ~200M E, 200-128-128-172, host-resident
    # data through the recompute-cache hybrid
    "cfg4s": dict(V=13_900_000, avg_degree=14.4, dims=[200, 128, 128, 172], n=1, seed=0,
                  name="3-layer GCN 200-128-128-172, per-GPU share of the ogbn-papers100M-shape "
                       "config 4 (13.9M V / ~200M E synthetic)"),
    # one GPU's share of BASELINE config 5 (it-2004-shape 41M V / 1.15B E
    # over 8 GPUs): 5.15M V / ~144M E, 3-layer GAT 256-128-128-64
    "cfg5s": dict(V=5_150_000, avg_degree=28.0, dims=[256, 128, 128, 64], n=1, seed=0,
                  model="gat",
                  name="3-layer GAT 256-128-128-64, per-GPU share of the it-2004-shape config 5 "
                       "(5.15M V / ~144M E synthetic)"),
}
METRIC = "full-graph GCN epoch GTEPS (L*|E|/epoch_s)"
GAT_METRIC = METRIC.replace("GCN", "GAT")


def model_of(cfg):
    return cfg.get("model", "gcn")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu=0):
        self.rows, self.gpu, self.proc = [], gpu, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for nm, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------
def build_inputs(cfg, m):
    import paper_2311_14898_b200 as H
    t0 = time.time()
    spec = H.SynthSpec(num_vertices=cfg["V"], avg_degree=cfg["avg_degree"], seed=cfg["seed"])
    ds = H.synth_dataset(spec, cfg["dims"][0], cfg["dims"][-1])
    t1 = time.time()
    a = H.partition_vertices(ds.graph, m, seed=cfg["seed"])
    p = H.split_chunks(ds.graph, a, cfg["n"])
    # dedup plan on the GPU: sort/unique of the chunks' raw neighbour ids
    # (ht_gplan_build, bit-identical with the host planner)
    from paper_2311_14898_b200 import _native as N
    ngpu = N.device_count()
    dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, ngpu) if ngpu else None
    tp = time.time()
    plan = H.plan_for_partition(p, device=dev)
    log(f"[bench] {'GPU' if ngpu else 'host'} dedup planner {time.time() - tp:.2f}s")
    chosen = "identity"
    if cfg["n"] > 1:
        r = H.reorganize(p)
        plan_r = H.plan_for_partition(r.partition, device=dev)
        if H.comm_cost(plan_r.volumes) <= H.comm_cost(plan.volumes):
            p, plan, chosen = r.partition, plan_r, "reorganized"
    t2 = time.time()
    log(f"[bench] synth {t1 - t0:.1f}s  partition+plan {t2 - t1:.1f}s  |E|={ds.graph.num_edges}")
    return ds, p, plan, chosen


def pcie_peaks():
    """Measured PCIe peaks of this box (GB/s): [h2d, d2h, bidir, zc_read, zc_write]."""
    from paper_2311_14898_b200 import _native as N
    out = np.zeros(5)
    try:
        N.call("ht_pcie_probe", 0, 1 << 30, N.ptr(out))
    except Exception as exc:  # noqa: BLE001 - report, do not fail the bench
        log(f"[bench] pcie probe failed: {exc}")
        return None
    return [float(x) for x in out]


def dedup_report():
    """Host<->GPU bytes per epoch of the deduplicated ('full') plan vs the
    non-deduplicated ('baseline') plan on BASELINE config 1 (m=4, n=4,
    reorganized) - the configuration where chunks share neighbours.  At the
    bench workload's m=1, n=1 the two plans coincide."""
    import paper_2311_14898_b200 as H
    c = CONFIGS["cfg1"]
    ds = H.synth_dataset(H.SynthSpec(num_vertices=c["V"], avg_degree=c["avg_degree"], seed=0),
                         c["dims"][0], c["dims"][-1])
    p = H.reorganize(H.split_chunks(ds.graph, H.partition_vertices(ds.graph, 4, seed=0), 4)).partition
    plan = H.plan_for_partition(p)
    f = sum(host_bytes_per_epoch(plan, c["dims"], "full"))
    b = sum(host_bytes_per_epoch(plan, c["dims"], "baseline"))
    v = plan.volumes
    return {"config": "cfg1 m=4 n=4 reorganized", "host_gb_full": f / 1e9,
            "host_gb_baseline": b / 1e9, "reduction": 1.0 - f / b,
            "volumes": {"v_ori": v.v_ori, "v_p2p": v.v_p2p, "v_ru": v.v_ru}}


def virtual_fleet_epochs(ds, dims, m=8, steps=2, warmup=1, precision="tf32", seed=0, device=0,
                         profile=False, n=1):
    """The reference-faithful HongTu path at the bench's scale: m virtual
    devices (the 8-GPU partition layout) on this one GPU, the deduplicated
    plan, host-resident vertex data and no HBM owner cache - every batch's
    unique neighbour rows cross PCIe once, peers' rows are fetched from the
    peer's slot buffer, owner pushes and flushes write the gradients back.
    Reports the epoch time and the metered host / peer bytes against the
    plan's prediction."""
    import paper_2311_14898_b200 as H
    g = ds.graph
    p = H.split_chunks(g, H.partition_vertices(g, m, seed=seed), n)
    if n > 1:
        r0 = H.reorganize(p)
        if H.comm_cost(H.plan_for_partition(r0.partition, device=device).volumes) <= \
                H.comm_cost(H.plan_for_partition(p, device=device).volumes):
            p = r0.partition
    plan = H.plan_for_partition(p, device=device)
    r = run_epochs(p, plan, ds, dims, "host", steps, warmup, precision, False, seed, cache="off",
                   profile=profile)
    tot = r["report"]["totals"]
    host = tot["h2d_bytes"] + tot["d2h_bytes"] + tot["dest_bytes"] + tot["chkpt_bytes"]
    L = len(dims) - 1
    ms = r["ms_total"] / steps
    pred = sum(host_bytes_per_epoch(plan, dims, "full")) - 4 * g.num_vertices * dims[L] - 9 * g.num_vertices
    return {"what": f"{m} virtual devices on one GPU, {n} batch(es) each, mode full, cache off, "
                    "host-resident store",
            "ms_per_step": ms, "value": L * g.num_edges / (ms / 1e3) / 1e9, "unit": "GTEPS",
            "metered_host_gb_per_step": host / steps / 1e9,
            "planned_host_gb_per_step": pred / 1e9,
            "metered_peer_gb_per_step": tot["d2d_bytes"] / steps / 1e9,
            "loss": r["losses"][-1]}


def profile_epoch(args, cfg, ds, p, plan):
    """bench.py --profile-epoch MODE: W warm-up epochs, then K epochs inside a
    profiler range, for ncu --replay-mode app-range --profile-from-start off
    (pcie__read_bytes / pcie__write_bytes / dram bytes of exactly those
    epochs, copy engines included).  Prints the plan's bytes for the same
    epochs; never a bench line (a number taken under a profiler is not one)."""
    dims = cfg["dims"]
    mode = args.profile_epoch
    if mode == "virt":
        r = virtual_fleet_epochs(ds, dims, steps=args.steps, warmup=args.warmup,
                                 precision=args.precision, seed=cfg["seed"], profile=True)
        out = {"mode": mode, "planned_host_gb_per_step": r["planned_host_gb_per_step"],
               "metered_host_gb_per_step": r["metered_host_gb_per_step"],
               "metered_peer_gb_per_step": r["metered_peer_gb_per_step"]}
    elif args.kind == "gat" or model_of(cfg) == "gat":  # GAT epochs (profiling)
        gd = cfg["dims"] if model_of(cfg) == "gat" else GAT_DIMS
        X = ds.features if model_of(cfg) == "gat" else np.random.default_rng(cfg["seed"]).standard_normal(
            (ds.graph.num_vertices, gd[0]), dtype=np.float32)
        y = (np.asarray(ds.labels) % gd[-1]).astype(np.int64)
        r = run_epochs(p, plan, ds, gd, "device" if mode == "value" else "host", args.steps,
                       args.warmup, args.precision, False, cfg["seed"], kind="gat", features=X,
                       labels=y, profile=True)
        out = {"mode": mode, "kind": "gat"}
    else:
        placement = "device" if mode == "value" else "host"
        r = run_epochs(p, plan, ds, dims, placement, args.steps, args.warmup, args.precision,
                       False, cfg["seed"], profile=True)
        h2d, d2h = host_bytes_per_epoch(plan, dims, cached=r["cache"], ckpt_hbm=r["ckpt_hbm"])
        out = {"mode": mode, "hbm_owner_cache": bool(r["cache"]), "ckpt_hbm": bool(r["ckpt_hbm"])}
        if placement == "host":
            out.update({"planned_h2d_gb_per_step": h2d / 1e9, "planned_d2h_gb_per_step": d2h / 1e9})
    out.update({"config_id": args.config, "steps": args.steps, "warmup": args.warmup,
                "ms_total_under_profiler": r.get("ms_total")})
    print(json.dumps(out), flush=True)


def dedup_at_scale(ds, dims, m=8, n=1, seed=0, device=None):
    """The same plan comparison on the bench graph itself, partitioned for m
    GPUs (the north star's 8-GPU layout): host bytes of one epoch through the
    deduplicated plan vs the non-deduplicated one, all classes and the
    neighbour class alone (SURVEY 8(d) formulas, fp32)."""
    import paper_2311_14898_b200 as H
    g = ds.graph
    p = H.split_chunks(g, H.partition_vertices(g, m, seed=seed), n)
    plan = H.plan_for_partition(p, device=device)
    f = sum(host_bytes_per_epoch(plan, dims, "full"))
    b = sum(host_bytes_per_epoch(plan, dims, "baseline"))
    v = plan.volumes
    nb = 4 * sum(dims[:-1])  # bytes per neighbour row over all layers (load + flush)
    return {"config": f"bench graph m={m} n={n}", "host_gb_full": f / 1e9,
            "host_gb_baseline": b / 1e9, "reduction": 1.0 - f / b,
            "neighbour_gb_full": 2 * v.v_ru * nb / 1e9,
            "neighbour_gb_baseline": 2 * v.v_ori * nb / 1e9,
            "neighbour_reduction": 1.0 - v.v_ru / v.v_ori,
            "volumes": {"v_ori": v.v_ori, "v_p2p": v.v_p2p, "v_ru": v.v_ru}}


def host_bytes_per_epoch(plan, dims, mode="full", cached=False, kind="gcn", ckpt_hbm=False):
    """Host<->GPU bytes of one epoch from the plan (SURVEY 8(d) formulas,
    fp32): neighbour loads/flushes + destination + checkpoint rows, plus the
    loss gradient rows this path writes to host.grad_h[L].  With the HBM
    owner cache the host is read once (the owned h^0 rows) and written once
    per produced row: h^{l+1} and agg^l per forward layer, grad_h^l per
    backward layer, grad_h^L after the loss; with the checkpoint tier in HBM
    (``checkpoints="auto"``) the agg^l rows are not written."""
    import paper_2311_14898_b200 as H
    L = len(dims) - 1
    V = int(plan.owner.shape[0])
    if cached:
        h2d = 4 * V * dims[0] + V * 9
        d2h = 4 * V * (sum(dims[1:]) + sum(dims[:L]) + dims[L])
        if kind == "gcn" and not ckpt_hbm:
            d2h += 4 * V * sum(dims[:L])
        return h2d, d2h
    pred = H.predicted_transfers(plan, mode)
    h2d = d2h = 0
    for l in range(L):
        h2d += 4 * (pred["fwd_h2d_rows"] * dims[l] + V * (dims[l] + dims[l + 1]))
        d2h += 4 * (V * (dims[l + 1] + dims[l]) + pred["bwd_d2h_rows"] * dims[l])
    d2h += 4 * V * dims[L]
    h2d += V * 9  # labels (int64) + mask (uint8) upload for the loss
    return h2d, d2h


def host_threads():
    """Threads the numpy/BLAS CPU path may use here (torchrun sets
    OMP_NUM_THREADS=1 per rank unless told otherwise)."""
    env = os.environ.get("OMP_NUM_THREADS")
    return int(env) if env and env.isdigit() and int(env) > 0 else os.cpu_count()


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_impl():
    """The CPU implementation of the path that the reference arm and the
    cpu_baseline time: the unmodified reference package ``chunktrain`` from
    ``baseline/_ref`` (kind "reference"), else the oracle port (kind "port").
    Neither loads this repository's native library."""
    if os.path.isdir(REF_DIR) and REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        from chunktrain import engine as E
        from chunktrain import partition as P

        def chunk(g, verts):
            return P.chunk_from_vertices(g, verts, 0, 0)

        def fwd(ch, h_nbr, W):
            return E.gcn_layer_forward(ch, h_nbr, W)

        def bwd(ch, agg, gout, W):
            return E.gcn_layer_backward_hybrid(ch, agg, gout, W)

        def src_of(ch):
            return ch.sources

        def nedges(ch):
            return int(ch.num_edges)

        def gfwd(ch, h_nbr, h_dst, W, a):
            return E.gat_layer_forward(ch, h_nbr, h_dst, W, a)

        def gbwd(ch, h_nbr, h_dst, gout, W, a):
            return E.gat_layer_backward_recompute(ch, h_nbr, h_dst, gout, W, a)

        return "reference", dict(chunk=chunk, fwd=fwd, bwd=bwd, gfwd=gfwd, gbwd=gbwd,
                                 loss=E.downstream_loss, sources=src_of, edges=nedges,
                                 what="chunktrain (unmodified reference, baseline/_ref)")
    except ImportError:
        from oracle import hongtu_oracle as O

        def chunk(g, verts):
            gd = {k: getattr(g, k) for k in ("csc_offsets", "csc_sources", "edge_weights")}
            gd["num_vertices"] = g.num_vertices
            return O.chunk_of(gd, verts)

        return "port", dict(chunk=chunk, fwd=O.gcn_chunk_forward, bwd=O.gcn_chunk_backward,
                            gfwd=O.gat_chunk_forward, gbwd=O.gat_chunk_backward,
                            loss=O.softmax_xent, sources=lambda ch: ch["sources"],
                            edges=lambda ch: int(ch["csc_local_src"].size),
                            what="oracle port (oracle/hongtu_oracle.py, numpy)")


def reference_graph(cfg):
    """The workload's graph and node data built without this repository's
    native library: chunktrain.synth when the reference is installed, else
    the same draws (synth_edges, pure numpy) + numpy parallel-edge removal +
    the oracle's graph builder."""
    spec_kw = dict(num_vertices=cfg["V"], avg_degree=cfg["avg_degree"], seed=cfg["seed"])
    if os.path.isdir(REF_DIR) and REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        from chunktrain import synth as S
        ds = S.synth_dataset(S.SynthSpec(**spec_kw), cfg["dims"][0], cfg["dims"][-1])
        return ds.graph, ds.labels, ds.mask
    except ImportError:
        from types import SimpleNamespace

        from oracle import hongtu_oracle as O
        from paper_2311_14898_b200 import synth as PS  # numpy draws only
        spec = PS.SynthSpec(**spec_kw)
        src, dst, cl = PS.synth_edges(spec)
        _, keep = np.unique(dst * spec.num_vertices + src, return_index=True)
        gd = O.build_graph(src[keep], dst[keep], spec.num_vertices)
        _, y, mask = PS.synth_node_data(spec.num_vertices, cfg["dims"][0], cfg["dims"][-1],
                                        spec.seed, cluster_of=cl)
        return SimpleNamespace(**gd), y, mask


class ReferenceSampler:
    """One bounded sample of the epoch on the CPU reference path.

    A step runs, for a window of consecutive destination vertices holding
    ~``budget_edges`` in-edges (a different window each step, spread over
    the vertex range), exactly what the reference's train_epoch does per
    batch and layer (src/engine.py:409-477): gather h^l[N] from the full
    (V, d_l) host array, gcn_layer_forward, the loss on the last layer,
    gcn_layer_backward_hybrid from the agg checkpoint, and the flush of the
    neighbour gradients into the full (V, d_l) host gradient array - for
    every layer at its own width.  Nothing is extrapolated: the rate is the
    edges actually traversed (each edge once per layer, as GTEPS counts
    them) over the step's wall time."""

    def __init__(self, graph, labels, mask, dims, budget_edges=250_000, windows=16, seed=0,
                 model="gcn"):
        self.kind, self.api = reference_impl()
        self.dims = dims
        self.model = model
        V = int(graph.num_vertices)
        off = np.asarray(graph.csc_offsets)
        self.chunks = []
        for w in range(windows):
            v0 = (V * w) // windows
            v1 = int(np.searchsorted(off, off[v0] + budget_edges))
            v1 = min(max(v1, v0 + 1), V)
            verts = np.arange(v0, v1, dtype=np.int64)
            self.chunks.append((verts, self.api["chunk"](graph, verts)))
        rng = np.random.default_rng(seed)
        L = len(dims) - 1
        # host arrays of the layer inputs / input gradients (the HostStore)
        self.h = [rng.standard_normal((V, dims[l]), dtype=np.float32) for l in range(L)]
        self.g = [np.zeros((V, dims[l]), dtype=np.float32) for l in range(L)]
        self.W = [(rng.standard_normal((dims[l], dims[l + 1])) *
                   np.sqrt(2.0 / (dims[l] + dims[l + 1]))).astype(np.float32) for l in range(L)]
        self.gup = [rng.standard_normal((budget_edges, dims[l + 1]), dtype=np.float32) * 1e-3
                    for l in range(L)]
        self.A = [(rng.standard_normal(2 * dims[l + 1]) * 0.1).astype(np.float32) for l in range(L)]
        self.labels, self.mask = np.asarray(labels), np.asarray(mask)
        self.step_i = 0

    def step(self):
        """One timed sample; returns (seconds, edges traversed)."""
        verts, ch = self.chunks[self.step_i % len(self.chunks)]
        self.step_i += 1
        api, L = self.api, len(self.dims) - 1
        src = api["sources"](ch)
        nv = verts.size
        t0 = time.perf_counter()
        if self.model == "gat":  # engine.py:418-423, 455-470: no checkpoints, recompute
            for l in range(L):
                h_out, _ = api["gfwd"](ch, self.h[l][src], self.h[l][verts], self.W[l], self.A[l])
            _, grad = api["loss"](h_out, self.labels[verts], self.mask[verts])
            for l in reversed(range(L)):
                gout = grad if l == L - 1 else self.gup[l][:nv]
                out = api["gbwd"](ch, self.h[l][src], self.h[l][verts], gout, self.W[l], self.A[l])
                self.g[l][verts] += out[1]
                self.g[l][src] += out[0]
            dt = time.perf_counter() - t0
            return dt, L * api["edges"](ch)
        aggs = []
        for l in range(L):
            h_out, agg, _ = api["fwd"](ch, self.h[l][src], self.W[l])
            aggs.append(agg)
        _, grad = api["loss"](h_out, self.labels[verts], self.mask[verts])
        for l in reversed(range(L)):
            gout = grad if l == L - 1 else self.gup[l][:nv]
            gnbr, _ = api["bwd"](ch, aggs[l], gout, self.W[l])
            self.g[l][src] += gnbr
        dt = time.perf_counter() - t0
        return dt, L * api["edges"](ch)

    def describe(self):
        e = [self.api["edges"](c) for _, c in self.chunks]
        fw, bw = (("gat_layer_forward", "gat_layer_backward_recompute") if self.model == "gat"
                  else ("gcn_layer_forward", "gcn_layer_backward_hybrid"))
        return (f"{self.api['what']}: per step, one window of consecutive destinations "
                f"(~{int(np.mean(e))} in-edges; {len(e)} windows spread over the vertex range, "
                f"one per step in turn) through every layer: gather h^l[N] from the full "
                f"(V, d_l) host array, {fw}, downstream_loss, "
                f"{bw}, flush into the (V, d_l) gradient array; "
                f"GTEPS = edges traversed (once per layer) / step wall time, not extrapolated")


def reference_cpu_baseline(graph, labels, mask, dims, steps=3, warmup=1, model="gcn"):
    """cpu_baseline of the ours-arm line: a few ReferenceSampler steps."""
    rs = ReferenceSampler(graph, labels, mask, dims, model=model)
    for _ in range(warmup):
        rs.step()
    t = e = 0.0
    for _ in range(steps):
        dt, ne = rs.step()
        t, e = t + dt, e + ne
    return {"value": e / t / 1e9, "unit": "GTEPS", "cores": host_threads(), "kind": rs.kind,
            "sample": rs.describe() + f"; {steps} steps after {warmup} warm-up",
            "seconds": t, "edges": int(e),
            "note": "np.add.at / np.add.reduceat are single-threaded; BLAS may use all cores"}


# ---------------------------------------------------------------------------
# timed epochs
# ---------------------------------------------------------------------------
def run_epochs(p, plan, ds, dims, placement, steps, warmup, precision, timing, seed, rank=None,
               kind="gcn", features=None, labels=None, lean=False, checkpoints="auto",
               cache="auto", profile=False, hbm_budget_gb=None):
    import paper_2311_14898_b200 as H
    from paper_2311_14898_b200 import _native as N
    dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, N.device_count()) if rank is not None else 0
    # one process per GPU: a compact host store with only the rank's owned
    # rows (host memory per process ~ V/N; every host copy contiguous)
    rows = np.flatnonzero(plan.owner == rank) if rank is not None and placement == "host" else None
    fr, tot = N.mem_info(dev)
    log(f"[bench] {placement} store, {kind}: {fr / 2**30:.1f} of {tot / 2**30:.1f} GiB HBM free")
    host = H.HostStore(ds.graph.num_vertices, dims, dtype=np.float32, placement=placement,
                       device=dev, rows=rows)
    host.set_features(ds.features if features is None else features)
    labels = ds.labels if labels is None else labels
    fleet = H.DeviceFleet(plan, mode="full", dtype=np.float32, precision=precision, rank=rank,
                          devices=[dev] if rank is not None else None, lean=lean,
                          checkpoints=checkpoints, cache=cache, hbm_budget_gb=hbm_budget_gb)
    try:
        return _timed_epochs(H, N, p, fleet, host, ds, dims, steps, warmup, timing, seed, kind,
                             labels, profile)
    finally:
        host.agg.pending.clear()  # nobody reads these checkpoints: nothing to materialize
        fleet.close()  # device memory back before the next measurement (also on failure)
        del host, fleet  # an HBM store's arrays too (cfg4s needs the whole HBM per run)
        gc.collect()


def _timed_epochs(H, N, p, fleet, host, ds, dims, steps, warmup, timing, seed, kind, labels,
                  profile=False):
    model = H.init_model(kind, dims, seed=seed, lr=0.1, dtype=np.float32)
    losses = []
    for _ in range(warmup):
        losses.append(H.train_epoch(p, fleet, model, host, labels, ds.mask).loss)
    fleet.set_timing(timing)
    for d in fleet.devices:  # meters of the timed region only
        for k, v in d.counter_dict().items():
            setattr(d, k, 0)
    l0 = N.lib().ht_launches()
    if profile:  # counters of exactly the timed epochs (ncu app-range replay)
        N.call("ht_profile_range", 1)
    N.call("ht_fleet_mark", fleet._handle, 0)
    t0 = time.perf_counter()
    for _ in range(steps):
        losses.append(H.train_epoch(p, fleet, model, host, labels, ds.mask).loss)
    N.call("ht_fleet_mark", fleet._handle, 1)
    if profile:
        N.call("ht_profile_range", 0)
    ms = C.c_double(0)
    N.call("ht_fleet_elapsed", fleet._handle, C.byref(ms))
    wall = time.perf_counter() - t0
    launches = N.lib().ht_launches() - l0
    stats = {w: fleet.kernel_stats(w) for w in range(4)} if timing else {}
    rep = fleet.transfer_report()
    cache = fleet.cache_active
    ckpt_hbm = bool(host.agg.pending)
    return {"ms_total": ms.value, "wall_s": wall, "losses": losses, "launches": launches,
            "stats": stats, "report": rep, "cache": cache, "ckpt_hbm": ckpt_hbm,
            "recompute_layers": list(fleet.recompute_layers)}


def hybrid_budget_gb(V, dims):
    """An HBM budget (GB) for the recompute-cache hybrid on one device, one
    batch: the h + grad mirrors, the project-first buffers, the narrowest agg
    mirror and one scratch of the widest - the other agg mirrors do not fit
    and share the scratch (their agg^l re-aggregated in the backward)."""
    L = len(dims) - 1
    base = 4 * V * (sum(dims[:L]) + sum(dims))
    pw = max([(dims[l + 1] + 3) // 4 * 4 for l in range(L) if dims[l + 1] < dims[l]] or [0])
    base += 2 * 4 * V * pw
    return (base + 4 * V * (min(dims[:L]) + max(dims[:L])) + (1 << 20)) / 2 ** 30


GAT_DIMS = [256, 128, 128, 64]  # it-2004 / config 5 widths


def gat_measure(p, plan, ds, steps, warmup, precision, seed, rank, slowest, dims=None,
                native_data=False):
    """A 3-layer GAT epoch (value: HBM store; e2e: pinned host store).  By
    default BASELINE config 5's model (256-128-128-64) on the bench graph:
    config 5's 41M-vertex graph needs ~190 GB of pinned host rows, beyond one
    box's host memory, so the GAT path is measured on the same graph with
    synthetic 256-wide features and 64 classes; native_data: the dataset's
    own features / labels (the cfg5s per-GPU share)."""
    dims = GAT_DIMS if dims is None else dims
    V = ds.graph.num_vertices
    if native_data:
        X, y = ds.features, ds.labels
    else:
        rng = np.random.default_rng(seed)
        X = rng.standard_normal((V, dims[0]), dtype=np.float32)
        y = (np.asarray(ds.labels) % dims[-1]).astype(np.int64)
    L = len(dims) - 1
    E = ds.graph.num_edges
    out = {"workload": f"3-layer GAT {'-'.join(map(str, dims))} on the bench graph "
                       f"({V} V / {E} E), m=n=1, mode full",
           "metric": GAT_METRIC, "unit": "GTEPS"}
    val = run_epochs(p, plan, ds, dims, "device", steps, warmup, precision, True, seed,
                     rank=rank, kind="gat", features=X, labels=y)
    ms_v = slowest(val["ms_total"]) / steps
    e2e = run_epochs(p, plan, ds, dims, "host", steps, warmup, precision, True, seed,
                     rank=rank, kind="gat", features=X, labels=y)
    ms_e = slowest(e2e["ms_total"]) / steps
    lf, msf, bf = val["stats"][0]
    lb, msb, bb = val["stats"][1]
    lg, msg, flops = val["stats"][2]
    hb = host_bytes_per_epoch(plan, dims, cached=e2e["cache"], kind="gat") if e2e["cache"] else None
    out.update({
        "value": L * E / (ms_v / 1e3) / 1e9, "ms_per_step": ms_v,
        "e2e": {"value": L * E / (ms_e / 1e3) / 1e9, "unit": "GTEPS", "ms_per_step": ms_e,
                "wall_ms_per_step": e2e["wall_s"] / steps * 1e3,
                "hbm_owner_cache": bool(e2e["cache"]),
                "h2d_bytes_per_step": hb[0] if hb else None,
                "d2h_bytes_per_step": hb[1] if hb else None},
        "edge_kernels": {"fwd_ms_per_step": msf / steps, "bwd_ms_per_step": msb / steps,
                         "fwd_gbs": bf / (msf / 1e3) / 1e9 if msf else None,
                         "bwd_gbs": bb / (msb / 1e3) / 1e9 if msb else None,
                         "bytes_per_step": (bf + bb) / steps,
                         "launches_per_step": (lf + lb) / steps,
                         "share_of_step": (msf + msb) / val["ms_total"] if val["ms_total"] else None},
        "gemm": {"ms_per_step": msg / steps, "tflops": flops / (msg / 1e3) / 1e12 if msg else None},
        "gpu_launches": int(val["launches"]),
        "gpu_launches_e2e": int(e2e["launches"]),
        "losses": {"value": val["losses"][-1], "e2e": e2e["losses"][-1]},
    })
    return out


def gat_config_line(args, cfg, config, p, plan, ds, rk, slowest, hbm_peak, hbm_src):
    """The contract line of a GAT workload (cfg5s): value / e2e / roofline of
    the edge kernels / cpu_baseline, like the GCN line."""
    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        r = gat_measure(p, plan, ds, args.steps, args.warmup, args.precision, cfg["seed"], rk,
                        slowest, dims=cfg["dims"], native_data=True)
    ek = r["edge_kernels"]
    ms_ek = ek["fwd_ms_per_step"] + ek["bwd_ms_per_step"]
    achieved = ek["bytes_per_step"] / (ms_ek / 1e3) / 1e9 if ms_ek else 0.0
    cpu = None
    if not args.no_cpu_baseline:
        cpu = reference_cpu_baseline(ds.graph, ds.labels, ds.mask, cfg["dims"], model="gat")
    pcie = pcie_peaks()
    e2e_b = (r["e2e"]["h2d_bytes_per_step"] or 0) + (r["e2e"]["d2h_bytes_per_step"] or 0)
    e2e_s = r["e2e"]["ms_per_step"] / 1e3
    pcie_line = {"bound": "pcie", "what": "host<->GPU bytes of the e2e epoch (plan) / epoch time",
                 "source": "plan", "achieved": e2e_b / e2e_s / 1e9 if e2e_b else None, "unit": "GB/s",
                 "peak": pcie[2] if pcie else None,
                 "peak_source": "measured (copy engines, both directions at once)",
                 "frac": e2e_b / e2e_s / 1e9 / pcie[2] if pcie and e2e_b else None,
                 "d2h_bound_frac": (r["e2e"]["d2h_bytes_per_step"] or 0) / e2e_s / 1e9 / pcie[1]
                 if pcie else None}
    n_gpus = int(os.environ.get("WORLD_SIZE", "1"))
    out = {"metric": GAT_METRIC, "value": r["value"], "unit": "GTEPS",
           "n_gpus": n_gpus if n_gpus > 1 else args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": ("f32 edge softmax / aggregation, tf32 tcgen05 GEMMs (3xTF32 projections)"
                     if args.precision == "tf32" else "f32"),
           "data": "synthetic (seeded clustered power-law graph, random-init weights)",
           "config": config, "e2e": r["e2e"],
           "roofline": {"bound": "hbm", "kernel": "k_gat_dst / k_gat_src (edge softmax "
                        "aggregation, forward + backward)", "achieved": achieved,
                        "peak": hbm_peak, "peak_source": hbm_src, "unit": "GB/s",
                        "frac": achieved / hbm_peak if hbm_peak else None, "traffic": None,
                        "algorithmic_bytes_per_launch": ek["bytes_per_step"] / ek["launches_per_step"]
                        if ek["launches_per_step"] else None,
                        "share_of_step": ek["share_of_step"]},
           "gemm": r["gemm"], "gpu_launches": r["gpu_launches"],
           "gpu_launches_e2e": r["gpu_launches_e2e"], "cpu_baseline": cpu,
           "roofline_pcie": pcie_line,
           "clocks": clk.summary(), "losses": r["losses"]}
    return out


def workload_config(config_id, cfg, E, m, ordering):
    return {"workload": cfg["name"], "config_id": config_id, "vertices": cfg["V"],
            "edges": E, "dims": cfg["dims"], "m": m, "n": cfg["n"], "mode": "full",
            "ordering": ordering,
            "l2": ("inputs larger than L2 (no flush)" if 4 * cfg["V"] * sum(cfg["dims"]) > 126e6
                   else "inputs fit in the 126 MB L2 (not flushed between steps)")}


def reference_full_epoch_cfg1(seed=0):
    """BASELINE.md §3's plan for the CPU reference: one whole
    ``chunktrain.engine.train_epoch`` of config 1 (2-layer GCN 64-128-16,
    100K V / 1.87M E, m=4, n=4, reorganized, float32) through the unmodified
    package - setup untimed, the epoch timed end to end (~20 s on the
    container's cores).  None when the reference is not installed."""
    if not os.path.isdir(REF_DIR):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from chunktrain import devices as D
    from chunktrain import engine as E
    from chunktrain import partition as P
    from chunktrain import planner as PL
    from chunktrain import synth as S
    c = CONFIGS["cfg1"]
    ds = S.synth_dataset(S.SynthSpec(num_vertices=c["V"], avg_degree=c["avg_degree"], seed=seed),
                         c["dims"][0], c["dims"][-1])
    p = P.split_chunks(ds.graph, P.partition_vertices(ds.graph, 4, seed=seed), c["n"])
    p = PL.reorganize(p).partition
    plan = PL.plan_for_partition(p)
    model = E.init_model("gcn", c["dims"], seed=seed, lr=0.1, dtype=np.float32)
    host = D.HostStore(ds.graph.num_vertices, c["dims"], dtype=np.float32)
    host.set_features(ds.features)
    fleet = D.DeviceFleet(plan, mode="full", dtype=np.float32)
    t0 = time.perf_counter()
    res = E.train_epoch(p, fleet, model, host, ds.labels, ds.mask)
    dt = time.perf_counter() - t0
    L = len(c["dims"]) - 1
    return {"what": "chunktrain.engine.train_epoch, config 1 (m=4, n=4, reorganized, float32), "
                    "one whole epoch", "seconds": dt,
            "gteps": L * ds.graph.num_edges / dt / 1e9, "edges": int(ds.graph.num_edges),
            "loss": float(res.loss), "cores": host_threads()}


def reference_arm(args, cfg, n_gpus):
    """bench.py --impl reference: the reference's own CPU implementation of
    the path (ReferenceSampler), W warm-up + K timed steps, each a bounded
    sample of the workload; the JSON line reports exactly those K steps."""
    dims = cfg["dims"]
    t0 = time.time()
    graph, labels, mask = reference_graph(cfg)
    log(f"[bench-ref] graph {time.time() - t0:.1f}s |E|={graph.num_edges}")
    rs = ReferenceSampler(graph, labels, mask, dims, seed=cfg["seed"], model=model_of(cfg))
    # numpy has nothing to warm beyond the first touch of the host arrays:
    # one warm-up sample (reported as executed) keeps the run to minutes
    warm = min(args.warmup, 1)
    for _ in range(warm):
        rs.step()
    t = e = 0.0
    for _ in range(args.steps):
        dt, ne = rs.step()
        t, e = t + dt, e + ne
    v = e / t / 1e9
    metric = GAT_METRIC if model_of(cfg) == "gat" else METRIC
    out = {"impl": "reference", "metric": metric, "value": v, "unit": "GTEPS",
           "n_gpus": n_gpus, "steps": args.steps, "warmup": warm,
           "warmup_requested": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": workload_config(args.config, cfg, int(graph.num_edges), n_gpus, "identity"),
           "edges_per_step": e / args.steps,
           "cpu_baseline": {"value": v, "unit": "GTEPS", "cores": host_threads(), "kind": rs.kind,
                            "sample": rs.describe(),
                            "note": "np.add.at / np.add.reduceat are single-threaded"},
           "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    try:  # the reference's own full epoch at config 1, beside the samples
        out["full_epoch_cfg1"] = reference_full_epoch_cfg1(cfg["seed"])
    except Exception as exc:  # noqa: BLE001 - report, do not fail the arm
        out["full_epoch_cfg1"] = {"error": str(exc)[:200]}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--only-value", action="store_true", help="profiling: HBM-resident run only")
    ap.add_argument("--no-gat", action="store_true", help="skip the GAT (config 5 model) line")
    ap.add_argument("--kind", default="gcn", choices=["gcn", "gat"],
                    help="profiling: model of the --only-value run")
    ap.add_argument("--profile-epoch", default=None, choices=["value", "e2e", "virt"],
                    help="profiling: K epochs inside a cudaProfilerStart/Stop range (ncu app-range)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    N_gpus = args.gpus if world == 1 else world
    cfg = CONFIGS[args.config]
    dims = cfg["dims"]
    L = len(dims) - 1
    if args.impl == "reference":
        # the CPU reference arm runs on rank 0 only; no process group, no GPU,
        # no native library of this repository
        if rank == 0:
            reference_arm(args, cfg, N_gpus)
        return
    if world > 1:
        # host plumbing only (IPC handles, loss partials, max-over-ranks
        # timing); the data path is CUDA IPC + device-side barriers
        import torch.distributed as dist
        dist.init_process_group("gloo")
    m = N_gpus
    ds, p, plan, chosen = build_inputs(cfg, m)
    E = ds.graph.num_edges
    config = workload_config(args.config, cfg, E, m, chosen)

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured" if "hbm_gbs" in peaks else "fallback"

    rk = rank if world > 1 else None  # torchrun: one process per GPU (rank mode)

    def slowest(ms):  # device time, max over ranks
        if world > 1:
            from paper_2311_14898_b200 import dist as hd
            return hd.allreduce_max(ms)
        return ms

    if args.profile_epoch:  # profiling aid: counters of whole epochs
        profile_epoch(args, cfg, ds, p, plan)
        return
    if model_of(cfg) == "gat":  # a GAT workload (cfg5s): its own contract line
        out = gat_config_line(args, cfg, config, p, plan, ds, rk, slowest, hbm_peak, hbm_src)
        if rank == 0:
            print(json.dumps(out), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return
    if args.only_value and args.kind == "gat":  # profiling aid
        r = gat_measure(p, plan, ds, args.steps, args.warmup, args.precision, cfg["seed"], rk,
                        slowest)
        log(f"[bench] GAT: {json.dumps(r)}")
        return
    # ---- value: HBM-resident vertex store ----
    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk_v:
        val = run_epochs(p, plan, ds, dims, "device", args.steps, args.warmup, args.precision,
                         True, cfg["seed"], rank=rk)
    ms_v = slowest(val["ms_total"]) / args.steps
    if args.only_value:  # profiling aid: no e2e run, no JSON contract line
        log(f"[bench] value run: {ms_v:.2f} ms/epoch  stats {val['stats']}")
        return
    # ---- e2e: pinned host-resident vertex store through train_epoch ----
    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk_e:
        e2e = run_epochs(p, plan, ds, dims, "host", args.steps, args.warmup, args.precision,
                         True, cfg["seed"], rank=rk)
    ms_e = slowest(e2e["ms_total"]) / args.steps
    # opt-in lean epochs: no grad_h^0, no host h^L / grad_h^L
    e2e_lean = run_epochs(p, plan, ds, dims, "host", args.steps, args.warmup, args.precision,
                          False, cfg["seed"], rank=rk, lean=True)
    ms_el = slowest(e2e_lean["ms_total"]) / args.steps
    # the reference's host-side checkpoint cache (agg rows written through)
    e2e_hc = run_epochs(p, plan, ds, dims, "host", args.steps, args.warmup, args.precision,
                        False, cfg["seed"], rank=rk, checkpoints="host")
    ms_hc = slowest(e2e_hc["ms_total"]) / args.steps
    # the recompute-cache hybrid under an HBM budget: the widest agg mirror
    # does not fit, its agg^l is re-aggregated in the backward
    bud = hybrid_budget_gb(ds.graph.num_vertices, dims)
    e2e_b = None
    if world == 1 and cfg["n"] == 1:
        e2e_b = run_epochs(p, plan, ds, dims, "host", args.steps, args.warmup, args.precision,
                           False, cfg["seed"], rank=rk, hbm_budget_gb=bud)
    gat = None
    if not args.no_gat:
        with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk_g:
            gat = gat_measure(p, plan, ds, args.steps, args.warmup, args.precision, cfg["seed"],
                              rk, slowest)
        gat["clocks"] = clk_g.summary()
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    cached = e2e["cache"]
    ckpt_hbm = e2e["ckpt_hbm"]
    h2d, d2h = host_bytes_per_epoch(plan, dims, cached=cached, ckpt_hbm=ckpt_hbm)
    hc_h2d, hc_d2h = host_bytes_per_epoch(plan, dims, cached=e2e_hc["cache"])
    plan_h2d, plan_d2h = host_bytes_per_epoch(plan, dims)
    base_h2d, base_d2h = host_bytes_per_epoch(plan, dims, "baseline")
    virt = None
    if world == 1 and args.config == "cfg2":  # (8 virtual devices' staging fits cfg 2)
        try:
            virt = virtual_fleet_epochs(ds, dims, precision=args.precision, seed=cfg["seed"],
                                        device=int(os.environ.get("LOCAL_RANK", "0")))
        except Exception as exc:  # noqa: BLE001 - report, do not fail the bench
            log(f"[bench] virtual-fleet run failed: {exc}")
    dedup = dedup_report()
    try:
        dedup["at_scale"] = dedup_at_scale(ds, dims, device=int(os.environ.get("LOCAL_RANK", "0")))
    except Exception as exc:  # noqa: BLE001 - report, do not fail the bench
        log(f"[bench] dedup at scale failed: {exc}")
        try:  # the host planner gives the same sets (bit-identical)
            dedup["at_scale"] = dedup_at_scale(ds, dims, device=None)
        except Exception as exc2:  # noqa: BLE001
            log(f"[bench] dedup at scale (host planner) failed: {exc2}")
    pcie = pcie_peaks()
    pcie_bidir = pcie[2] if pcie else None
    # PCIe bytes of one epoch from hardware counters (ncu app-range capture of
    # this workload, profiles/r2_pcie_counters.json), the plan's bytes beside
    pc_src = os.path.join("profiles", "r2_pcie_counters.json")
    pc_e2e = pc_virt = None
    try:
        with open(os.path.join(ROOT, pc_src)) as fh:
            pcj = json.load(fh)
        if pcj.get("e2e", {}).get("config_id") == args.config and m == 1 and cached:
            pc_e2e = pcj["e2e"]
        if pcj.get("virt", {}).get("config_id") == args.config:
            pc_virt = pcj["virt"]
    except (OSError, ValueError):
        pass
    pcie_bytes = pc_e2e["pcie_bytes"] if pc_e2e else h2d + d2h
    if virt and pc_virt:
        vs = virt["ms_per_step"] / 1e3
        virt["pcie_counter_bytes_per_step"] = pc_virt["pcie_bytes"]
        virt["pcie_counter_gbs"] = pc_virt["pcie_bytes"] / vs / 1e9
        virt["pcie_frac_of_bidir_peak"] = pc_virt["pcie_bytes"] / vs / 1e9 / pcie_bidir if pcie_bidir else None
        virt["pcie_counter_file"] = pc_src

    # dominant kernel of the value run: the aggregation kernels (fwd CSC + bwd CSR)
    lf, msf, bf = val["stats"][0]
    lb, msb, bb = val["stats"][1]
    agg_ms = msf + msb
    achieved = (bf + bb) / (agg_ms / 1e3) / 1e9 if agg_ms > 0 else 0.0
    lg, msg, flops = val["stats"][2]
    lt, mst, tb = e2e["stats"][3]
    traffic, traffic_src = None, None
    try:  # DRAM bytes per bracket from the committed ncu launch list of this workload
        with open(os.path.join(ROOT, "profiles", "r3_traffic.json")) as fh:
            tj = json.load(fh)
        if tj.get("config_id") == args.config and tj.get("m") == m:
            traffic, traffic_src = tj["dram_bytes_per_launch"], tj["source"]
    except (OSError, ValueError, KeyError):
        pass
    roofline = {"bound": "hbm", "kernel": "k_seg_work_* (CSC forward + CSR backward aggregation "
                "work lists)",
                "achieved": achieved, "peak": hbm_peak, "peak_source": hbm_src, "unit": "GB/s",
                "frac": achieved / hbm_peak if hbm_peak else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": (bf + bb) / (lf + lb) if lf + lb else None,
                # DRAM view of the same brackets: ncu DRAM bytes per bracket over the
                # bracket's average event time (L2 hits make `frac` exceed 1)
                "dram_gbs": traffic / (agg_ms / (lf + lb) / 1e3) / 1e9 if traffic and lf + lb else None,
                "dram_frac": traffic / (agg_ms / (lf + lb) / 1e3) / 1e9 / hbm_peak
                if traffic and lf + lb and hbm_peak else None,
                "launches_per_step": (lf + lb) / args.steps,
                "share_of_step": agg_ms / val["ms_total"] if val["ms_total"] else None}
    tf32_peak = None
    try:  # measured TF32 tensor-core ceiling (cuBLAS, profiles/tools/tf32_peak.py)
        with open(os.path.join(ROOT, "profiles", "r2_tf32_rates_tma_epilogue.json")) as fh:
            tf32_peak = float(json.load(fh)["cublas_tf32_tflops_8192"])
    except (OSError, ValueError, KeyError):
        pass
    cpu = None
    if not args.no_cpu_baseline:
        cpu = reference_cpu_baseline(ds.graph, ds.labels, ds.mask, dims)
    value = L * E / (ms_v / 1e3) / 1e9
    e2e_v = L * E / (ms_e / 1e3) / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": N_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": ("f32 aggregation / tf32 tcgen05 GEMMs (3xTF32 forward projections)"
                  if args.precision == "tf32" else "f32"),
        "data": "synthetic (seeded clustered power-law graph, random-init Glorot weights)",
        "config": config,
        "e2e": {"value": e2e_v, "unit": "GTEPS", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e,
                "wall_ms_per_step": e2e["wall_s"] / args.steps * 1e3,
                "timing": "ms_per_step: CUDA events on the fleet streams; wall_ms_per_step: "
                          "host perf_counter around the same K train_epoch calls",
                "hbm_owner_cache": bool(cached),
                "checkpoints_in_hbm": bool(ckpt_hbm),
                "pcie_gbs": (h2d + d2h) / (ms_e / 1e3) / 1e9,
                "transfer_kernel_ms_per_step": mst / args.steps},
        "e2e_lean": {"value": L * E / (ms_el / 1e3) / 1e9, "unit": "GTEPS", "ms_per_step": ms_el,
                     "d2h_bytes_per_step": d2h - 4 * int(plan.owner.shape[0]) * (2 * dims[L] + dims[0])
                     if cached and e2e_lean["ckpt_hbm"] == ckpt_hbm else None,
                     "what": "DeviceFleet(lean=True): grad_h^0 not produced, no host copies of "
                             "h^L / grad_h^L (opt-in; not the reference's host contents)"},
        "e2e_host_checkpoints": {
            "value": L * E / (ms_hc / 1e3) / 1e9, "unit": "GTEPS", "ms_per_step": ms_hc,
            "h2d_bytes_per_step": hc_h2d, "d2h_bytes_per_step": hc_d2h,
            "what": "DeviceFleet(checkpoints='host'): agg checkpoints written through to "
                    "host.agg every epoch (the reference's host-side checkpoint cache)"},
        "e2e_hbm_budget": {
            "value": L * E / (e2e_b["ms_total"] / args.steps / 1e3) / 1e9, "unit": "GTEPS",
            "ms_per_step": e2e_b["ms_total"] / args.steps, "hbm_budget_gb": bud,
            "cache": bool(e2e_b["cache"]), "recompute_layers": e2e_b["recompute_layers"],
            "what": "DeviceFleet(hbm_budget_gb=...): the owner cache under a budget that holds "
                    "the h / grad mirrors, the narrowest agg mirror and one scratch - the other "
                    "layers' agg^l re-aggregated in the backward from the h^l mirror (the "
                    "recompute-cache hybrid; a project-first layer needs no agg^l)"}
        if e2e_b else None,
        "epoch_s": {"hbm_resident": ms_v / 1e3, "host_resident": ms_e / 1e3},
        "host_gb_per_epoch": {"measured_path": (h2d + d2h) / 1e9,
                              "hbm_owner_cache": bool(cached),
                              "dedup_full_plan": (plan_h2d + plan_d2h) / 1e9,
                              "non_dedup_baseline_plan": (base_h2d + base_d2h) / 1e9},
        "gpu_launches": int(val["launches"]),
        "gpu_launches_e2e": int(e2e["launches"]),
        "roofline": roofline,
        "gemm": {"ms_per_step": msg / args.steps, "tflops": flops / (msg / 1e3) / 1e12 if msg else None,
                 "precision": args.precision, "tf32_peak_tflops": tf32_peak,
                 "tf32_peak_source": "cuBLAS TF32 8192^3 on this B200 (profiles/r2_tf32_rates_tma_epilogue.json)"
                 if tf32_peak else None,
                 "frac_of_tf32_peak": (flops / (msg / 1e3) / 1e12) / tf32_peak if msg and tf32_peak else None,
                 "note": "useful 2*M*K*N flops (3xTF32 forward projections issue 3x the MMAs); "
                         "the backward GEMMs are HBM-bound at these shapes"},
        "cpu_baseline": cpu,
        "roofline_pcie": {
            "bound": "pcie", "what": "all host<->GPU bytes of the e2e epoch / epoch time",
            "source": "ncu" if pc_e2e else "plan",
            "counter_bytes_per_step": pc_e2e["pcie_bytes"] if pc_e2e else None,
            "counter_file": pc_src if pc_e2e else None,
            "plan_bytes_per_step": h2d + d2h,
            "plan_gbs": (h2d + d2h) / (ms_e / 1e3) / 1e9,
            "d2h_bound_frac": (d2h / (ms_e / 1e3) / 1e9) / pcie[1] if pcie else None,
            "achieved": pcie_bytes / (ms_e / 1e3) / 1e9, "unit": "GB/s",
            "peak": pcie_bidir, "peak_source": "measured (copy engines, both directions at once)",
            "frac": (pcie_bytes / (ms_e / 1e3) / 1e9) / pcie_bidir if pcie_bidir else None,
            "peaks_gbs": {"h2d": pcie[0], "d2h": pcie[1], "bidir": pcie[2],
                          "zero_copy_read": pcie[3], "zero_copy_write": pcie[4]} if pcie else None},
        "dedup": dedup,
        "virtual_fleet_m8": virt,
        "clocks": clk_e.summary(),
        "clocks_value_run": clk_v.summary(),
        "losses": {"value": val["losses"][-1], "e2e": e2e["losses"][-1]},
        "gat": gat,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
