"""PCIe counter evidence of whole epochs (ncu --replay-mode app-range over
bench.py --profile-epoch MODE, one epoch inside cudaProfilerStart/Stop):
pcie__read_bytes.sum (the GPU reading host memory: H2D) and
pcie__write_bytes.sum (D2H), 512-byte granularity, next to the bytes the
plan predicts for the same epoch.  Writes the JSON bench.py's roofline_pcie
reads.

    python profiles/tools/pcie_counters.py OUT.json e2e=CSV,LOG virt=CSV,LOG
"""
import csv
import json
import sys


def counters(path):
    out = {}
    for r in csv.reader(open(path)):
        if len(r) == 13 and r[0] != "ID":
            out[r[10]] = float(r[12].replace(",", ""))
    return out


def plan_line(path):
    for line in open(path):
        if line.startswith("{"):
            return json.loads(line)
    return {}


if __name__ == "__main__":
    res = {"what": "ncu --replay-mode app-range, one epoch between cudaProfilerStart/Stop "
                   "(bench.py --profile-epoch MODE --steps 1); pcie__read_bytes = host->GPU, "
                   "pcie__write_bytes = GPU->host (512 B granularity); times under the "
                   "profiler are not bench values"}
    for arg in sys.argv[2:]:
        mode, files = arg.split("=")
        csvp, logp = files.split(",")
        c, p = counters(csvp), plan_line(logp)
        rd, wr = c.get("pcie__read_bytes.sum"), c.get("pcie__write_bytes.sum")
        e = {"config_id": p.get("config_id"), "pcie_read_bytes": rd, "pcie_write_bytes": wr,
             "pcie_bytes": (rd or 0) + (wr or 0),
             "dram_bytes": (c["dram__bytes_read.sum"] + c["dram__bytes_write.sum"])
             if "dram__bytes_read.sum" in c else None,
             "range_ns_under_profiler": c.get("gpu__time_duration.sum")}
        if "planned_h2d_gb_per_step" in p:
            e["planned_h2d_bytes"] = p["planned_h2d_gb_per_step"] * 1e9
            e["planned_d2h_bytes"] = p["planned_d2h_gb_per_step"] * 1e9
            e["planned_bytes"] = e["planned_h2d_bytes"] + e["planned_d2h_bytes"]
        if "planned_host_gb_per_step" in p:
            e["planned_bytes"] = p["planned_host_gb_per_step"] * 1e9
            e["metered_bytes"] = p["metered_host_gb_per_step"] * 1e9
        if e.get("planned_bytes"):
            e["counter_over_plan"] = e["pcie_bytes"] / e["planned_bytes"]
        res[mode] = e
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(res, indent=1))
