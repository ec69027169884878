"""DRAM traffic of the bench's dominant kernel class from an ncu launch list.

    python profiles/make_traffic.py LAUNCHES.csv EPOCHS > profiles/r2_traffic.json

The launch list is `ncu --profile-from-start off --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum,... --clock-control none --csv` of
`bench.py --profile-epoch value --steps 1 --warmup 2` (EPOCHS = 1: only the
epoch inside the profiler range is captured).  The aggregation class
(bench.py `roofline`) is the forward CSC + backward CSR work-list launches
(r1: the segment gathers with their piece / fixup kernels); bench.py times it
as L forward + L backward brackets per epoch, so the traffic per bracket is
(DRAM read + write of those kernels) / (EPOCHS * 2 L).  bench.py reports it
as `roofline.traffic` for the workload it was captured on.
"""
import collections
import csv
import json
import re
import sys

AGG = re.compile(r"k_seg_(work|gather|pieces|fixup)")


def main(path, epochs, layers=3):
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.defaultdict(dict)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], None)
            per[d["ID"]]["name"] = d["Kernel Name"]
            if unit is not None:
                per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * unit
    # kernels after the last SGD step belong to no epoch (e.g. a deferred
    # checkpoint aggregated when the fleet is closed): not counted
    ids = sorted(per, key=int)
    last_sgd = max((int(k) for k in ids if "k_sgd" in per[k]["name"]), default=None)
    tot, n = 0.0, 0
    for k in ids:
        v = per[k]
        if last_sgd is not None and int(k) > last_sgd:
            continue
        if AGG.search(v["name"]):
            tot += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
            n += 1
    brackets = epochs * 2 * layers
    print(json.dumps({"config_id": "cfg2", "m": 1, "kernel_class": "k_seg_work_* (CSC fwd + CSR bwd work lists)",
                      "dram_bytes_per_launch": tot / brackets, "brackets": brackets,
                      "kernel_launches": n, "source": path,
                      "capture": "ncu --profile-from-start off --metrics dram__bytes_read.sum,"
                                 "dram__bytes_write.sum --clock-control none, bench.py "
                                 "--profile-epoch value --steps 1 --warmup 2"},
                     indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
