"""Summarise one `ncu --set full` capture (.ncu-rep) into the metrics the
roofline discussion uses: duration, DRAM bytes and throughput, L2 hit rate,
tensor-pipe activity, occupancy limits and the top warp-stall reasons.

    python profiles/summarize_ncu.py gpurun_out/prof_seg.ncu-rep
"""
import csv
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print("-" * 60)
        for i, n in enumerate(h):
            if n in KEYS:
                print(f"{n:64s} {v[i]} {u[i]}")
        pre, post = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
        stalls = []
        for i, n in enumerate(h):
            if n.startswith(pre) and n.endswith(post):
                try:
                    stalls.append((float(v[i]), n[len(pre):-len(post)]))
                except ValueError:
                    pass
        for val, n in sorted(stalls, reverse=True)[:6]:
            print(f"  stalled warps per issue: {n:40s} {val:.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
