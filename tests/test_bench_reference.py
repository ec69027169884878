"""The bench's CPU reference arm (`bench.py --impl reference`) times the
reference's own CPU path and must not load this repository's native
library or touch a GPU."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import json, sys, types
sys.argv = ["bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "1"]
import bench
bench.main()
maps = open("/proc/self/maps").read()
print(json.dumps({"so_loaded": "libhongtu_b200" in maps,
                  "cuda_loaded": "libcuda.so" in maps}))
"""


def test_reference_arm_runs_without_native_library():
    r = subprocess.run([sys.executable, "-c", SNIPPET], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert line["impl"] == "reference"
    assert line["steps"] == 2 and line["warmup"] == 1
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert "not extrapolated" in line["cpu_baseline"]["sample"]
    assert not probe["so_loaded"], "reference arm loaded libhongtu_b200.so"
    assert not probe["cuda_loaded"]
