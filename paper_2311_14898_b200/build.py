"""Build the native library in-tree: ``python -m paper_2311_14898_b200.build``.

nvcc cross-compiles for sm_100a only (no GPU needed).  Each translation unit
compiles to an object in ``build/`` (in parallel, rebuilt when it or any
header changed); the objects link into ``lib/libhongtu_b200.so``, which links
the CUDA runtime statically and travels with the repository snapshot to the
GPU box.
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(HERE, "..", "include")
OBJ = os.path.join(HERE, "build")
OUT = os.path.join(HERE, "lib", "libhongtu_b200.so")
SOURCES = ["ht_runtime.cu", "ht_fleet.cu", "ht_gcn.cu", "ht_gat_layers.cu", "ht_probe.cu",
           "ht_gplan.cu", "ht_prep.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O3,-fopenmp",
                 "-Xptxas", "-v", f"-I{INCLUDE}"]
LINK_FLAGS = [*ARCH, "-shared", "-cudart", "static", "-lgomp"]


def _headers():
    out = []
    for root in (CSRC, INCLUDE):
        out += [os.path.join(root, f) for f in os.listdir(root) if f.endswith((".h", ".cuh"))]
    return out


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def _obj(src):
    return os.path.join(OBJ, os.path.splitext(src)[0] + ".o")


def _stale_objs(force):
    newest_hdr = max((_mtime(h) for h in _headers()), default=0.0)
    out = []
    for s in SOURCES:
        o = _obj(s)
        if force or _mtime(o) < max(_mtime(os.path.join(CSRC, s)), newest_hdr):
            out.append(s)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    stale = _stale_objs(force)
    if not stale and _mtime(OUT) >= max(_mtime(_obj(s)) for s in SOURCES):
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

    def compile_one(src):
        cmd = [nvcc, *COMPILE_FLAGS, "-c", "-o", _obj(src) + ".tmp", os.path.join(CSRC, src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode == 0:
            os.replace(_obj(src) + ".tmp", _obj(src))
        return src, res

    with ThreadPoolExecutor(max_workers=min(len(stale), os.cpu_count() or 4) or 1) as ex:
        results = list(ex.map(compile_one, stale))
    failed = [(s, r) for s, r in results if r.returncode != 0]
    for s, r in results:
        if verbose or r.returncode != 0:
            sys.stderr.write(f"== {s}\n{r.stdout}{r.stderr}")
    if failed:
        raise RuntimeError("nvcc failed on " + ", ".join(s for s, _ in failed))
    cmd = [nvcc, *LINK_FLAGS, "-o", OUT + ".tmp", *[_obj(s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libhongtu_b200.so")
    os.replace(OUT + ".tmp", OUT)
    return OUT


def build_variant(name: str, defines: list) -> str:
    """A same-box A/B build: every source compiled with extra ``-D`` flags
    into ``build/<name>/`` and linked to ``lib/variants/<name>/`` (load it
    with ``HT_LIB=<path>``).  Not part of the product build."""
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    odir = os.path.join(OBJ, name)
    out = os.path.join(HERE, "lib", "variants", name, "libhongtu_b200.so")
    os.makedirs(odir, exist_ok=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    flags = [f"-D{d}" for d in defines]

    def compile_one(src):
        o = os.path.join(odir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, *COMPILE_FLAGS, *flags, "-c", "-o", o, os.path.join(CSRC, src)]
        return o, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for o, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"variant {name}: nvcc failed on {o}")
    res = subprocess.run([nvcc, *LINK_FLAGS, "-o", out, *[o for o, _ in results]],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"variant {name}: link failed")
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
