"""D2H / H2D copy-engine throughput into large pinned host buffers of
different provenance (does the host store's allocation method matter?)."""
import ctypes as C, mmap, os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2311_14898_b200 import _native as N

GB = 1 << 30
dev = C.c_void_p()
N.call("ht_dev_alloc", 0, 2 * GB, C.byref(dev))
cuda = C.CDLL("libcudart.so") if False else None


def probe(name, host_addr, nbytes):
    # sweep 2 GB copies across the buffer, both directions
    for direction in ("d2h", "h2d"):
        t = time.perf_counter()
        moved = 0
        off = 0
        while off + 2 * GB <= nbytes:
            dst, src = (host_addr + off, dev.value) if direction == "d2h" else (dev.value, host_addr + off)
            N.call("ht_memcpy", dst, src, 2 * GB)
            moved += 2 * GB
            off += 2 * GB
        dt = time.perf_counter() - t
        print(f"{name:40s} {direction}: {moved / dt / 1e9:6.1f} GB/s over {moved / 1e9:.0f} GB", flush=True)


for size_gb in (2, 18):
    p = C.c_void_p()
    N.call("ht_host_alloc", size_gb * GB, C.byref(p))
    C.memset(p.value, 0, size_gb * GB)
    probe(f"cudaHostAlloc {size_gb} GB", p.value, size_gb * GB)
    N.call("ht_host_free", p.value)

# THP-backed anonymous mapping registered with CUDA
size = 18 * GB
m = mmap.mmap(-1, size + 2 * 1024 * 1024, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
buf = (C.c_char * len(m)).from_buffer(m)
addr = (C.addressof(buf) + (2 << 20) - 1) & ~((2 << 20) - 1)
try:
    libc = C.CDLL("libc.so.6")
    MADV_HUGEPAGE = 14
    print("madvise", libc.madvise(C.c_void_p(addr), C.c_size_t(size), MADV_HUGEPAGE))
except OSError as e:
    print("madvise failed", e)
C.memset(addr, 0, size)
N.call("ht_host_register", addr, size)
probe("mmap+THP+cudaHostRegister 18 GB", addr, size)
N.call("ht_host_unregister", addr)
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
print([l for l in open("/proc/meminfo") if "Huge" in l])
