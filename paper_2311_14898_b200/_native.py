"""ctypes binding of the C ABI in include/hongtu_b200.h.

The shared library ``lib/libhongtu_b200.so`` is built in-tree by
``__graft_entry__.build()`` (or ``python -m paper_2311_14898_b200.build``).
There is no fallback: if the library is missing every entry point raises
``NativeLibraryError`` with the build command.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

from .errors import ChunktrainError, DeviceError, PlanError, SimulationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# HT_LIB: an alternative build of the same library (same-box A/B timing)
LIB_PATH = os.environ.get("HT_LIB") or os.path.join(_HERE, "lib", "libhongtu_b200.so")

HT_OK, HT_EINVAL, HT_ECUDA, HT_ESTATE, HT_ELIVE, HT_ENOMEM = 0, -1, -2, -3, -4, -5

i32, i64, f32, f64, vp = C.c_int, C.c_int64, C.c_float, C.c_double, C.c_void_p
P_I64 = C.POINTER(C.c_int64)
P_F64 = C.POINTER(C.c_double)


class NativeLibraryError(ChunktrainError):
    """The CUDA extension is not built or cannot be loaded."""


_SIGS = {
    "ht_last_error": (C.c_char_p, []),
    "ht_version": (i32, []),
    "ht_device_count": (i32, [C.POINTER(i32)]),
    "ht_host_alloc": (i32, [i64, C.POINTER(vp)]),
    "ht_host_free": (i32, [vp]),
    "ht_host_register": (i32, [vp, i64]),
    "ht_host_unregister": (i32, [vp]),
    "ht_dev_alloc": (i32, [i32, i64, C.POINTER(vp)]),
    "ht_dev_free": (i32, [i32, vp]),
    "ht_memcpy": (i32, [vp, vp, i64]),
    "ht_memset": (i32, [vp, i32, i64]),
    "ht_build_graph": (i32, [vp, vp, i64, i64, vp, vp, vp, vp, vp, vp]),
    "ht_build_graph_dedup32": (i32, [vp, vp, i64, i64, vp, vp, vp, vp, vp, vp, vp]),
    "ht_dedup_edges": (i32, [vp, vp, i64, i64, vp, P_I64]),
    "ht_csr_perm": (i32, [i64, i64, vp, vp, vp, vp]),
    "ht_ldg_partition": (i32, [i64, vp, vp, vp, vp, vp, i64, i64, vp]),
    "ht_chunk_fill": (i32, [vp, vp, vp, vp, i64, vp, P_I64, vp, vp, vp, vp, vp, vp]),
    "ht_set_op": (i32, [i32, vp, i64, vp, i64, vp, P_I64]),
    "ht_intersect_count": (i64, [vp, i64, vp, i64]),
    "ht_slot_layout": (i32, [i64, vp, vp, vp, P_I64]),
    "ht_reorganize": (i32, [i64, i64, vp, vp, i32, vp, vp]),
    "ht_gplan_build": (i32, [i32, i32, i32, i64, vp, vp, vp, C.POINTER(vp)]),
    "ht_gplan_count": (i32, [vp, P_I64]),
    "ht_gplan_sizes": (i32, [vp, vp, vp, vp]),
    "ht_gplan_fetch": (i32, [vp, vp]),
    "ht_gplan_free": (i32, [vp]),
    "ht_fleet_create": (i32, [i32, i32, vp, i32, i32, C.POINTER(vp)]),
    "ht_fleet_destroy": (i32, [vp]),
    "ht_fleet_create_rank": (i32, [i32, i32, i32, i32, i32, i32, C.POINTER(vp)]),
    "ht_fleet_ipc_export": (i32, [vp, vp]),
    "ht_fleet_ipc_import": (i32, [vp, i32, vp]),
    "ht_fleet_set_sets": (i32, [vp, i32, i32, vp, i64, vp, i64, vp, i64, vp, i64, vp, vp, i64,
                                vp, i64]),
    "ht_fleet_set_fetch": (i32, [vp, i32, i32, i32, vp, i64]),
    "ht_fleet_set_chunk": (i32, [vp, i32, i32, i64, i64, i64, vp, vp, vp, vp, vp, vp]),
    "ht_fleet_finalize": (i32, [vp]),
    "ht_fleet_capacity": (i32, [vp, i32, P_I64]),
    "ht_begin_layer": (i32, [vp, i32, i32, i32]),
    "ht_comm_fwd": (i32, [vp, i32, vp, vp]),
    "ht_comm_bwd": (i32, [vp, i32, vp, vp]),
    "ht_dest_rows": (i32, [vp, i32, i32, i32, i32, vp, vp]),
    "ht_epoch_begin": (i32, [vp, i32, vp]),
    "ht_forward_layer": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, i32]),
    "ht_loss": (i32, [vp, i32, vp, vp, i64, i64, vp, P_F64]),
    "ht_loss_value": (i32, [vp, P_F64]),
    "ht_backward_layer": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, i32]),
    "ht_sgd": (i32, [vp, i32, vp, vp, f32, vp]),
    "ht_sgd2": (i32, [vp, i32, vp, vp, vp, f32, vp, vp]),
    "ht_gat_epoch_begin": (i32, [vp, i32, vp]),
    "ht_fleet_set_cache": (i32, [vp, i32]),
    "ht_fleet_set_host_rows": (i32, [vp, vp, i64]),
    "ht_fleet_set_lean": (i32, [vp, i32]),
    "ht_fleet_set_budget": (i32, [vp, i64]),
    "ht_fleet_recompute_state": (i32, [vp, C.POINTER(i64)]),
    "ht_fleet_set_checkpoints": (i32, [vp, i32]),
    "ht_fleet_checkpoint_read": (i32, [vp, i32, vp]),
    "ht_fleet_alias_store": (i32, [vp, i32, vp, vp, vp]),
    "ht_fleet_cache_state": (i32, [vp, C.POINTER(i32)]),
    "ht_gat_forward_layer": (i32, [vp, i32, i32, i32, vp, vp, f32, vp, vp, i32]),
    "ht_gat_backward_layer": (i32, [vp, i32, i32, i32, vp, vp, f32, vp, vp, vp, i32]),
    "ht_fleet_sync": (i32, [vp]),
    "ht_set_timing": (i32, [vp, i32]),
    "ht_kernel_stats": (i32, [vp, i32, P_I64, P_F64, P_F64]),
    "ht_fleet_mark": (i32, [vp, i32]),
    "ht_fleet_elapsed": (i32, [vp, P_F64]),
    "ht_fleet_elapsed_between": (i32, [vp, i32, i32, P_F64]),
    "ht_launches": (i64, []),
    "ht_gemm_test": (i32, [i32, i32, vp, vp, vp, vp, i64, i32, i32]),
    "ht_pcie_probe": (i32, [i32, i64, vp]),
    "ht_gemm_rate": (i32, [i32, i32, i64, i32, i32, i32, vp]),
    "ht_profile_range": (i32, [i32]),
    "ht_mem_info": (i32, [i32, P_I64, P_I64]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the native library; raises loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"native library {LIB_PATH} is missing; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` from the repo root")
            try:
                h = C.CDLL(LIB_PATH)
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def check(rc: int, kind=None):
    """Map a native status code onto the package's exception types."""
    if rc == HT_OK:
        return
    msg = lib().ht_last_error().decode(errors="replace")
    if kind is not None:
        raise kind(msg)
    if rc == HT_ECUDA:
        raise DeviceError(msg)
    if rc in (HT_ESTATE, HT_ELIVE):
        raise SimulationError(msg)
    raise PlanError(msg) if "plan" in msg else SimulationError(msg)


def call(name, *args, kind=None):
    check(getattr(lib(), name)(*args), kind)


def ptr(a) -> int | None:
    """Data pointer of a numpy array (or DeviceArray), None for None."""
    if a is None:
        return None
    if hasattr(a, "device_ptr"):
        return a.device_ptr
    return a.ctypes.data


def device_count() -> int:
    n = i32(0)
    call("ht_device_count", C.byref(n))
    return int(n.value)


# ---------------------------------------------------------------------------
# pinned host arrays
# ---------------------------------------------------------------------------

_pinned_ranges: dict[int, int] = {}


def _free_pinned(p: int):
    _pinned_ranges.pop(p, None)
    if _lib is not None:
        _lib.ht_host_free(p)


def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy array in pinned, portable, mapped host memory (zero-copy
    readable/writable by every GPU)."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    p = vp()
    call("ht_host_alloc", max(nbytes, 16), C.byref(p), kind=DeviceError)
    addr = int(p.value)
    buf = (C.c_byte * max(nbytes, 16)).from_address(addr)
    weakref.finalize(buf, _free_pinned, addr)
    _pinned_ranges[addr] = max(nbytes, 16)
    arr = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype).reshape(shape)
    return arr


def pinned_zeros(shape, dtype) -> np.ndarray:
    a = pinned_empty(shape, dtype)
    a.fill(0)
    return a


def is_pinned(a: np.ndarray) -> bool:
    if hasattr(a, "device_ptr"):
        return True
    lo = a.ctypes.data
    hi = lo + a.nbytes
    for base, size in _pinned_ranges.items():
        if base <= lo and hi <= base + size:
            return True
    return False


def staged(a: np.ndarray, dtype=None) -> np.ndarray:
    """A pinned, C-contiguous array with a's contents (a itself if it
    already qualifies)."""
    dtype = np.dtype(dtype or a.dtype)
    if (hasattr(a, "device_ptr") or
            (a.dtype == dtype and a.flags.c_contiguous and is_pinned(a))):
        return a
    out = pinned_empty(a.shape, dtype)
    out[...] = a
    return out


def mem_info(device: int = 0):
    """(free, total) HBM bytes of a device."""
    fr, tot = C.c_int64(0), C.c_int64(0)
    call("ht_mem_info", device, C.byref(fr), C.byref(tot))
    return int(fr.value), int(tot.value)
