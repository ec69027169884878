"""The C-ABI library loads on a CPU-only host and exports every entry
point declared in include/hongtu_b200.h (no compute calls here)."""

import ctypes
import os
import re

from conftest import ROOT

from paper_2311_14898_b200 import _native


def _declared():
    text = open(os.path.join(ROOT, "include", "hongtu_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ht_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    names = _declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(_native.exported_symbols()) == set(_declared())


def test_last_error_and_version():
    lib = _native.lib()
    assert lib.ht_version() >= 1
    n = ctypes.c_int(-1)
    assert lib.ht_device_count(ctypes.byref(n)) == 0
    assert n.value >= 0
    # an invalid call reports through the thread-local error string
    out = ctypes.c_int64(0)
    assert lib.ht_set_op(7, None, 0, None, 0, None, ctypes.byref(out)) != 0
    assert b"unknown set op" in lib.ht_last_error()


def test_library_is_sm100a():
    import subprocess
    res = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True)
    assert "sm_100a" in res.stdout, res.stdout[:500]
