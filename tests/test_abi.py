"""The C-ABI library builds, loads and exports every entry point include/trd.h declares
(CPU only: no compute calls)."""
import ctypes
import os
import subprocess

import pytest

from paper_2305_09044_b200 import build as B
from paper_2305_09044_b200 import trd as T


def test_library_builds_and_exports_all_declared_symbols():
    lib_path = B.build()
    assert os.path.exists(lib_path)
    lib = T.load_library(lib_path)
    names = T.declared_symbols()
    assert len(names) >= 12
    for n in ["trd_init", "trd_sketch", "trd_sweep", "trd_reconstruct", "trd_error"]:
        assert n in names
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for n in names:
        assert n in exported, n
        assert hasattr(lib, n)
    assert lib.trd_version().startswith(b"libtrd")


def test_sm100a_code_in_library():
    """The fat binary carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    lib_path = B.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_rejected_without_gpu():
    """Argument validation happens before anything touches the device."""
    lib = T.load_library()
    cfg = T.trd_config()
    cfg.order = 2                       # N < 3 -> TRD_ERR_SHAPE
    sh = T.trd_shard()
    ctx = ctypes.c_void_p()
    arr = (ctypes.c_void_p * 8)()
    assert lib.trd_init(ctypes.byref(cfg), ctypes.byref(sh), arr, None, ctypes.byref(ctx)) in (1, 2)
    assert ctx.value is None
    assert lib.trd_init(None, None, None, None, ctypes.byref(ctx)) == 1
    cfg.order = 3
    for m in range(3):
        cfg.dims[m] = 4
        cfg.ranks[m] = 99               # rank > TRD_MAX_RANK
    assert lib.trd_init(ctypes.byref(cfg), ctypes.byref(sh), arr, None, ctypes.byref(ctx)) in (1, 2)
    assert lib.trd_sweep(None, 1, None) == 1
    assert lib.trd_destroy(None) is None
