"""CPU-side checks of the boundary: the C-ABI library loads, exports exactly the
symbols include/lsg_sgmv.h declares, and host-side validation works without a GPU
(validation runs before any CUDA call)."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2310_18547_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lsg_sgmv.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lsg_[a-z_0-9]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (lsg_[a-z_0-9]+)", out))
    missing = set(declared_functions()) - exported
    assert not missing, missing
    L = _lib.lib()
    for name in declared_functions():
        assert getattr(L, name) is not None


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_status_strings_and_version():
    L = _lib.lib()
    assert L.lsg_version() >= 100
    assert b"LSG_EINVAL" in L.lsg_status_string(-1)
    assert L.lsg_status_string(0) == b"LSG_OK"


def _table(**kw):
    t = _lib.WeightTable(C.c_void_p(16), C.c_void_p(32), 4096 * 16, 16 * 4096, 8, 2, 4096, 4096, 16, 0)
    for k, v in kw.items():
        setattr(t, k, v)
    return t


@pytest.mark.parametrize("field,value,msg", [
    ("rank", 0, b"rank"), ("rank", 5000, b"rank"), ("h_in", 0, b"dims"), ("num_layers", 0, b"layer"),
    ("a_layer_stride", 10, b"strides"), ("dtype", 7, b"dtype")])
def test_host_validation_without_gpu(field, value, msg):
    L = _lib.lib()
    t = _table(**{field: value})
    st = L.lsg_sgmv(C.c_void_p(16), 4096, C.c_void_p(16), 4096, C.byref(t), C.c_void_p(16), C.c_void_p(16),
                    1, 4, 0, None)
    assert st in (_lib.LSG_EINVAL, _lib.LSG_EUNSUPPORTED)
    assert msg in L.lsg_last_error()


def test_layer_and_null_checks_without_gpu():
    L = _lib.lib()
    t = _table()
    assert L.lsg_sgmv(C.c_void_p(16), 4096, C.c_void_p(16), 4096, C.byref(t), C.c_void_p(16), C.c_void_p(16),
                      1, 4, 2, None) == _lib.LSG_EINVAL
    assert b"layer" in L.lsg_last_error()
    assert L.lsg_sgmv(None, 4096, C.c_void_p(16), 4096, C.byref(t), C.c_void_p(16), C.c_void_p(16), 1, 4, 0,
                      None) == _lib.LSG_EINVAL
    # an empty batch is a successful no-op, like lora_addon on an empty Batch (sgmv.cpp:139)
    assert L.lsg_sgmv(None, 0, None, 0, C.byref(t), None, None, 0, 0, 0, None) == _lib.LSG_OK
    assert L.lsg_set_option(_lib.LSG_OPT_FORCE_CLUSTER, 99) == _lib.LSG_EINVAL
    assert L.lsg_set_option(_lib.LSG_OPT_FORCE_CLUSTER, 0) == _lib.LSG_OK


def test_launch_planning_is_host_only():
    """The plan for the headline shape: the cluster split-K fast path, one wave."""
    L = _lib.lib()
    t = _table(num_slots=64)
    info = _lib.LaunchInfo()
    assert L.lsg_query_launch(C.byref(t), 64, 64, _lib.KERNEL_FUSED, C.byref(info)) == 0
    assert info.path == 0 and info.tile_rows == 1 and info.cluster >= 2
    assert info.smem_bytes <= 227 * 1024
    assert L.lsg_query_launch(C.byref(t), 1, 64, _lib.KERNEL_FUSED, C.byref(info)) == 0  # Identical
    # one row per cluster for every popularity (tile-scan); co-resident at 3 CTAs/SM
    assert info.tile_rows == 1 and info.grid_ctas <= 148 * 2 and info.smem_bytes <= 75 * 1024
    t2 = _table(h_in=136)
    assert L.lsg_query_launch(C.byref(t2), 4, 4, _lib.KERNEL_FUSED, C.byref(info)) == 0
    assert info.path == 1  # h_in not a multiple of 128 -> generic kernel


def test_dropin_library_defines_exactly_the_reference_sgmv_cpp_symbols():
    """liblorasim_sgmv_b200.so replaces core/src/sgmv.cpp one for one: its lorasim:: text
    symbols (outside this repo's lorasim::b200 extras) are exactly the ones sgmv.cpp defines
    (tests/golden/sgmv_cpp_symbols.txt, from the reference compiled by make_golden.py), so a
    reference build that drops sgmv.cpp links it with no duplicate and no missing symbol."""
    import subprocess
    so = os.path.join(ROOT, "paper_2310_18547_b200", "lib", "liblorasim_sgmv_b200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", so], capture_output=True, text=True, check=True).stdout
    ours = sorted({ln.split(" T ", 1)[1] for ln in out.splitlines()
                   if " T " in ln and "lorasim::" in ln and "lorasim::b200::" not in ln})
    golden = [ln for ln in open(os.path.join(ROOT, "tests", "golden", "sgmv_cpp_symbols.txt")).read().splitlines() if ln]
    assert ours == golden
