"""The C-ABI library loads and exports every symbol include/lgdm.h declares (CPU only;
no compute calls), and host-side argument validation fails cleanly."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2301_06503_b200 import lgdm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lgdm.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    # debug-build-only entry points (compiled with -DLGDM_PHASE_TIMING) are not exported
    text = re.sub(r"#ifdef LGDM_PHASE_TIMING.*?#endif", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lgdm_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = lgdm.load()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), f"liblgdm.so does not export {s}"
    assert sorted(lgdm.EXPORTS) == syms


def test_nm_dynamic_symbols():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", lgdm.LIB_PATH], capture_output=True,
                         text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_enums_match_header():
    text = open(HEADER).read()
    for name, val in (("LGDM_BAR2", 1), ("LGDM_QUAD4", 2), ("LGDM_HEX8", 3)):
        assert re.search(rf"{name}\s*=\s*{val}\b", text)
    for code, name in lgdm.STATUS.items():
        assert re.search(rf"{name}\s*=\s*{code}\b", text)
    assert C.sizeof(lgdm.Material) == 12 * 8 + 8


def test_invalid_arguments_fail_before_any_device_work():
    L = lgdm.load()
    h = C.c_void_p()
    coords = np.zeros((4, 2))
    conn = np.array([[0, 1, 2, 3]], dtype=np.int64)
    mat = lgdm.material(E=3e4, nu=0.2, k=10, kappa0=1e-4, alpha=0.99, beta=300, h=3e4,
                        h_sigma=3e4, c=2, R=0.05, n=5, t=1)
    st = L.lgdm_create_mesh(9, 4, coords.ctypes.data, 1, conn.ctypes.data, C.byref(mat), 0, 4, 0,
                            4, 0, None, C.byref(h))
    assert st == 1 and b"unknown element type" in L.lgdm_last_error()
    bad = lgdm.material(E=-1.0, nu=0.2, k=10, kappa0=1e-4, alpha=0.99, beta=300, h=3e4,
                        h_sigma=3e4, c=2, R=0.05, n=5, t=1)
    st = L.lgdm_create_mesh(2, 4, coords.ctypes.data, 1, conn.ctypes.data, C.byref(bad), 0, 4, 0,
                            4, 0, None, C.byref(h))
    assert st == 1 and b"material" in L.lgdm_last_error()
    conn_bad = np.array([[0, 1, 2, 7]], dtype=np.int64)
    st = L.lgdm_create_mesh(2, 4, coords.ctypes.data, 1, conn_bad.ctypes.data, C.byref(mat), 0, 4,
                            0, 4, 0, None, C.byref(h))
    assert st == 1 and b"out of range" in L.lgdm_last_error()
    st = L.lgdm_create_mesh(2, 4, coords.ctypes.data, 1, conn.ctypes.data, C.byref(mat), 0, 4, 3,
                            2, 0, None, C.byref(h))
    assert st == 1
    assert L.lgdm_assemble(None, None, None) == 1
    assert L.lgdm_launch_count(None) == -1


def test_empty_and_degenerate_inputs_rejected():
    """Edge cases of the boundary (include/lgdm.h, lgdm_create_mesh): an empty mesh (no
    elements, fewer than 2 nodes), an empty owned range, a mixed-order node in no element or
    both corner and midside -- each LGDM_ERR_INVALID_ARGUMENT before any device is touched."""
    L = lgdm.load()
    h = C.c_void_p()
    mat = lgdm.material(E=3e4, nu=0.2, k=10, kappa0=1e-4, alpha=0.99, beta=300, h=3e4,
                        h_sigma=3e4, c=2, R=0.05, n=5, t=1)
    coords = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=float)
    conn = np.array([[0, 1, 2, 3]], dtype=np.int64)
    for etype in (lgdm.QUAD4, lgdm.QUAD8):
        st = L.lgdm_create_mesh(etype, 4, coords.ctypes.data, 0, conn.ctypes.data, C.byref(mat), 0,
                                4, 0, 4, 0, None, C.byref(h))
        assert st == 1 and b"bad sizes" in L.lgdm_last_error()
        st = L.lgdm_create_mesh(etype, 1, coords.ctypes.data, 1, conn.ctypes.data, C.byref(mat), 0,
                                1, 0, 1, 0, None, C.byref(h))
        assert st == 1 and b"bad sizes" in L.lgdm_last_error()
    for b, e in ((2, 2), (0, 0), (0, 5), (-1, 2)):   # empty / out-of-range owned ranges
        st = L.lgdm_create_mesh(lgdm.QUAD4, 4, coords.ctypes.data, 1, conn.ctypes.data,
                                C.byref(mat), 0, 4, b, e, 0, None, C.byref(h))
        assert st == 1 and b"owned node range" in L.lgdm_last_error()
    x8 = np.array([[0, 0], [2, 0], [2, 2], [0, 2], [1, 0], [2, 1], [1, 2], [0, 1], [5, 5]], float)
    c8 = np.array([[0, 1, 2, 3, 4, 5, 6, 7]], dtype=np.int64)
    st = L.lgdm_create_mesh(lgdm.QUAD8, 9, x8.ctypes.data, 1, c8.ctypes.data, C.byref(mat), 0, 9,
                            0, 9, 0, None, C.byref(h))
    assert st == 1 and b"belongs to no element" in L.lgdm_last_error()
    c8b = np.array([[0, 1, 2, 3, 4, 5, 6, 7], [4, 8, 6, 5, 0, 1, 2, 3]], dtype=np.int64)
    st = L.lgdm_create_mesh(lgdm.QUAD8, 9, x8.ctypes.data, 2, c8b.ctypes.data, C.byref(mat), 0, 9,
                            0, 9, 0, None, C.byref(h))
    assert st == 1 and b"corner of one element and a midside" in L.lgdm_last_error()
    assert not h.value


def test_no_gpu_means_loud_failure():
    """Without a CUDA device the library refuses to run (there is no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = lgdm.load()
    h = C.c_void_p()
    coords = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=float)
    conn = np.array([[0, 1, 2, 3]], dtype=np.int64)
    mat = lgdm.material(E=3e4, nu=0.2, k=10, kappa0=1e-4, alpha=0.99, beta=300, h=3e4,
                        h_sigma=3e4, c=2, R=0.05, n=5, t=1)
    st = L.lgdm_create_mesh(2, 4, coords.ctypes.data, 1, conn.ctypes.data, C.byref(mat), 0, 4, 0,
                            4, 0, None, C.byref(h))
    assert st == 5 and b"no CUDA device" in L.lgdm_last_error()
