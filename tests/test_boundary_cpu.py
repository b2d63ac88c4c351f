"""The C-ABI boundary without a GPU: the library loads, exports every symbol that
include/libwhit.h declares, and its host-side validation / workspace sizing
behave as documented (no compute call is made)."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "libwhit.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(whit_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    import paper_2604_00048_b200._lib as lib
    return lib.lib()


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), n


def test_binding_covers_header():
    import paper_2604_00048_b200._lib as lib
    assert sorted(n for n, _, _ in lib.SIGNATURES) == header_functions()


def test_built_for_sm100a():
    """The shared library carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import subprocess
    so = os.path.join(ROOT, "paper_2604_00048_b200", "libwhit.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_status_strings(L):
    assert L.whit_version() == 100
    assert L.whit_status_string(0) == b"WHIT_OK"
    assert L.whit_status_string(6) == b"WHIT_ERR_STATE"


def test_ws_bytes(L):
    import paper_2604_00048_b200 as P
    # invalid -> 0
    assert L.whit_ws_bytes(0, 100, 128, 0, 1) == 0
    assert L.whit_ws_bytes(4, 100, 128, 0, 1) == 0
    assert L.whit_ws_bytes(2, 2, 128, 0, 1) == 0
    assert L.whit_ws_bytes(2, 100, 128, 7, 1) == 0
    # holds the D z plane + fp64 checkpoints (5 doubles per series per 16 steps at d = 2, plus the
    # backward's 2; two spare chunk slots for the twisted path's halves) + info + the binary-W bit plane
    # (1 bit per date) and one flag per warp + one twisted-path flag per warp
    T, B = 3288, 262144
    n = P.whit_ws_bytes(2, T, B, torch.float32, True)
    dz = (T - 2) * B * 4
    ck = ((T + 15) // 16 + 2) * (5 + 2) * B * 8
    bits = ((T + 31) // 32) * B * 4 + 2 * (B // 32) * 4
    assert dz + ck + 4 * B + bits <= n <= dz + ck + 4 * B + bits + 4096
    assert P.whit_ws_bytes(2, T, B, torch.float64, True) > n


def test_create_validation(L):
    h = ctypes.c_void_p()
    buf = ctypes.c_void_p(1 << 20)  # never dereferenced: validation fails first or create is host-only
    big = 1 << 40
    assert L.whit_ws_create(None, 2, 100, 128, 0, 1, buf, big, None) == 1
    assert L.whit_ws_create(ctypes.byref(h), 0, 100, 128, 0, 1, buf, big, None) == 1
    assert L.whit_ws_create(ctypes.byref(h), 2, 100, 128, 9, 1, buf, big, None) == 1
    assert L.whit_ws_create(ctypes.byref(h), 2, 2, 128, 0, 1, buf, big, None) == 2
    assert L.whit_ws_create(ctypes.byref(h), 2, 100, 130, 0, 1, buf, big, None) == 3   # B % 4
    assert L.whit_ws_create(ctypes.byref(h), 2, 100, 130, 1, 1, buf, big, None) == 0   # f64: B % 2 ok
    L.whit_ws_destroy(h)
    assert L.whit_ws_create(ctypes.byref(h), 2, 100, 128, 0, 1, None, big, None) == 4
    assert L.whit_ws_create(ctypes.byref(h), 2, 100, 128, 0, 1, ctypes.c_void_p((1 << 20) + 16), big, None) == 3
    assert L.whit_ws_create(ctypes.byref(h), 2, 100, 128, 0, 1, buf, 1000, None) == 4
    assert b"required" in L.whit_last_error()


def test_call_validation_before_launch(L):
    h = ctypes.c_void_p()
    assert L.whit_ws_create(ctypes.byref(h), 2, 100, 128, 0, 1, ctypes.c_void_p(1 << 20), 1 << 40, None) == 0
    p = ctypes.c_void_p(1 << 24)
    q = ctypes.c_void_p((1 << 24) + 4)
    # backward before any forward: state error
    assert L.whit_backward(p, h, None, p, p) == 6
    # null pointers, shape mismatch, misalignment, aliasing
    assert L.whit_forward(None, p, p, 2, 100, 128, p, h) == 1
    assert L.whit_forward(p, p, p, 2, 101, 128, ctypes.c_void_p(1 << 25), h) == 2
    assert L.whit_forward(p, p, p, 3, 100, 128, ctypes.c_void_p(1 << 25), h) == 2
    assert L.whit_forward(q, p, p, 2, 100, 128, ctypes.c_void_p(1 << 25), h) == 3
    assert L.whit_forward(p, p, p, 2, 100, 128, p, h) == 1
    assert L.whit_forward(p, p, p, 2, 100, 128, p, None) == 1
    n = ctypes.c_int64()
    assert L.whit_failures(h, ctypes.byref(n), None) == 6
    L.whit_ws_destroy(h)
    L.whit_ws_destroy(None)


def test_path_and_diagnostic_entry_points_validate(L):
    """whit_ws_set_twist / whit_twist_groups / whit_wbits_detected: argument and state checks on the host."""
    h = ctypes.c_void_p()
    assert L.whit_ws_create(ctypes.byref(h), 2, 100, 128, 0, 1, ctypes.c_void_p(1 << 20), 1 << 40, None) == 0
    for mode in (-1, 0, 1, 2):
        assert L.whit_ws_set_twist(h, mode) == 0
    assert L.whit_ws_set_twist(h, 3) == 1 and L.whit_ws_set_twist(h, -2) == 1
    assert L.whit_ws_set_twist(None, 0) == 1
    a, b = ctypes.c_int64(), ctypes.c_int64()
    assert L.whit_twist_groups(h, ctypes.byref(a), ctypes.byref(b)) == 6      # no forward yet
    assert L.whit_wbits_detected(h, ctypes.byref(a), ctypes.byref(b)) == 6
    assert L.whit_twist_groups(h, None, ctypes.byref(b)) == 1
    assert L.whit_wbits_detected(None, ctypes.byref(a), ctypes.byref(b)) == 1
    L.whit_ws_destroy(h)


def test_python_binding_refuses_cpu_tensors():
    import paper_2604_00048_b200 as P
    y = torch.zeros(10, 4)
    with pytest.raises(ValueError):
        P.smooth(y, y, torch.ones(8, 4), 2)


def test_python_binding_rejects_mismatched_lambda_mode_and_shapes():
    """The pointer ABI cannot see tensor shapes; the binding checks lambda's mode and the planes' shapes
    against the workspace before any launch (host-only: works without a GPU)."""
    import types

    import pytest
    import torch
    from paper_2604_00048_b200 import _lib as L

    ws = types.SimpleNamespace(T=50, B=8, d=2, C=1, per_date=True, dtype=torch.float32, device_check=False)
    y = torch.zeros(50, 8)
    with pytest.raises(ValueError, match="lambda shape"):
        L._shapes(ws, "whit_forward", torch.zeros(8), ("y", y, "TB"))
    with pytest.raises(ValueError, match="y shape"):
        L._shapes(ws, "whit_forward", torch.zeros(48, 8), ("y", torch.zeros(49, 8), "TB"))
    L._shapes(ws, "whit_forward", torch.zeros(48, 8), ("y", y, "TB"))
    with pytest.raises(ValueError, match="contiguous"):
        L._shapes(ws, "whit_forward", torch.zeros(48, 8), ("y", torch.zeros(8, 50).t(), "TB"))
    with pytest.raises(TypeError, match="dtype"):
        L._shapes(ws, "whit_forward", torch.zeros(48, 8), ("y", torch.zeros(50, 8, dtype=torch.float64), "TB"))
    ws3 = types.SimpleNamespace(T=50, B=8, d=2, C=3, per_date=False, dtype=torch.float32, device_check=False)
    L._shapes(ws3, "whit_forward_bands", torch.zeros(8), ("y", torch.zeros(3, 50, 8), "CTB"), C=3)
    with pytest.raises(ValueError):
        L._shapes(ws3, "whit_forward_bands", torch.zeros(8), ("y", torch.zeros(2, 50, 8), "CTB"), C=3)


def test_missing_library_fails_loudly(tmp_path):
    """Without libwhit.so the package refuses to import (no CPU fallback)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WHIT_LIB_PATH=str(tmp_path / "missing" / "libwhit.so"))
    out = subprocess.run([sys.executable, "-c", "import paper_2604_00048_b200"], cwd=root, env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode != 0 and "ImportError" in out.stderr and "no CPU fallback" in out.stderr
