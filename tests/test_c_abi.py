"""The C-ABI used from plain C (no Python in the loop): compile tests/c/abi_smoke.c against
include/libwhit.h and libwhit.so; host checks run here, the GPU run on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2604_00048_b200")


def _build(tmp_path):
    exe = str(tmp_path / "abi_smoke")
    cmd = ["gcc", "-std=c99", "-O1", os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", "-L", PKG, "-lwhit", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{PKG}", "-Wl,-rpath,/usr/local/cuda/lib64", "-lm", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_c_consumer_host(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "host"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "host ok" in out.stdout


@pytest.mark.gpu
def test_c_consumer_gpu(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "gpu ok" in out.stdout
