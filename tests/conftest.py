import os
import sys

# The library picks the twisted (two-ended) path for small batches by default; the suite's tests target the
# sequential kernels unless they ask for the twisted path explicitly (test_gpu_twist.py: whit_ws_set_twist).
os.environ.setdefault("WHIT_TWIST", "0")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long CPU test")
