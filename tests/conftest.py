import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long CPU test")


def _has_gpu():
    try:
        import ctypes
        rt = ctypes.CDLL("libcudart.so.12")
    except OSError:
        try:
            import torch
            return torch.cuda.is_available()
        except Exception:
            return False
    n = ctypes.c_int(0)
    return rt.cudaGetDeviceCount(ctypes.byref(n)) == 0 and n.value > 0


HAS_GPU = None


def pytest_collection_modifyitems(config, items):
    global HAS_GPU
    marker_expr = config.getoption("-m") or ""
    if "gpu" in marker_expr and "not gpu" not in marker_expr:
        return  # explicitly asked for GPU tests: let them fail loudly without a device
    if HAS_GPU is None:
        HAS_GPU = _has_gpu()
    if not HAS_GPU:
        skip = pytest.mark.skip(reason="no CUDA device")
        for it in items:
            if "gpu" in it.keywords:
                it.add_marker(skip)
