import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _gpu_status():
    """(device count, reason) as seen by the product library itself: libspin.so
    links the CUDA runtime statically, so no framework is involved."""
    try:
        from paper_2503_15921_b200 import _lib

        n = _lib.device_count()
        return n, "" if n else _lib.load().spin_last_error().decode()
    except Exception as e:  # library missing or not loadable
        return 0, f"libspin.so not loadable: {e}"


def _gpu_selected(config) -> bool:
    expr = (config.getoption("-m") or "").replace(" ", "")
    return "gpu" in expr and "notgpu" not in expr


def pytest_collection_modifyitems(config, items):
    gpu_items = [it for it in items if "gpu" in it.keywords]
    if not gpu_items:
        return
    n, why = _gpu_status()
    if n > 0:
        return
    if _gpu_selected(config):
        # `-m gpu` on a box without a usable device or library is a failure, not a skip
        config._spin_no_gpu_reason = why or "no device"
        return
    skip = pytest.mark.skip(reason=f"no CUDA device ({why})")
    for it in gpu_items:
        it.add_marker(skip)


def pytest_runtest_setup(item):
    why = getattr(item.config, "_spin_no_gpu_reason", None)
    if why is not None and "gpu" in item.keywords:
        pytest.fail(f"-m gpu selected but no usable GPU: {why}", pytrace=False)
