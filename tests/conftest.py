import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session")
def cuda_available():
    import torch
    return torch.cuda.is_available()


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(autouse=True)
def _debug_library_record(request):
    """Under the DI_DEBUG library (DI_LIB=.../libdeepinverse_exp.so built with -DDI_DEBUG): after every GPU test, the
    host-mapped failure record of the bounded mbarrier waits / device asserts must be clean."""
    yield
    if "gpu" not in request.keywords or not os.environ.get("DI_LIB"):
        return
    import ctypes
    from paper_1701_03891_b200 import binding
    lib = binding.load()
    if not hasattr(lib, "di_debug_report"):
        return
    buf = ctypes.create_string_buffer(256)
    code = lib.di_debug_report(buf, 256)
    assert code in (0, -1), buf.value.decode()
