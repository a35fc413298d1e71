import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True, scope="session")
def _generic_lane_kernel_by_default():
    """The suite builds lane decoders for dozens of ad-hoc codes; compiling a
    specialised kernel for each (NVRTC, about a minute per code) would only
    slow it down.  Tests run the generic kernel unless they ask for the
    specialised one (tests/test_gpu_specialised.py, tests/test_jit_source.py)."""
    import paper_1505_01466_b200 as pb
    prev = pb.set_default_options(specialize=-1)
    yield
    pb.set_default_options(**prev)
