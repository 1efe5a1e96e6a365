import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def _gpu_box():
    """A machine with an NVIDIA device node: GPU tests must run there, never skip."""
    import glob

    return bool(glob.glob("/dev/nvidia[0-9]*"))


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    if _gpu_box() and any("gpu" in it.keywords for it in items):
        # a B200 box whose CUDA context cannot be created (e.g. a device left faulted): fail
        # loudly instead of reporting skipped parity tests as a pass
        raise pytest.UsageError("GPU device nodes present but torch.cuda.is_available() is False")
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def dev():
    import paper_2201_00194_b200 as fs

    d = fs.Device(0)
    yield d
    d.close()


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.orc()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    return oracle.ref()
