import os
import sys

import pytest

# One hardware work queue per CUDA stream: the one-GPU transport tests run P and D on
# separate streams of the same device, with spin-waits between them; with the default 8
# connections two streams can share a queue, and a wait at its head would block the other
# stream's work behind it (a false dependency).  Set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def pytest_sessionstart(session):
    """Build libkvx.so (sm_100a, in-tree) if it is missing or stale before any test module
    imports the binding -- a fresh checkout carries no built library (nvcc cross-compiles
    without a GPU; a no-op when the library is up to date)."""
    import __graft_entry__ as g
    g._lib_builder().build()


@pytest.fixture(scope="session")
def o1():
    from oracle import o1 as _o1
    _o1.lib()
    return _o1


@pytest.fixture(autouse=True, scope="module")
def _release_gpu_memory():
    """Return each module's cached device memory (GB-sized pools) before the next module --
    e.g. the bench contract test launches bench.py, which needs 71 GB of the same GPU."""
    yield
    import gc
    gc.collect()
    import torch
    if torch.cuda.is_available() and torch.cuda.is_initialized():
        torch.cuda.empty_cache()
