import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and libdpipe.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        # plain fp32 references must not silently run in TF32
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def _release_cuda_memory(request):
    """After each GPU test: drop the test's tensors and return the caching allocator's free blocks, so a
    long single-process `-m gpu` run (the full-size c2 / c3 / c5 trainers back to back) starts every test
    from an unfragmented pool instead of reaching cudaMalloc / cudaFree in the middle of a backward."""
    yield
    if "gpu" not in request.keywords:
        return
    import gc

    import torch

    if torch.cuda.is_available():
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
