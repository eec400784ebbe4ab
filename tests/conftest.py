import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


@pytest.fixture(autouse=True)
def _release_gpu_memory(request):
    """After every GPU test, hand the caching allocator's free blocks back to the driver:
    the full-size config tests hold tens of GB, and the multi-process tests that follow
    start their own CUDA contexts on the same GPU."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    import gc

    import torch
    if torch.cuda.is_available() and torch.cuda.is_initialized():
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


@pytest.fixture(scope="session")
def tables():
    with open(os.path.join(GOLDEN, "tables.json")) as f:
        return json.load(f)


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    return {k: z[k] for k in z.files}


def golden_forward_cases():
    return sorted(f for f in os.listdir(GOLDEN) if f.startswith("fwd_") and f.endswith(".npz"))
