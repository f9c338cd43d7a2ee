import os
import sys
from pathlib import Path

import hypothesis
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

# reference test profile (pkg/tests/conftest.py:1-8): reproducible examples
hypothesis.settings.register_profile("gridshift", deadline=None, derandomize=True, max_examples=60)
hypothesis.settings.load_profile("gridshift")

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgridshift_cuda.so")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def _cuda_visible() -> bool:
    if os.environ.get("GRIDSHIFT_FORCE_GPU_TESTS"):
        return True
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_visible():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def exact_sums():
    """Run the engine with order-independent exact sums (GS_SUMS_EXACT) --
    the tests that pin every device reduction against tests/exact_model.py."""
    import paper_2104_00303_b200 as gs

    with gs.sum_order("exact"):
        yield


@pytest.fixture
def reference_sums():
    """Run the engine with reference-order sums (GS_SUMS_REFERENCE): every
    iterate equals the reference's bit for bit -- the tests that assert
    bitwise trajectories."""
    import paper_2104_00303_b200 as gs

    with gs.sum_order("reference"):
        yield
