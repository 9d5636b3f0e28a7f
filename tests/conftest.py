import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

REFERENCE_SRC = Path("/root/reference/pkg/src")
GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (runs on the B200 via gpurun)")
    config.addinivalue_line(
        "markers", "reference: needs the read-only reference in /root/reference")


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    cuda = has_cuda()
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_ref = pytest.mark.skip(reason="reference not mounted")
    for item in items:
        if "gpu" in item.keywords and not cuda:
            item.add_marker(skip_gpu)
        if "reference" in item.keywords and not REFERENCE_SRC.exists():
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def pc():
    """The package with its CUDA library loaded (GPU tests)."""
    import paper_2412_03898_b200 as pc
    from paper_2412_03898_b200 import _lib
    _lib.load_library()
    return pc


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def ref_pkg():
    """The live reference (build container only)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not mounted")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import pacloud
    return pacloud
