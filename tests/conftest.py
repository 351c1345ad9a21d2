import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and libqadc_b200.so")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def golden(name):
    return np.load(GOLDEN / name)


def cases(npz, prefix="c"):
    """Yield dicts of per-case arrays from a golden npz (keys c{i}_{field})."""
    n = int(npz["n"])
    for i in range(n):
        pre = f"{prefix}{i}_"
        yield {k[len(pre):]: npz[k] for k in npz.files if k.startswith(pre)}


@pytest.fixture(scope="session")
def gpu():
    """Skip-free guard for -m gpu tests: fail loudly if the B200 path is
    unavailable (no silent CPU fallback)."""
    import torch

    from paper_1704_07355_b200 import _native
    if not _native.library_available():
        pytest.fail("libqadc_b200.so is not built")
    _native.require_device()
    torch.cuda.set_device(0)
    return True
