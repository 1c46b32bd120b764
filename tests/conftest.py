import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2510_03283_b200.refpath import ensure_macesim  # noqa: E402

ensure_macesim()  # the unmodified reference scheduler (baseline/_ref), importable as `macesim`


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libmace_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    for item in items:
        if item.fspath.basename.startswith("diag_"):
            item.add_marker(pytest.mark.skip)


@pytest.fixture(scope="session")
def ctx():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected without a CUDA device")
    from paper_2510_03283_b200.build import build
    from paper_2510_03283_b200._lib import Ctx

    build()
    return Ctx(0)
