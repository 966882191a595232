import os
import pathlib
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; runs on the gpurun box")
    config.addinivalue_line("markers", "slow: longer CPU tests")


@pytest.fixture(scope="session")
def repo():
    return REPO


@pytest.fixture(scope="session")
def built():
    """Make sure the in-tree native artefacts exist (build is incremental)."""
    from paper_2508_01989_b200 import build
    if not (build.LIB / "taichi_sim").exists() or not (build.LIB / "libtaichi_b200.so").exists():
        build.build_all()
    return build.LIB


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cap = torch.cuda.get_device_capability(0)
    assert cap == (10, 0), f"expected a B200 (sm_100), got {cap}"
    return True
