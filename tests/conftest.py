import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2403_16526_b200", "libmdg.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2403_16526_b200", "csrc"),
                        "-j8", "-s"], check=True)
    mdo = os.path.join(ROOT, "oracle", "_build", "libmdo.so")
    if not os.path.exists(mdo):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def oracle():
    import pyoracle

    return pyoracle.mdo()


@pytest.fixture(scope="session")
def ref():
    import pyoracle

    if not pyoracle.ref_available():
        pytest.skip("oracle/_ref (reference build) not available")
    return pyoracle.ref()


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    from paper_2403_16526_b200 import _capi

    assert _capi.lib().mdg_device_ok() == 1, "libmdg needs an sm_100a device"
    return torch.device("cuda:0")


@pytest.fixture
def deterministic(cuda):
    """libmdg's deterministic mode (mdg_set_deterministic) for one test."""
    from paper_2403_16526_b200 import ops

    prev = ops.set_deterministic(True)
    yield
    ops.set_deterministic(prev)
