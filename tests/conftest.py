import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_AVAILABLE = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libwarpred_ref.so"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the reference built from /root/reference)")


@pytest.fixture(scope="session")
def orc():
    from oracle.bindings import Oracle, build

    build()
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    if not REF_AVAILABLE:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    from oracle.bindings import Ref

    return Ref()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    torch.cuda.set_device(0)
    return torch.device("cuda:0")
