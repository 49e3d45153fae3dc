import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session", autouse=True)
def _built_checkers():
    """The oracle (and oracle/_ref when /root/reference exists) are test infrastructure."""
    from oracle import oracle

    if not os.path.exists(oracle.ORACLE_SO) or (
            os.path.isdir("/root/reference/proj") and not os.path.exists(oracle.REF_SO)):
        oracle.build()


@pytest.fixture()
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device")
    return torch.device("cuda:0")
