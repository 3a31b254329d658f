import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def restatement():
    from oracle.oracle import Restatement, build
    build(reference=os.path.isdir("/root/reference/proj"))
    return Restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import REFERENCE_SO, Reference, build
    if not os.path.exists(REFERENCE_SO):
        if os.path.isdir("/root/reference/proj"):
            build(reference=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return Reference()


@pytest.fixture(scope="session")
def cuda_ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_14856_b200.api import Context
    return Context(0)
