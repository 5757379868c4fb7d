import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def engine():
    import paper_2410_01799_b200 as sc

    return sc.Engine(0)


@pytest.fixture(scope="session")
def ref():
    """The reference compiled unchanged (oracle/_ref), else the C restatement."""
    from oracle.pyoracle import LIBS, Oracle

    return Oracle("ref") if os.path.exists(LIBS["ref"]) else Oracle("orc")


@pytest.fixture(scope="session")
def orc():
    from oracle.pyoracle import Oracle

    return Oracle("orc")
