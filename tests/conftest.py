import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle_port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def oracle_ref():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref/libminimod_ref.so not built (needs /root/reference)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def mm():
    import paper_2007_06048_b200 as mm
    return mm


def load_golden(name):
    import numpy as np
    return dict(np.load(GOLDEN / f"{name}.npz"))
