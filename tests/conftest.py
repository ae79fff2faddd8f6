import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import REF_CHECK_SO, Oracle
    if not REF_CHECK_SO.exists():
        pytest.skip("oracle/_ref not built (reference sources absent on this host)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def fsk():
    import paper_2602_03067_b200 as fsk
    fsk.lib()
    return fsk
