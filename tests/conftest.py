import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    config.addinivalue_line("markers", "ref: needs the reference library built into oracle/_ref")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libwsref.so not built (needs /root/reference)")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    from paper_2104_08265_b200 import Context
    c = Context(0)
    yield c
    c.close()
