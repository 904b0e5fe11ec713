import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def R():
    import oracle

    return oracle.Restatement()


@pytest.fixture(scope="session")
def REF():
    import oracle

    if not oracle.reference_available():
        pytest.skip("reference build (oracle/_ref) not present")
    return oracle.Reference()


@pytest.fixture(scope="session")
def eng():
    import paper_0912_2555_b200 as e

    e._abi.lib()
    return e


@pytest.fixture(scope="session")
def ctx(eng):
    return eng.default_context()
