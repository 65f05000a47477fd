import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def ref_fast():
    from oracle.oracle import RefLib, ref_available
    if not ref_available(fast=True):
        pytest.skip("oracle/_ref fast build missing")
    return RefLib(fast=True)


@pytest.fixture(scope="session")
def ctx():
    import paper_1203_1269_b200.gpemu as g
    return g.Context(0, "dag")
