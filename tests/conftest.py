import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libmfx.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def build_mfx():
    """Compile libmfx.so if it is missing or stale.  build.py is loaded by
    path: importing the package itself raises until the library exists."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_mfx_build", os.path.join(ROOT, "paper_2211_15605_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


@pytest.fixture(scope="session")
def mfx_built():
    return build_mfx()
