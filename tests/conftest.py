import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    # GSC_AB_LIB: run the suite against another build of the same sources (e.g. the bounds-checked
    # debug library of tools/bounds_build.py)
    if os.environ.get("GSC_AB_LIB"):
        from paper_2502_14938_b200 import _abi
        _abi.SO_PATH = os.environ["GSC_AB_LIB"]
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def c1():
    import scenegen as sg
    cfg = sg.config("C1")
    return cfg, cfg.scene()
