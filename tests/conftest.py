import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: builds 50k+ block instances")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle

    oracle.build()
    return oracle


@pytest.fixture(autouse=True)
def _checked_build_guards():
    """With the checked library (PP_LIB=...checked.so) every test ends with a guard-zone sweep of
    the live device buffers; overwritten guards found there or at any free fail the test."""
    yield
    if "checked" not in os.environ.get("PP_LIB", ""):
        return
    from paper_2511_18296_b200 import _lib

    if _lib._lib is None:
        return
    import ctypes

    n = ctypes.c_int64(0)
    assert _lib._lib.pp_debug_check_guards(ctypes.byref(n)) == 0, _lib._lib.pp_last_error()
    assert n.value == 0, f"{n.value} device buffer guard zone(s) overwritten (see stderr)"
