"""pytest plugin for running the reference's own test suite with the device drop-ins installed:
install() runs in pytest_configure, i.e. before the suite's modules are collected, so their
`from pitplan.evaluate import ...` bindings (test_evaluate.py:8-15) already get the drop-ins.
At exit the path counters (device calls per entry point, calls handed to reference code) are
written to $PP_SUITE_COUNTERS.  Test infrastructure only (tests/test_reference_suite_gpu.py)."""

import json
import os


def pytest_configure(config):
    from paper_2511_18296_b200 import evaluate as ev
    from paper_2511_18296_b200.install import install

    config._pp_patched = install()
    ev.reset_path_counters()


def pytest_unconfigure(config):
    from paper_2511_18296_b200 import evaluate as ev

    out = os.environ.get("PP_SUITE_COUNTERS")
    if out:
        with open(out, "w") as fh:
            json.dump({"patched": getattr(config, "_pp_patched", []), **ev.path_counters()}, fh, indent=1)


def pytest_runtest_teardown(item):
    """With the checked library (PP_LIB=...checked.so): a guard-zone sweep after every test."""
    if "checked" not in os.environ.get("PP_LIB", ""):
        return
    import ctypes

    from paper_2511_18296_b200 import _lib

    if _lib._lib is None:
        return
    n = ctypes.c_int64(0)
    assert _lib._lib.pp_debug_check_guards(ctypes.byref(n)) == 0, _lib._lib.pp_last_error()
    assert n.value == 0, f"{n.value} device buffer guard zone(s) overwritten (see stderr)"
