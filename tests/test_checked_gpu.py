"""The checked build (libpitplan_b200_checked.so, -DPP_CHECKED) is the memory-safety stand-in for
compute-sanitizer on this GPU pool: guard zones around every device buffer.  Negative control: a
one-byte store past the end of a buffer must be reported by pp_debug_check_guards (run in a child
process, whose guard counter is its own).  The full suite under the checked library is
tools/run_checked.sh."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2511_18296_b200", "libpitplan_b200_checked.so")

CHILD = r"""
import ctypes, numpy as np
from paper_2511_18296_b200 import _lib
from paper_2511_18296_b200.engine import Engine
from paper_2511_18296_b200.model import ScenarioTables
from tests._fixtures import config
c = config("C1")
eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["greedy"])
eng.get_schedule()  # period masses allocated and computed
lib = _lib.load()
n = ctypes.c_int64(-1)
assert lib.pp_debug_check_guards(ctypes.byref(n)) == 0 and n.value == 0, n.value
h = ctypes.CDLL(_lib.LIB_PATH)
h.pp_debug_corrupt_guard.argtypes = [ctypes.c_void_p]
assert h.pp_debug_corrupt_guard(eng._h) == 0
assert lib.pp_debug_check_guards(ctypes.byref(n)) == 0 and n.value == 1, n.value
print("GUARD-CONTROL-OK", _lib.LIB_PATH)
"""


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked library not built (build_checked())")
def test_guard_zone_catches_an_out_of_bounds_store():
    env = dict(os.environ, PP_LIB=CHECKED, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GUARD-CONTROL-OK" in r.stdout and "checked" in r.stdout
    assert "guard of a" in r.stderr  # the report names the overwritten buffer


def test_release_build_has_no_guard_check():
    import ctypes

    from paper_2511_18296_b200 import _lib

    if "checked" in os.environ.get("PP_LIB", ""):
        pytest.skip("running against the checked library")
    n = ctypes.c_int64(0)
    assert _lib.load().pp_debug_check_guards(ctypes.byref(n)) != 0
