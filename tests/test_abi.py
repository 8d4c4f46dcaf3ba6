"""The C-ABI library loads and exports every entry point include/pitplan_b200.h declares
(CPU test: no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2511_18296_b200 import _lib
from paper_2511_18296_b200.errors import DeviceError, InvalidArgs, PitplanError, raise_for_status

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "pitplan_b200.h")


def _declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^PP_API\s+[\w\s\*]*?\b(pp_\w+)\s*\(", src, flags=re.M)))


def test_header_lists_entry_points():
    names = _declared()
    assert "pp_eval_candidates" in names and "pp_check_feasible" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_abi_version_and_error_channel():
    lib = _lib.load()
    assert lib.pp_abi_version() == _lib.ABI_VERSION
    assert isinstance(lib.pp_last_error(), bytes)


def test_null_arguments_are_errors_not_crashes():
    lib = _lib.load()
    assert lib.pp_ctx_create(0, None) == 1
    assert b"NULL" in lib.pp_last_error()
    assert lib.pp_set_instance(None, 1, 1, 0, None, None, None, None, None, None) == 1


def test_status_mapping():
    with pytest.raises(InvalidArgs):
        raise_for_status(1, "x")
    with pytest.raises(DeviceError):
        raise_for_status(3, "x")
    with pytest.raises(PitplanError):
        raise_for_status(5, "x")


def test_no_gpu_context_creation_fails_loudly():
    lib = _lib.load()
    n = ctypes.c_int()
    rc = lib.pp_device_count(ctypes.byref(n))
    if rc == 0 and n.value > 0:
        pytest.skip("a GPU is present")
    from paper_2511_18296_b200.engine import Engine

    with pytest.raises(PitplanError):
        Engine(0)


def _struct_fields(name):
    src = open(HDR).read()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), src, flags=re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    return re.findall(r"\*?\s*(\w+);", body)


def test_header_abi_version_and_struct_layouts_match_ctypes():
    src = open(HDR).read()
    assert int(re.search(r"#define PP_ABI_VERSION (\d+)", src).group(1)) == _lib.ABI_VERSION
    for cname, py in (("pp_cand_out", _lib.PPCandOut), ("pp_move_out", _lib.PPMoveOut), ("pp_best", _lib.PPBest)):
        want = [f.rstrip("_") for f in _struct_fields(cname)]
        got = [f[0].rstrip("_") for f in py._fields_]
        assert want == got, (cname, want, got)


def test_install_rebinds_reference_names_on_cpu():
    """install.py rebinds every reference entry point (hybrid.py:22-28 binds by value) and
    uninstall restores them; `ScheduleEvaluator` becomes the evaluator factory and the
    reference's own objects stay reachable through install.original (the LP-instance path and
    polish_schedule's: no self-recursion after install).  No compute runs."""
    import os
    import sys

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "pitplan")):
        pytest.skip("baseline/_ref (pip install of the reference) absent")
    from paper_2511_18296_b200 import evaluate as ev
    from paper_2511_18296_b200.install import install, uninstall

    if ref not in sys.path:
        sys.path.append(ref)
    import pitplan.evaluate as PE
    import pitplan.hybrid as PH

    orig = (PH.evaluate_candidates_parallel, PH.polish_schedule, PE.ScheduleEvaluator)
    done = install()
    try:
        assert PH.evaluate_candidates_parallel is ev.evaluate_candidates_parallel
        assert PH.polish_schedule is ev.polish_schedule
        assert PH.ScheduleEvaluator is ev.evaluator_for and PE.ScheduleEvaluator is ev.evaluator_for
        assert "pitplan.hybrid.lns_repair" in done and "pitplan.colgen.price_column" in done
        from paper_2511_18296_b200.install import original

        assert original("pitplan.hybrid", "polish_schedule") is orig[1]
        assert ev._reference_fn("pitplan.hybrid", "polish_schedule") is orig[1]
        assert original("pitplan.evaluate", "ScheduleEvaluator") is orig[2]
    finally:
        uninstall()
    assert (PH.evaluate_candidates_parallel, PH.polish_schedule, PE.ScheduleEvaluator) == orig
