"""The reference's own hot-path tests, run unchanged with the device drop-ins installed
(test_evaluate.py, test_hybrid.py, test_acceptance.py::TestKernelDeterminism and
::TestDeterminismCriterion incl. pause/resume byte identity, plus the column-generation and SAA
suites that reach the evaluator).  The suite is staged from /root/reference by
tools/stage_reference_tests.py into baseline/_ref/pkg_tests (git-ignored, shipped with the
snapshot); the test skips when it is absent.  Must pass, and the engine must have done the work:
the device counters are asserted; reference calls may come only from multi-mode LP instances."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "pkg_tests")

TARGETS = [
    "test_evaluate.py",
    "test_hybrid.py",
    "test_acceptance.py::TestKernelDeterminism",
    "test_acceptance.py::TestDeterminismCriterion",
    "test_acceptance.py::TestOracleOptimality",
    "test_acceptance.py::TestMonotoneTraces",
    "test_colgen.py",
    "test_saa.py",
]


def test_reference_suite_with_dropins_installed(tmp_path):
    if not os.path.isfile(os.path.join(SUITE, "test_evaluate.py")):
        pytest.skip("reference suite not staged (tools/stage_reference_tests.py)")
    counters = tmp_path / "counters.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, REF, env.get("PYTHONPATH", "")])
    env["PP_SUITE_COUNTERS"] = str(counters)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ref_suite_plugin", "-p", "no:cacheprovider",
           "--rootdir", SUITE, *[os.path.join(SUITE, t) for t in TARGETS]]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=3000)
    log = os.path.join(ROOT, "gpurun_out", "reference_suite.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    with open(log, "w") as fh:
        fh.write(r.stdout + "\n---- stderr ----\n" + r.stderr)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    c = json.load(open(counters))
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite_counters.json"), "w") as fh:
        json.dump(c, fh, indent=1)
    assert "pitplan.hybrid.evaluate_candidates_parallel" in c["patched"]
    dev = c["device"]
    for name in ("pp_eval_candidates", "pp_check_feasible", "pp_npv_relaxed", "pp_repair"):
        assert dev.get(name, 0) > 0, (name, c)
    assert set(c["reference"]) <= {"ScheduleEvaluator", "polish_schedule"}, c
