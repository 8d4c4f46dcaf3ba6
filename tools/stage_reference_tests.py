"""Stage the reference's own test suite next to its pip install (baseline/_ref/pkg_tests/, git-ignored
like the install itself, shipped to the GPU box with the snapshot), so tests/test_reference_suite_gpu.py
can run it there with the device drop-ins installed.  Run here, where /root/reference exists;
__graft_entry__.build() calls it."""

from __future__ import annotations

import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
DST = os.path.join(ROOT, "baseline", "_ref", "pkg_tests")


def stage() -> bool:
    if not os.path.isdir(SRC) or not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "pitplan")):
        return False
    os.makedirs(DST, exist_ok=True)
    for name in os.listdir(SRC):
        if name.endswith(".py"):
            shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
    return True


if __name__ == "__main__":
    print("staged" if stage() else "nothing to stage", file=sys.stderr)
