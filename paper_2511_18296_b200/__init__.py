"""B200-native move-evaluation engine for open-pit scheduling (arxiv 2511.18296).

Drop-in for the reference evaluator path (`pitplan.evaluate.evaluate_candidates_parallel`
and its feasibility / repair helpers), running hand-written sm_100a kernels through a
C ABI (include/pitplan_b200.h).  See DESIGN.md.
"""

from .errors import DeviceError, ExtensionMissing, InvalidArgs, PitplanError, ShapeMismatch, ValidationError
from .model import UNMINED, BlockModel, CandidateMove, ScenarioTables, Schedule, ViolationReport

__all__ = [
    "UNMINED",
    "BlockModel",
    "CandidateMove",
    "DeviceError",
    "ExtensionMissing",
    "InvalidArgs",
    "PitplanError",
    "ScenarioTables",
    "Schedule",
    "ShapeMismatch",
    "ValidationError",
    "ViolationReport",
    "Engine",
    "evaluate_candidates_parallel",
    "check_feasible",
    "install",
]


def __getattr__(name):  # lazy: importing the package must not require the built library
    if name == "Engine":
        from .engine import Engine

        return Engine
    if name in ("evaluate_candidates_parallel", "check_feasible"):
        from . import evaluate

        return getattr(evaluate, name)
    if name == "install":
        from .install import install

        return install
    raise AttributeError(name)
