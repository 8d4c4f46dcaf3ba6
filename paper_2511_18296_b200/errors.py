"""Exception tree of the evaluation engine.

Mirrors the reference's `pitplan.errors` (errors.py:4-110) for the classes the
hot path can raise.  When the reference package is importable the classes
subclass its own, so callers catching `pitplan.errors.InvalidArgs` (as the
GA/LNS loop and the reference tests do) also catch ours.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on whether pitplan is on sys.path
    from pitplan import errors as _ref_errors
except Exception:  # noqa: BLE001
    _ref_errors = None


def _base(name: str, fallback):
    if _ref_errors is not None and hasattr(_ref_errors, name):
        return getattr(_ref_errors, name)
    return fallback


class PitplanError(_base("PitplanError", Exception)):
    """Base class for all engine errors (errors.py:4)."""


class InvalidArgs(PitplanError, _base("InvalidArgs", Exception)):
    """Caller passed arguments outside an operation's preconditions (errors.py:16)."""


class ValidationError(PitplanError, _base("ValidationError", Exception)):
    """Data violates a documented invariant (errors.py:12)."""


class ShapeMismatch(PitplanError, _base("ShapeMismatch", Exception)):
    """Array dimensions disagree with the instance (errors.py:24)."""


class RepairStalled(PitplanError, _base("RepairStalled", Exception)):
    """No feasible insertion exists; carries the best-effort schedule (errors.py:52-57)."""

    def __init__(self, message, schedule=None):
        super().__init__(message)
        self.schedule = schedule


class DeviceError(PitplanError):
    """The sm_100a extension reported a CUDA failure (no CPU fallback exists)."""


class ExtensionMissing(PitplanError, ImportError):
    """The compiled sm_100a extension is not built or cannot be loaded."""


# status codes returned by every extern "C" entry point (include/pitplan_b200.h)
_STATUS = {
    1: InvalidArgs,
    2: ShapeMismatch,
    3: DeviceError,
    4: ValidationError,
    5: PitplanError,
}


def raise_for_status(code: int, message: str) -> None:
    if code == 0:
        return
    raise _STATUS.get(code, PitplanError)(message or f"pitplan_b200 status {code}")
