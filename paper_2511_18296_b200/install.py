"""Install the B200 engine behind the reference's own plug-in points.

The reference has no operator registry: the GA/LNS/SA and column-generation loops
reach the evaluator through module-level names, and `pitplan.hybrid` binds
`evaluate_candidates_parallel` / `check_feasible` by value at import
(hybrid.py:22-28), as does `pitplan.colgen` for `check_feasible` (colgen.py:23).
`install()` therefore rebinds the names in every module that holds them, so the
unchanged loops (`lns_repair` hybrid.py:252, `HybridSearch._measure` hybrid.py:600,
`_crossover` hybrid.py:721, DW integerisation colgen.py:573) run on the GPU.
"""

from __future__ import annotations

import importlib

from . import evaluate as _ev
from . import hybrid_batch as _hb


def _patches():
    E = _ev.evaluator_for  # device evaluator; the reference class for out-of-scope LP instances
    return {
        "pitplan.evaluate": {
            "evaluate_candidates_parallel": _ev.evaluate_candidates_parallel,
            "check_feasible": _ev.check_feasible,
            "ScheduleEvaluator": E,
        },
        "pitplan.hybrid": {
            "evaluate_candidates_parallel": _ev.evaluate_candidates_parallel,
            "check_feasible": _ev.check_feasible,
            "_precedence_repair_pass": _ev.precedence_repair_pass,
            "lns_repair": _ev.lns_repair,
            "ScheduleEvaluator": E,
            "polish_schedule": _ev.polish_schedule,
        },
        "pitplan.colgen": {"check_feasible": _ev.check_feasible, "lns_repair": _ev.lns_repair,
                           "ScheduleEvaluator": E, "price_column": _ev.price_column},
        "pitplan.saa": {},
        "pitplan": {"check_feasible": _ev.check_feasible},
        # the GA generation of the unchanged HybridSearch class: batched fitness, native mutation
        "pitplan.hybrid:HybridSearch": {"_member": _hb.member, "_measure": _hb.measure, "_mutate": _hb.mutate},
    }


_saved: list[tuple[object, str, object]] = []
_originals: dict[tuple[str, str], object] = {}


def original(module: str, name: str):
    """The reference's own `module.name` as it was before the first install(), or None."""
    return _originals.get((module, name))


def original_attr(target: str, name: str):
    """The reference's own attribute `name` of `module:Class` / `module.Class` before install()."""
    key = target.replace(":", ".") if ":" in target else target
    fn = _originals.get((key, name)) or _originals.get((target, name))
    if fn is None:  # never installed: the class's current attribute is the reference's
        mod, _, cls = (target.replace(":", ".")).rpartition(".")
        fn = getattr(getattr(importlib.import_module(mod), cls), name)
    return fn


def _resolve(target: str):
    if ":" in target:
        mod, cls = target.split(":", 1)
        return getattr(importlib.import_module(mod), cls)
    return importlib.import_module(target)


def install() -> list[str]:
    """Rebind the reference entry points; returns the patched 'module.name' list."""
    done = []
    for modname, names in _patches().items():
        try:
            mod = _resolve(modname)
        except (ImportError, AttributeError):
            continue
        for name, fn in names.items():
            if hasattr(mod, name):
                cur = getattr(mod, name)
                _saved.append((mod, name, cur))
                _originals.setdefault((modname.replace(":", "."), name), cur)
                setattr(mod, name, fn)
                done.append(f"{modname.replace(':', '.')}.{name}")
    return done


def uninstall() -> None:
    while _saved:
        mod, name, orig = _saved.pop()
        setattr(mod, name, orig)
