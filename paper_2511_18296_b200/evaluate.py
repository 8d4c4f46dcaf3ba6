"""Drop-in replacements for the reference evaluator entry points.

    evaluate_candidates_parallel   pitplan/evaluate.py:306-430
    check_feasible                 pitplan/evaluate.py:82-105
    precedence_repair_pass         pitplan/hybrid.py:493-510  (`_precedence_repair_pass`)
    unmine_fixpoint                pitplan/hybrid.py:199-211  (first step of `lns_repair`)
    ScheduleEvaluator              pitplan/evaluate.py:126-258 (npv_relaxed / per_scenario_npv /
                                   objective on the device for the single-mode fast path)
    lns_repair                     pitplan/hybrid.py:169-274  (destroy step and every insertion
                                   evaluation on the device; candidate ranking by the
                                   reference's own neighbour-similarity helper)

Same signatures, argument meaning, return types and error behaviour as the
reference; the work runs in the sm_100a kernels of csrc/pitplan_b200.cu through the
C ABI.  Objects are duck-typed: a `pitplan` Instance / ScenarioSet /
UncertaintyFactors / Schedule, or this package's own `BlockModel` with a
`ScenarioTables` (then `scenarios` carries both vmax and sigma and `sigma` is only
a switch).  When `pitplan` is importable the reference's own `CandidateMove` and
`ViolationReport` classes are returned.
"""

from __future__ import annotations

import csv
import threading
from collections import OrderedDict

import numpy as np

from .engine import DEFAULT_PSI_WEIGHTS, Engine
from .errors import InvalidArgs
from .model import BlockModel, CandidateMove, ScenarioTables, ViolationReport

_MAX_CACHED = 4
_tls = threading.local()  # one engine cache per host thread (contexts are not thread-safe)


def _types():
    try:
        from pitplan.evaluate import CandidateMove as RefMove
        from pitplan.evaluate import ViolationReport as RefReport

        return RefMove, RefReport
    except Exception:  # noqa: BLE001
        return CandidateMove, ViolationReport


def _cache() -> OrderedDict:
    c = getattr(_tls, "engines", None)
    if c is None:
        c = _tls.engines = OrderedDict()
    return c


class _Entry:
    __slots__ = ("instance", "bm", "engine", "scen_key", "scen_refs", "params", "rook")

    def __init__(self, instance, bm, engine):
        self.instance = instance  # strong ref: keeps id(instance) from being reused
        self.bm = bm
        self.engine = engine
        self.scen_key = None
        self.scen_refs = None
        self.params = None
        self.rook = None


def _device() -> int:
    return int(getattr(_tls, "device", 0))


def set_device(device: int) -> None:
    """CUDA device used by the drop-in functions on this thread."""
    _tls.device = int(device)


def _entry(instance) -> _Entry:
    cache = _cache()
    key = id(instance)
    e = cache.get(key)
    if e is not None and e.instance is instance:
        cache.move_to_end(key)
        return e
    bm = instance if isinstance(instance, BlockModel) else BlockModel.from_instance(instance)
    eng = Engine(_device())
    eng.set_instance(bm)
    e = _Entry(instance, bm, eng)
    cache[key] = e
    while len(cache) > _MAX_CACHED:
        _, old = cache.popitem(last=False)
        old.engine.close()
    return e


def _psi_weights(params):
    if params is None:
        return DEFAULT_PSI_WEIGHTS
    return tuple(float(w) for w in params.psi_weights)


def _bind_scenarios(e: _Entry, scenarios, sigma, params):
    weights = _psi_weights(params)
    if e.params != weights:
        e.engine.set_geology(weights)
        e.params = weights
    if scenarios is None:
        return
    key = (id(scenarios), id(sigma))
    if e.scen_key == key and e.scen_refs is not None and e.scen_refs[0] is scenarios and e.scen_refs[1] is sigma:
        return
    if isinstance(scenarios, ScenarioTables):
        tables = scenarios
    else:
        tables = ScenarioTables.from_reference(e.bm, scenarios, sigma)
    e.engine.set_scenarios(tables)
    e.scen_key = key
    e.scen_refs = (scenarios, sigma)


def _assignment(schedule) -> np.ndarray:
    return np.asarray(getattr(schedule, "assignment", schedule))


def evaluate_candidates_parallel(
    instance,
    schedule,
    candidates,
    scenarios,
    s,
    sigma,
    worker_count: int = 1,
    literal_kernel_value: bool = False,
    net_mining_cost: bool = False,
    params=None,
    trace_path=None,
):
    """Best insertion period per candidate plus the overall best move.

    Reference: pitplan/evaluate.py:306-430.  Output is bit-identical to the reference
    for every candidate order; `worker_count` is validated and otherwise ignored (the
    result never depended on it).  Infeasible candidates come back with improvement -inf.
    """
    if worker_count < 1:
        raise InvalidArgs("worker_count must be >= 1")
    cand = np.fromiter((int(b) for b in candidates), dtype=np.int64)
    e = _entry(instance)
    B = e.bm.n_blocks
    if cand.size and (cand.min() < -B or cand.max() >= B):
        raise InvalidArgs("candidate block id out of range")
    cand = np.where(cand < 0, cand + B, cand)  # Python negative indexing, as assign[b] would
    _bind_scenarios(e, None if literal_kernel_value and scenarios is None else scenarios, sigma, params)
    eng = e.engine
    if s is not None and not (0 <= int(s) < max(eng.n_scenarios, 1)):
        raise InvalidArgs(f"scenario index {s} out of range")
    eng.set_schedule(_assignment(schedule))
    res = eng.eval_candidates(
        cand, None if s is None else int(s), net=net_mining_cost, literal=literal_kernel_value,
        use_sigma=sigma is not None, trace=trace_path is not None,
    )
    Move, _ = _types()
    bt = res["best_t"].tolist()
    bv = res["best_val"].tolist()
    fe = res["feasible"].tolist()
    moves = [Move(block=b, period=t, improvement=v, feasible=bool(f))
             for b, t, v, f in zip(cand.tolist(), bt, bv, fe)]
    best = None
    if res["best"] is not None:
        gb, gt, gv = res["best"]
        best = Move(block=gb, period=gt, improvement=gv, feasible=True)
    if trace_path:
        _write_trace(trace_path, cand, res["trace_feas"], res["trace_val"])
    return moves, best


def _write_trace(path, cand, feas, val):
    """Per-(candidate, period) CSV, rows sorted like `sorted(trace_rows)` (evaluate.py:423-428)."""
    C, T = val.shape if val.ndim == 2 else (0, 0)
    b = np.repeat(cand, T)
    t = np.tile(np.arange(T), C)
    f = feas.reshape(-1).astype(np.int64)
    v = val.reshape(-1)
    # tuples (b, t, feasible, value): duplicates of a candidate give identical rows
    order = np.lexsort((v, f, t, b))
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["candidate", "period", "feasible", "value"])
        for k in order.tolist():
            w.writerow([int(b[k]), int(t[k]), int(f[k]), repr(float(v[k]))])


def check_feasible(instance, schedule):
    """Precedence-pair count, capacity excess and violation (evaluate.py:82-105)."""
    e = _entry(instance)
    r = e.engine.check_feasible(_assignment(schedule)[None, :])
    _, Report = _types()
    return Report(precedence_violations=int(r["pred_count"][0]), capacity_excess=float(r["excess"][0]),
                  violation=float(r["violation"][0]))


def check_feasible_batch(instance, assignments):
    """check_feasible for a population [P][B]; returns the dict of arrays."""
    return _entry(instance).engine.check_feasible(assignments)


def precedence_repair_pass(instance, assign: np.ndarray) -> None:
    """In-place `_precedence_repair_pass` (hybrid.py:493-510) in topological waves."""
    e = _entry(instance)
    out, _ = e.engine.repair(np.asarray(assign)[None, :], mode="push")
    assign[...] = out[0]


def precedence_repair_batch(instance, assignments: np.ndarray) -> np.ndarray:
    out, _ = _entry(instance).engine.repair(assignments, mode="push")
    return out


def unmine_fixpoint(instance, assign: np.ndarray):
    """The unmine fixpoint opening `lns_repair` (hybrid.py:199-211), in place; returns the
    block ids it unmined (the additions to the repair pool)."""
    e = _entry(instance)
    out, u = e.engine.repair(np.asarray(assign)[None, :], mode="unmine", unmined=True)
    assign[...] = out[0]
    return np.nonzero(u[0])[0]


def lns_repair(
    instance,
    schedule,
    unassigned,
    scenarios,
    sigma,
    max_iters: int = 100,
    seed: int = 0,
    realism_threshold: float = 0.5,
    destroy_fraction: float = 0.0,
    candidate_width: int = 16,
    strict: bool = False,
    only_positive: bool = False,
    net_mining_cost: bool = False,
    params=None,
):
    """Destroy-and-reinsert repair (hybrid.py:169-274), same signature and result.

    Destroy (hybrid.py:199-235): the unmine fixpoint and the over-capacity ejection run on the
    device (pp_repair + pp_eject, bit-exact period masses).  Repair (238-263): the geological
    consistency of every block comes from the device (pp_get_spatial) instead of 50k Python
    calls; each insertion round evaluates its candidates with the device kernel; the ranking
    by scheduled-neighbour similarity and the realism fallback are the reference's own code.
    The reference's helpers are restated in model.py (rook_neighbor_map,
    scheduled_neighbor_similarity), so pitplan is not required."""
    from .errors import RepairStalled
    from .model import rook_neighbor_map, scheduled_neighbor_similarity

    e = _entry(instance)
    _bind_scenarios(e, scenarios, sigma, params)
    sched = schedule.copy()
    before = check_feasible(instance, sched)
    pool: set[int] = {int(b) for b in unassigned}
    grades = getattr(scenarios, "grades", None)
    if grades is None:
        raise InvalidArgs("lns_repair needs scenarios with grades[S][B] (mean grade ranking, hybrid.py:214)")
    mean_grade = np.asarray(grades).mean(axis=0)
    a, added = e.engine.lns_destroy(np.asarray(sched.assignment)[None, :], mean_grade, destroy_fraction)
    sched.assignment[...] = a[0]
    pool.update(int(b) for b in np.nonzero(added[0])[0])

    spatial = e.engine.spatial()
    rook = e.rook if e.rook is not None else rook_neighbor_map(e.bm)
    e.rook = rook
    iters = 0
    stalled = False
    while pool and iters < max_iters:
        sims = scheduled_neighbor_similarity(sched.assignment, pool, mean_grade, rook)
        ranked = sorted(pool, key=lambda b: (-sims[b], b))
        cand = ranked[:candidate_width]
        moves, best = evaluate_candidates_parallel(
            instance, sched, cand, scenarios, None, sigma,
            net_mining_cost=net_mining_cost, params=params,
        )
        if best is None or (only_positive and best.improvement <= 0.0):
            stalled = best is None
            break
        chosen = best
        if spatial[best.block] < realism_threshold:
            feasible = [m for m in moves if m.feasible]
            feasible.sort(key=lambda m: (-spatial[m.block], m.block))
            chosen = feasible[0]
        sched.assignment[chosen.block] = chosen.period
        pool.discard(chosen.block)
        iters += 1

    after = check_feasible(instance, sched)
    if after.violation > before.violation:
        return schedule.copy()
    if stalled and strict:
        raise RepairStalled("no feasible insertion for remaining blocks", schedule=sched)
    return sched


def _reference_evaluator():
    try:
        from pitplan.evaluate import ScheduleEvaluator as Ref

        return Ref
    except Exception:  # noqa: BLE001
        return None


class _DeviceNpv:
    """Device half of the ScheduleEvaluator drop-in: relaxed NPV and per-scenario NPV of a schedule
    (evaluate.py:222-258) through pp_npv_relaxed when the stage-2 fast path applies (one mode, one
    rock type, positive rate: evaluate.py:149-150)."""

    def _dev_init(self, instance, scenarios, sigma):
        self._dev_args = (instance, scenarios, sigma)

    def _dev_entry(self):
        instance, scenarios, sigma = self._dev_args
        e = _entry(instance)
        if not e.bm.single_mode_fast:
            return None
        _bind_scenarios(e, scenarios, sigma, None)
        return e

    def _dev_npv(self, schedule, per_scenario):
        e = self._dev_entry()
        if e is None:
            return None
        r = e.engine.npv_relaxed(_assignment(schedule)[None, :], use_sigma=self._dev_args[2] is not None,
                                 per_scenario=per_scenario)
        return (float(r[0][0]), r[1][0]) if per_scenario else float(r[0])


def _make_evaluator_class():
    Ref = _reference_evaluator()
    base = (Ref, _DeviceNpv) if Ref is not None else (_DeviceNpv,)

    class ScheduleEvaluator(*base):
        """Drop-in for pitplan.evaluate.ScheduleEvaluator (evaluate.py:126-258): npv_relaxed,
        per_scenario_npv and objective run on the device (bit-exact) on the single-mode fast path;
        everything else (and the LP path) is the reference's own code when it is installed."""

        def __init__(self, instance, scenarios, sigma=None):
            if Ref is not None:
                Ref.__init__(self, instance, scenarios, sigma)
            self._dev_init(instance, scenarios, sigma)

        def npv_relaxed(self, schedule):
            v = self._dev_npv(schedule, False)
            if v is None:
                if Ref is None:
                    raise InvalidArgs("only the single-mode stage-2 fast path exists without the reference")
                return Ref.npv_relaxed(self, schedule)
            return v

        def per_scenario_npv(self, schedule):
            r = self._dev_npv(schedule, True)
            if r is None:
                if Ref is None:
                    raise InvalidArgs("only the single-mode stage-2 fast path exists without the reference")
                return Ref.per_scenario_npv(self, schedule)
            return r[1]

        def objective(self, schedule):
            """f(x) for a feasible schedule (evaluate.py:236-243)."""
            report = check_feasible(self._dev_args[0], schedule)
            if not report.feasible:
                try:
                    from pitplan.errors import InfeasibleSchedule
                except Exception:  # noqa: BLE001
                    InfeasibleSchedule = InvalidArgs  # noqa: N806
                raise InfeasibleSchedule(
                    f"schedule has violation {report.violation:.6g}; use the relaxed evaluator")
            return self.npv_relaxed(schedule)

    return ScheduleEvaluator


ScheduleEvaluator = _make_evaluator_class()


def clear_cache() -> None:
    cache = _cache()
    while cache:
        _, e = cache.popitem()
        e.engine.close()
