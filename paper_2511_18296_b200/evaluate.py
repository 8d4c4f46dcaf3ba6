"""Drop-in replacements for the reference evaluator entry points.

    evaluate_candidates_parallel   pitplan/evaluate.py:306-430
    check_feasible                 pitplan/evaluate.py:82-105
    precedence_repair_pass         pitplan/hybrid.py:493-510  (`_precedence_repair_pass`)
    unmine_fixpoint                pitplan/hybrid.py:199-211  (first step of `lns_repair`)
    ScheduleEvaluator              pitplan/evaluate.py:126-258 (npv_relaxed / per_scenario_npv /
                                   objective on the device for the single-mode fast path)
    polish_schedule                pitplan/hybrid.py:326-490  (every option of a block evaluated in one
                                   batched device call)
    lns_repair                     pitplan/hybrid.py:169-274  (destroy step and every insertion
                                   evaluation on the device; candidate ranking by the
                                   reference's own neighbour-similarity helper)
    price_column                   pitplan/colgen.py:207-293  (the sequence greedy on the device)

Same signatures, argument meaning, return types and error behaviour as the
reference; the work runs in the sm_100a kernels of csrc/ through the C ABI, and no
function here executes reference code: `pitplan` is imported only for its record types
(CandidateMove, ViolationReport, SequenceColumn) and exception classes.  Objects are
duck-typed: a `pitplan` Instance / ScenarioSet / UncertaintyFactors / Schedule, or this
package's own `BlockModel` with a `ScenarioTables` (then `scenarios` carries both vmax
and sigma and `sigma` is only a switch).

One explicit exception, counted in REFERENCE_CALLS and logged: the multi-mode / multi-rock
stage-2 LP (evaluate.py:185-220) is out of scope, so for such an instance the
installed `ScheduleEvaluator` factory returns the reference's own evaluator class and
`polish_schedule` runs the reference's own function (captured by install() before it
rebinds the name).  Single-mode instances never reach the reference.
"""

from __future__ import annotations

import collections
import csv
import logging
import os
import threading
from collections import OrderedDict

import numpy as np

from .engine import DEFAULT_PSI_WEIGHTS, Engine
from .errors import InvalidArgs, ShapeMismatch
from .model import BlockModel, CandidateMove, ScenarioTables, ViolationReport

_MAX_CACHED = 4
_POLISH_CHUNK = int(os.environ.get('PP_POLISH_CHUNK', '64'))  # first speculative chunk (blocks)
_POLISH_CHUNK_MAX = 128
_tls = threading.local()  # one engine cache per host thread (contexts are not thread-safe)
_log = logging.getLogger(__name__)

# Calls routed to the reference's own code (only the out-of-scope multi-mode LP path).
REFERENCE_CALLS: collections.Counter = collections.Counter()


def path_counters() -> dict:
    """{"device": calls per C-ABI compute entry point, "reference": calls handed to reference code}."""
    from . import _lib

    return {"device": _lib.device_calls(), "reference": dict(REFERENCE_CALLS)}


def reset_path_counters() -> None:
    from . import _lib

    _lib.reset_device_calls()
    REFERENCE_CALLS.clear()


def _reference_fn(module: str, name: str):
    """The reference's own function `module.name` as it was before install() rebound it."""
    from . import install as _inst

    fn = _inst.original(module, name)
    if fn is None:
        import importlib

        fn = getattr(importlib.import_module(module), name)
    return fn


def _to_reference(what: str) -> None:
    REFERENCE_CALLS[what] += 1
    if REFERENCE_CALLS[what] == 1:
        _log.warning("%s: multi-mode / multi-rock stage-2 LP instance -- the reference's own code runs "
                     "(out of scope for the device engine)", what)


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
    __slots__ = ("instance", "bm", "engine", "scen_key", "scen_refs", "params", "rook", "rook_pad", "rook_on_device")

    def __init__(self, instance, bm, engine):
        self.instance = instance  # strong ref: keeps id(instance) from being reused
        self.bm = bm
        self.engine = engine
        self.scen_key = None
        self.scen_refs = None
        self.params = None
        self.rook = None
        self.rook_pad = None
        self.rook_on_device = False


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


def _bind_sigma_only(e: _Entry, sigma, params):
    """literal_kernel_value=True with scenarios=None: unit = mass * 100 needs no value table, but the
    sigma row does (evaluate.py:348-353): bind sigma[S][T] with an all-zero value table."""
    weights = _psi_weights(params)
    if e.params != weights:
        e.engine.set_geology(weights)
        e.params = weights
    if sigma is None:
        return
    key = (None, id(sigma))
    if e.scen_key == key and e.scen_refs is not None and e.scen_refs[1] is sigma:
        return
    sig = np.asarray(getattr(sigma, "sigma", sigma), dtype=np.float64)
    e.engine.set_scenarios(ScenarioTables(vmax=np.zeros((sig.shape[0], e.bm.n_blocks)), sigma=sig))
    e.scen_key = key
    e.scen_refs = (None, sigma)


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
    if cand.size and (cand.min() < 0 or cand.max() >= B):
        # the reference would index assign[b] Python-style for -B <= b < 0 and report the negative
        # id; the engine takes block ids in [0, B) only (documented difference)
        raise InvalidArgs("candidate block id out of range [0, n_blocks)")
    if literal_kernel_value and scenarios is None:
        _bind_sigma_only(e, sigma, params)
    else:
        _bind_scenarios(e, scenarios, sigma, params)
    eng = e.engine
    if s is not None:
        n_s = max(eng.n_scenarios, 1)
        if not (-n_s <= int(s) < n_s):
            raise InvalidArgs(f"scenario index {s} out of range")
        s = int(s) % n_s  # v[s] / sigma[s] with Python indexing (evaluate.py:302, 353)
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


_LNS_GRAPH_WMAX = 64  # pp_lns_insert's candidate_width limit


def _rook_csr(pad: np.ndarray):
    """model.rook_padded's [B][L] table (-1 padding, reference order) as a CSR."""
    valid = pad >= 0
    ptr_ = np.zeros(pad.shape[0] + 1, dtype=np.int32)
    np.cumsum(valid.sum(axis=1), out=ptr_[1:])
    return ptr_, pad[valid].astype(np.int32)


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
    calls; each insertion round evaluates its candidates with the device kernel, which also
    selects both keys -- the best move and the realism fallback's (k_realism); the ranking by
    scheduled-neighbour similarity is vectorised on the host.
    The reference's helpers are restated in model.py (rook_neighbor_map,
    scheduled_neighbor_similarity), so pitplan is not required."""
    from .errors import RepairStalled
    from .model import neighbor_similarity_array, rook_neighbor_map, rook_padded, scheduled_neighbor_similarity

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
    pad = e.rook_pad
    if pad is None:
        pad = e.rook_pad = rook_padded(rook, e.bm.n_blocks)
    in_pool = np.zeros(e.bm.n_blocks, dtype=bool)
    in_pool[list(pool)] = True
    iters = 0
    stalled = False
    if pad is not None and 1 <= candidate_width <= _LNS_GRAPH_WMAX and pool and max_iters > 0:
        # the whole insertion loop as one device-resident CUDA graph (pp_lns_insert): ranking,
        # evaluation, both selection keys, the decision and the update on the device per round
        if not e.rook_on_device:
            e.engine.set_rook(*_rook_csr(pad))
            e.rook_on_device = True
        a, in_pool, iters, stalled = e.engine.lns_insert(
            sched.assignment, in_pool, mean_grade, max_iters=max_iters, candidate_width=candidate_width,
            realism_threshold=realism_threshold, only_positive=only_positive, net=net_mining_cost,
            use_sigma=sigma is not None)
        sched.assignment[...] = a
        pool = set()  # (consumed)
    while pool and iters < max_iters:
        if pad is not None:  # vectorised ranking, identical order (model.neighbor_similarity_array)
            ids = np.flatnonzero(in_pool)
            sims = neighbor_similarity_array(sched.assignment, ids, mean_grade, pad)
            cand = ids[np.lexsort((ids, -sims))[:candidate_width]].tolist()
        else:
            sims = scheduled_neighbor_similarity(sched.assignment, pool, mean_grade, rook)
            ranked = sorted(pool, key=lambda b: (-sims[b], b))
            cand = ranked[:candidate_width]
        e.engine.set_schedule(sched.assignment)
        res = e.engine.eval_candidates(np.asarray(cand, dtype=np.int32), None, net=net_mining_cost,
                                       use_sigma=sigma is not None, realism=True)
        best = res["best"]  # (block, period, improvement) in evaluate.py:404-421 order
        if best is None or (only_positive and best[2] <= 0.0):
            stalled = best is None
            break
        chosen = best
        if spatial[best[0]] < realism_threshold:
            # the realism fallback (hybrid.py:256-263): the feasible candidate of highest
            # geological consistency, lowest block on ties -- selected on the device
            chosen = res["realism"]
        sched.assignment[chosen[0]] = chosen[1]
        pool.discard(chosen[0])
        in_pool[chosen[0]] = False
        iters += 1

    after = check_feasible(instance, sched)
    if after.violation > before.violation:
        return schedule.copy()
    if stalled and strict:
        raise RepairStalled("no feasible insertion for remaining blocks", schedule=sched)
    return sched


class _Stage2Count:
    """Stands in for the reference's `_stage2_cache` dict (evaluate.py:147), whose only outside use
    is `len()` in the run's timing.json (runstore.py:453): the number of stage-2 problems the
    device solved for this evaluator (no cache: re-solves are counted again)."""

    __slots__ = ("n",)

    def __init__(self):
        self.n = 0

    def __len__(self):
        return self.n


class ScheduleEvaluator:
    """Drop-in for pitplan.evaluate.ScheduleEvaluator (evaluate.py:126-258): npv_relaxed,
    per_scenario_npv and objective on the device (k_stage2 / k_stage2_big + k_npv_final),
    bit-exact, for instances on the stage-2 fast path (one mode, one rock type, positive rate,
    evaluate.py:149-150).  The multi-mode LP instances are refused here (InvalidArgs); the
    installed factory `evaluator_for` gives them the reference's own class.

    The attributes callers read (`values`, `masses`, `costs`, `discount` -- hybrid.py:673-678,
    saa.py:60-65 -- and len(`_stage2_cache`), runstore.py:453) are provided; `values` is built on
    first use, not at construction."""

    def __init__(self, instance, scenarios, sigma=None):
        n_b = getattr(scenarios, "n_blocks", None)
        if n_b is None and getattr(scenarios, "vmax", None) is not None:
            n_b = np.asarray(scenarios.vmax).shape[1]
        e = _entry(instance)
        if n_b is not None and int(n_b) != e.bm.n_blocks:
            raise InvalidArgs("scenario set does not match instance block count")
        if not e.bm.single_mode_fast:
            raise InvalidArgs("the device evaluator covers the single-mode stage-2 fast path only "
                              "(evaluate.py:149-150); use the reference evaluator for the LP path")
        self.instance = instance
        self.scenarios = scenarios
        self.sigma = sigma
        self._values = None
        self._stage2_cache = _Stage2Count()

    # -- the reference's attributes ------------------------------------------------------
    @property
    def masses(self) -> np.ndarray:
        return _entry(self.instance).bm.mass

    @property
    def costs(self) -> np.ndarray:
        return _entry(self.instance).bm.cost

    @property
    def discount(self) -> np.ndarray:
        return _entry(self.instance).bm.discount()

    @property
    def values(self) -> np.ndarray:
        """v[s][b][o] (scenario_mode_values, evaluate.py:108-124); single mode: o = 0."""
        if self._values is None:
            e = self._entry()
            self._values = e.engine.scenario_table()[:, :, None]
        return self._values

    def sigma_st(self, s: int, t: int) -> float:
        return 1.0 if self.sigma is None else float(np.asarray(getattr(self.sigma, "sigma", self.sigma))[s, t])

    def stage2_raw(self, s: int, t: int, blocks) -> float:
        """Unadjusted optimal processing value of the mined set (evaluate.py:153-164, sigma = 1),
        solved on the device (pp_stage2)."""
        blocks = tuple(int(b) for b in blocks)
        if not blocks:
            return 0.0
        e = self._entry()
        a = np.full(e.bm.n_blocks, -1, dtype=np.int32)
        a[list(blocks)] = t
        raw, _ = e.engine.stage2(a[None, :])
        self._stage2_cache.n += e.engine.n_scenarios
        return float(raw[0, t, s])

    _solve_stage2 = stage2_raw

    # -- device --------------------------------------------------------------------------
    def _entry(self) -> _Entry:
        e = _entry(self.instance)
        _bind_scenarios(e, self.scenarios, self.sigma, None)
        return e

    def _npv(self, schedules, per_scenario):
        e = self._entry()
        a = _assignment(schedules)
        r = e.engine.npv_relaxed(a if a.ndim == 2 else a[None, :], use_sigma=self.sigma is not None,
                                 per_scenario=per_scenario)
        self._stage2_cache.n += e.engine.n_scenarios * e.bm.n_periods * (a.shape[0] if a.ndim == 2 else 1)
        return r

    def npv_relaxed(self, schedule) -> float:
        """Stage-1 + stage-2 value evaluated as-is, violations ignored (evaluate.py:244-246)."""
        return float(self._npv(schedule, False)[0])

    def npv_relaxed_batch(self, assignments) -> np.ndarray:
        """npv_relaxed of a population [P][B] in one device call."""
        return self._npv(np.atleast_2d(np.asarray(assignments)), False)

    def per_scenario_npv(self, schedule) -> np.ndarray:
        """evaluate.py:248-258."""
        return self._npv(schedule, True)[1][0]

    def objective(self, schedule) -> float:
        """f(x) for a feasible schedule (evaluate.py:236-243)."""
        report = check_feasible(self.instance, schedule)
        if not report.feasible:
            try:
                from pitplan.errors import InfeasibleSchedule
            except Exception:  # noqa: BLE001
                InfeasibleSchedule = InvalidArgs  # noqa: N806
            raise InfeasibleSchedule(
                f"schedule has violation {report.violation:.6g}; use the relaxed evaluator")
        return self.npv_relaxed(schedule)


def evaluator_for(instance, scenarios, sigma=None):
    """What install() binds as `ScheduleEvaluator`: the device evaluator for fast-path instances;
    for a multi-mode LP instance (out of scope) the reference's own class, counted and logged."""
    if _entry(instance).bm.single_mode_fast:
        return ScheduleEvaluator(instance, scenarios, sigma)
    _to_reference("ScheduleEvaluator")
    return _reference_fn("pitplan.evaluate", "ScheduleEvaluator")(instance, scenarios, sigma)


def polish_schedule(instance, evaluator, schedule, max_sweeps: int = 5, pair_swaps=None):
    """Steepest-descent polish (hybrid.py:326-490), same result as the reference.

    The single-block sweep evaluates all options of a block (other period, unmine) in one
    pp_npv_moves call, which re-solves only the two periods each option changes (bit-exact relaxed
    NPV, so the `> best + 1e-9` decisions are the reference's); the small-instance swap / exchange /
    joint-insertion phases call the device evaluator per candidate, in the reference's order.
    Any evaluator object is accepted (its instance, scenarios and sigma are what count); a
    multi-mode LP instance -- out of scope -- runs the reference's own polish_schedule (counted,
    logged)."""
    e = _entry(instance)
    bm = e.bm
    if not bm.single_mode_fast:
        _to_reference("polish_schedule")
        return _reference_fn("pitplan.hybrid", "polish_schedule")(instance, evaluator, schedule, max_sweeps,
                                                                  pair_swaps)
    _bind_scenarios(e, evaluator.scenarios, evaluator.sigma, None)
    eng = e.engine
    use_sigma = evaluator.sigma is not None
    UN = -1
    masses = bm.mass
    cap = bm.capacity
    B, T = bm.n_blocks, bm.n_periods
    pp_, pi_, sp_, si_ = bm.csr()
    if pair_swaps is None:
        pair_swaps = B <= 32
    cur = schedule.copy()
    a = cur.assignment

    def npv_of(batch):
        return eng.npv_relaxed(np.asarray(batch), use_sigma=use_sigma)

    cur_val = float(npv_of(a[None, :])[0])
    load = np.zeros(T)
    for t in range(T):
        load[t] = masses[a == t].sum()

    def window(b):
        preds = pi_[pp_[b]:pp_[b + 1]]
        if np.any(a[preds] == UN):
            t_lo = None
        else:
            t_lo = int(max(a[preds].max(), 0)) if preds.size else 0
        ms_ = a[si_[sp_[b]:sp_[b + 1]]]
        ms_ = ms_[ms_ != UN]
        t_hi = int(ms_.min()) if ms_.size else T - 1
        return t_lo, t_hi

    for _ in range(max_sweeps):
        # The single-block sweep (hybrid.py:357-385) runs in the native driver: speculative chunks of
        # blocks whose options are valued against the current schedule in one incremental
        # pp_npv_moves evaluation, then decided in the reference's order; the first acceptance ends
        # a chunk (a block's options and values depend only on (a, load, cur_val), which change only
        # when a move is accepted), so the decisions are the sequential ones.
        a32 = a.astype(np.int32)
        cur_val, improved, _ = eng.polish_sweep(a32, load, cur_val, use_sigma=use_sigma, chunk0=_POLISH_CHUNK,
                                                chunk_max=_POLISH_CHUNK_MAX)
        a[...] = a32

        if pair_swaps:
            for b1 in range(B):
                t1 = int(a[b1])
                if t1 == UN:
                    continue
                for b2 in range(b1 + 1, B):
                    t2 = int(a[b2])
                    if t2 == UN or t2 == t1:
                        continue
                    if load[t1] - masses[b1] + masses[b2] > cap[t1]:
                        continue
                    if load[t2] - masses[b2] + masses[b1] > cap[t2]:
                        continue
                    a[b1], a[b2] = t2, t1
                    lo1, hi1 = window(b1)
                    lo2, hi2 = window(b2)
                    ok = lo1 is not None and lo1 <= t2 <= hi1 and lo2 is not None and lo2 <= t1 <= hi2
                    val = float(npv_of(a[None, :])[0]) if ok else -np.inf
                    if ok and val > cur_val + 1e-9:
                        cur_val = val
                        load[t1] += masses[b2] - masses[b1]
                        load[t2] += masses[b1] - masses[b2]
                        improved = True
                    else:
                        a[b1], a[b2] = t1, t2
                    t1 = int(a[b1])

            for b1 in range(B):  # 1-1 exchanges
                t1 = int(a[b1])
                if t1 == UN:
                    continue
                if np.any(a[si_[sp_[b1]:sp_[b1 + 1]]] != UN):
                    continue
                a[b1] = UN
                applied = False
                for b2 in range(B):
                    if b2 == b1 or a[b2] != UN:
                        continue
                    lo2, hi2 = window(b2)
                    if lo2 is None:
                        continue
                    for t2 in range(lo2, hi2 + 1):
                        room = load[t2] - (masses[b1] if t2 == t1 else 0.0) + masses[b2]
                        if room > cap[t2]:
                            continue
                        a[b2] = t2
                        val = float(npv_of(a[None, :])[0])
                        if val > cur_val + 1e-9:
                            cur_val = val
                            load[t1] -= masses[b1]
                            load[t2] += masses[b2]
                            improved = True
                            applied = True
                            break
                        a[b2] = UN
                    if applied:
                        break
                if not applied:
                    a[b1] = t1

            if B <= 12:  # joint pair insertion
                unmined = [b for b in range(B) if a[b] == UN]
                applied = False
                for b1 in unmined:
                    lo1, hi1 = window(b1)
                    if lo1 is None:
                        continue
                    for t1 in range(lo1, hi1 + 1):
                        if load[t1] + masses[b1] > cap[t1]:
                            continue
                        a[b1] = t1
                        load[t1] += masses[b1]
                        for b2 in unmined:
                            if b2 == b1 or a[b2] != UN:
                                continue
                            lo2, hi2 = window(b2)
                            if lo2 is None:
                                continue
                            for t2 in range(lo2, hi2 + 1):
                                if load[t2] + masses[b2] > cap[t2]:
                                    continue
                                a[b2] = t2
                                val = float(npv_of(a[None, :])[0])
                                if val > cur_val + 1e-9:
                                    cur_val = val
                                    load[t2] += masses[b2]
                                    improved = True
                                    applied = True
                                    break
                                a[b2] = UN
                            if applied:
                                break
                        if applied:
                            break
                        load[t1] -= masses[b1]
                        a[b1] = UN
                    if applied:
                        break
        if not improved:
            break
    return cur


def price_column(instance, duals, scenarios, sigma, equipment, seed, evaluator=None, node_cap: int = 5000,
                 capacity_slack: float = 1.0, noise: float = 0.0):
    """colgen.price_column (colgen.py:207-293), same signature and column.

    * the risk-adjusted ENPV table `_enpv_adjusted` (colgen.py:187-204) is `pp_enpv_table` of the
      column's scenario set (k_enpv_table, bit-identical);
    * the noise stream is `substream(seed, ...)` (rng.py:23-32, restated in synth.substream; the
      normal draws are numpy's own Generator, as in the reference);
    * the feasible-sequence greedy (colgen.py:236-254, one scan of every block per pick) runs in
      `pp_price_greedy`;
    * the capacity-slack trim (colgen.py:256-268) walks this package's topological order
      (synth.topological_order, blockmodel.py:228-245) and the column's value / reduced cost
      follow colgen.py:270-293.
    The returned column is the reference's `SequenceColumn` type when pitplan is importable."""
    from .model import UNMINED as UN
    from .synth import substream, topological_order

    e = _entry(instance)
    bm = e.bm
    rng = substream(seed[0], *seed[1:]) if isinstance(seed, tuple) else substream(seed, "price")
    _bind_scenarios(e, scenarios, sigma, None)
    enpv = e.engine.enpv_table(use_sigma=sigma is not None, factored=False)
    masses = bm.mass
    n_t = bm.n_periods
    score = enpv - duals.block[:, None] - np.outer(masses, duals.capacity)
    if noise > 0:
        scale = max(float(np.abs(score).max()), 1e-9)
        score = score + rng.normal(0.0, noise * scale, size=score.shape)
    cap_t = bm.capacity
    cap = np.array([cap_t[t] * capacity_slack for t in range(n_t)], dtype=np.float64)
    a32, _ = e.engine.price_greedy(score, cap, node_cap)
    assign = a32.astype(int)
    in_col = assign != UN

    # trim back to the hard capacity if the slack let the sequence overfill (colgen.py:256-268)
    if capacity_slack > 1.0:
        pp_, pi_, sp_, si_ = bm.csr()
        topo = None
        for t in range(n_t):
            load = float(masses[assign == t].sum())
            if load <= cap_t[t]:
                continue
            if topo is None:
                topo = topological_order(bm)
            for b in topo[::-1].tolist():
                if assign[b] != t:
                    continue
                if np.all(assign[si_[sp_[b]:sp_[b + 1]]] == UN):
                    assign[b] = UN
                    in_col[b] = False
                    load -= masses[b]
                if load <= cap_t[t]:
                    break

    if not in_col.any():
        return None, float("inf")
    mass_t = np.array([float(masses[assign == t].sum()) for t in range(n_t)])
    column = _sequence_column(equipment, assign, mass_t)
    if evaluator is not None:
        column.value = evaluator.npv_relaxed(column.schedule())
    else:
        mined = assign != UN
        column.value = float(enpv[mined, assign[mined]].sum())
    charge = float(duals.block[assign != UN].sum())
    charge += float(duals.capacity @ mass_t)
    charge += float(duals.convexity[equipment])
    column.reduced_cost = column.value - charge
    return column, column.reduced_cost


def _sequence_column(equipment, assign, mass_t):
    """A colgen.SequenceColumn (colgen.py:60-80) -- the reference's record type when importable."""
    try:
        from pitplan.colgen import SequenceColumn
    except Exception:  # noqa: BLE001
        from .model import SequenceColumn
    return SequenceColumn(id=-1, equipment=equipment, assignment=assign, mass_per_period=mass_t, value=0.0)


def clear_cache() -> None:
    cache = _cache()
    while cache:
        _, e = cache.popitem()
        e.engine.close()
