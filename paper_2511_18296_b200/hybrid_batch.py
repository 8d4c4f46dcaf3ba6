"""Batched GA generation for the reference's HybridSearch.

The reference measures every GA member one at a time -- `HybridSearch._measure` runs
`npv_relaxed` and `check_feasible` per schedule (hybrid.py:595-606) -- and mutates each child
with a Python loop over the neighbourhood's blocks (`_mutate`, hybrid.py:692-714).  install()
rebinds three methods of the unchanged class:

* `_member` returns a member whose (npv, violation) are filled lazily: members created between
  two reads of any member's fitness are measured together, one `pp_npv_relaxed` +
  `pp_check_feasible` call over the whole batch (a GA generation's offspring, hybrid.py:752-763;
  the initial population; a restore).  Measurement draws no random numbers and the device values
  of a schedule do not depend on its batch, so every fitness, and the whole run, is unchanged.
* `_measure` keeps the reference's digest-keyed cache (`_eval_cache`) and joins the batch.
* `_mutate` runs the same per-block rule natively (pp_host_mutate) on the caller's Generator
  stream, leaving the Generator exactly where the reference's loop would.

Non-PCG64 generators and evaluators without a batch entry point take the per-member path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check, ptr


class _Batch:
    """Schedules waiting for measurement, keyed by digest, for one HybridSearch."""

    __slots__ = ("search", "items")

    def __init__(self, search):
        self.search = search
        self.items: dict[str, list] = {}  # digest -> [schedule, members...]

    def add(self, key, schedule, member=None):
        ent = self.items.get(key)
        if ent is None:
            ent = self.items[key] = [schedule]
        if member is not None:
            ent.append(member)

    def flush(self):
        if not self.items:
            return
        items, self.items = self.items, {}
        search = self.search
        keys = list(items)
        assigns = np.stack([np.asarray(items[k][0].assignment) for k in keys])
        npv, viol = _measure_many(search, assigns)
        cache = search._eval_cache
        for k, v, w in zip(keys, npv.tolist(), viol.tolist()):
            cache[k] = (v, w)
            for m in items[k][1:]:
                m._set(v, w)


def _measure_many(search, assigns: np.ndarray):
    """(npv[P], violation[P]) of P schedules: one device call each when the evaluator is this
    package's, else the evaluator's own npv_relaxed per schedule."""
    from . import evaluate as ev

    evaluator = search.evaluator
    if isinstance(evaluator, ev.ScheduleEvaluator):
        npv = evaluator.npv_relaxed_batch(assigns)
    else:
        from .model import Schedule

        npv = np.array([evaluator.npv_relaxed(Schedule(a.copy())) for a in assigns], dtype=np.float64)
    viol = ev.check_feasible_batch(search.instance, assigns)["violation"]
    return np.asarray(npv, dtype=np.float64), np.asarray(viol, dtype=np.float64)


class LazyMember:
    """Duck-types hybrid._Member (schedule, npv, violation; hybrid.py:549-552)."""

    __slots__ = ("schedule", "_npv", "_violation", "_batch")

    def __init__(self, schedule, batch=None, npv=float("nan"), violation=float("nan")):
        self.schedule = schedule
        self._npv = npv
        self._violation = violation
        self._batch = batch

    def _set(self, npv, violation):
        self._npv, self._violation, self._batch = npv, violation, None

    @property
    def npv(self) -> float:
        if self._batch is not None:
            self._batch.flush()
        return self._npv

    @property
    def violation(self) -> float:
        if self._batch is not None:
            self._batch.flush()
        return self._violation

    def __repr__(self):
        return f"_Member(npv={self.npv!r}, violation={self.violation!r})"


def _batch_of(search) -> _Batch:
    b = search.__dict__.get("_pp_batch")
    if b is None:
        b = search.__dict__["_pp_batch"] = _Batch(search)
    return b


def member(self, schedule):
    """HybridSearch._member (hybrid.py:608-610), measured lazily in batches."""
    key = schedule.digest()
    hit = self._eval_cache.get(key)
    if hit is not None:
        return LazyMember(schedule, None, hit[0], hit[1])
    b = _batch_of(self)
    m = LazyMember(schedule, b)
    b.add(key, schedule, m)
    return m


def measure(self, schedule):
    """HybridSearch._measure (hybrid.py:595-603): digest-keyed cache, then the pending batch."""
    key = schedule.digest()
    hit = self._eval_cache.get(key)
    if hit is None:
        b = _batch_of(self)
        b.add(key, schedule)
        b.flush()
        hit = self._eval_cache[key]
    return hit


def mutate(self, assign, rng, blocks, rate):
    """HybridSearch._mutate (hybrid.py:692-714) through pp_host_mutate, exact RNG consumption."""
    bg = rng.bit_generator
    a = assign
    if not isinstance(bg, np.random.PCG64) or a.dtype != np.int64 or not a.flags.c_contiguous:
        return _reference_mutate(self, assign, rng, blocks, rate)
    bm = _block_model(self)
    pp_, pi_, sp_, si_ = bm.csr()
    blk = np.ascontiguousarray(np.asarray(blocks), dtype=np.int64)
    lib = _lib.load()
    state = bg.state
    has0, half0 = int(state["has_uint32"]), int(state["uinteger"])
    need = blk.size + 64 + blk.size // 8
    while True:
        raw = bg.random_raw(need)
        has = ctypes.c_int32(has0)
        half = ctypes.c_uint32(half0)
        used = ctypes.c_int64(0)
        rc = lib.pp_host_mutate(ptr(a), bm.n_blocks, ptr(blk), blk.size, ptr(pp_), ptr(pi_), ptr(sp_), ptr(si_),
                                bm.n_periods, float(rate), ptr(raw), raw.size, ctypes.byref(has),
                                ctypes.byref(half), ctypes.byref(used))
        bg.state = state
        if rc == 2:  # PP_ERR_SHAPE: the raw block ran out; the array is untouched
            need *= 2
            continue
        check(rc)
        break
    if used.value:
        bg.random_raw(used.value)
    st = bg.state
    st["has_uint32"] = int(has.value)
    st["uinteger"] = int(half.value)
    bg.state = st


def _block_model(search):
    """The search instance's BlockModel: the engine entry's when one exists, else built once."""
    from . import evaluate as ev
    from .model import BlockModel

    bm = search.__dict__.get("_pp_bm")
    if bm is None:
        inst = search.instance
        e = ev._cache().get(id(inst))
        bm = inst if isinstance(inst, BlockModel) else (e.bm if e is not None and e.instance is inst
                                                        else BlockModel.from_instance(inst))
        search.__dict__["_pp_bm"] = bm
    return bm


def _reference_mutate(self, assign, rng, blocks, rate):
    from . import install as _inst

    fn = _inst.original_attr("pitplan.hybrid.HybridSearch", "_mutate")
    return fn(self, assign, rng, blocks, rate)
