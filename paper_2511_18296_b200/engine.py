"""`Engine`: one device context holding an instance, a scenario set and the current
schedule, exposing the hot path with host (numpy) or device (torch) buffers.

Host-buffer calls are synchronous and are what the drop-in `evaluate_candidates_parallel`
uses; device-buffer calls (`*_device`) only enqueue work on a CUDA stream and are what
the benchmark times with inputs resident in HBM.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import PPBest, PPCandOut, PPMoveOut, check, ptr
from .errors import InvalidArgs, ShapeMismatch
from .model import BlockModel, ScenarioTables, cvar_k

DEFAULT_PSI_WEIGHTS = (0.4, 0.35, 0.25)  # UncertaintyParams.psi_weights (uncertainty.py:147)


class PinnedPool:
    """Page-locked host arrays (pp_host_alloc) for host<->device copies that DMA directly."""

    def __init__(self):
        self.lib = _lib.load()
        self._ptrs = []

    def empty(self, shape, dtype) -> np.ndarray:
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) if np.ndim(shape) else int(shape)
        p = ctypes.c_void_p()
        check(self.lib.pp_host_alloc(max(n * dt.itemsize, 1), ctypes.byref(p)))
        self._ptrs.append(p.value)
        buf = (ctypes.c_char * max(n * dt.itemsize, 1)).from_address(p.value)
        return np.frombuffer(buf, dtype=dt, count=n).reshape(shape)

    def close(self):
        while self._ptrs:
            self.lib.pp_host_free(self._ptrs.pop())


def _i32(a, n=None, name="array") -> np.ndarray:
    out = np.ascontiguousarray(np.asarray(a), dtype=np.int32)
    if n is not None and out.size != n:
        raise ShapeMismatch(f"{name} has {out.size} entries, expected {n}")
    return out


class Engine:
    """A pitplan_b200 context on one CUDA device."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = ctypes.c_void_p()
        check(self.lib.pp_ctx_create(int(device), ctypes.byref(h)))
        self._h = h
        self.device = int(device)
        self.bm: BlockModel | None = None
        self.n_scenarios = 0
        self.has_sigma = False
        self._keep = []
        self._eval_cache = None
        # last host arrays passed without a copy and their addresses (an ndarray's buffer cannot
        # move while a reference is held, and ndarray.ctypes costs ~1.4 us per access)
        self._sched_obj = self._sched_ptr = self._cand_obj = self._cand_ptr = None

    # -- lifecycle -----------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.pp_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @property
    def handle(self):
        return self._h

    def stream(self) -> int:
        s = ctypes.c_void_p()
        check(self.lib.pp_ctx_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def synchronize(self, stream=None):
        check(self.lib.pp_synchronize(self._h, stream))

    # -- static tables ---------------------------------------------------------------
    def set_instance(self, bm: BlockModel):
        B, T = bm.n_blocks, bm.n_periods
        disc = np.ascontiguousarray(bm.discount())
        check(self.lib.pp_set_instance(
            self._h, B, T, bm.n_edges, ptr(bm.edges_i), ptr(bm.edges_j), ptr(bm.mass),
            ptr(np.ascontiguousarray(bm.cost)), ptr(bm.capacity), ptr(disc)))
        self.bm = bm
        self.n_scenarios = 0
        # a new instance (possibly another block count): forget the cached host arrays
        self._sched_obj = self._sched_ptr = self._cand_obj = self._cand_ptr = None
        self._eval_cache = None

    def set_geology(self, psi_weights=DEFAULT_PSI_WEIGHTS, diameter: float | None = None):
        bm = self._need_bm()
        w1, w2, w3 = (float(w) for w in psi_weights)
        diam = bm.diameter() if diameter is None else float(diameter)
        check(self.lib.pp_set_geology(self._h, ptr(bm.alteration), ptr(bm.structural),
                                      ptr(bm.dist_intrusion), w1, w2, w3, diam))

    def set_scenarios(self, tables: ScenarioTables):
        """Bind a scenario set: a host value table vmax[S][B], or -- vmax None -- grades[S][B] from
        which the device builds it (pp_set_scenarios_grades)."""
        bm = self._need_bm()
        S = tables.n_scenarios
        sig = None
        if tables.sigma is not None:
            sig = np.ascontiguousarray(tables.sigma, dtype=np.float64)
            if sig.shape != (S, bm.n_periods):
                raise ShapeMismatch("sigma must be [S][T]")
        if tables.vmax is not None:
            vmax = np.ascontiguousarray(tables.vmax, dtype=np.float64)
            if vmax.ndim != 2 or vmax.shape[1] != bm.n_blocks:
                raise ShapeMismatch("scenario value table does not match the instance")
            check(self.lib.pp_set_scenarios(self._h, S, ptr(vmax), ptr(sig)))
        else:
            g = np.ascontiguousarray(tables.grades, dtype=np.float64)
            if g.ndim != 2 or g.shape[1] != bm.n_blocks:
                raise ShapeMismatch("scenario grades do not match the instance")
            rec = np.ascontiguousarray(bm.recovery_by_mode, dtype=np.float64)
            pc = np.ascontiguousarray(bm.processing_cost_by_mode, dtype=np.float64)
            check(self.lib.pp_set_scenarios_grades(self._h, S, ptr(g), int(bm.n_modes), float(bm.price), ptr(rec),
                                                   rec.size, ptr(pc), pc.size, ptr(sig)))
        self.n_scenarios = int(S)
        self.has_sigma = sig is not None
        self._tables = tables

    def set_vae_decoder(self, decoder):
        """Upload a model.VaeDecoder (the VAE's decoder MLP and normalisation)."""
        bm = self._need_bm()
        widths = np.array(decoder.widths, dtype=np.int32)
        if widths[-1] != bm.n_blocks:
            raise ShapeMismatch("the decoder's output width differs from the instance's block count")
        params = decoder.packed()
        nm = np.ascontiguousarray(decoder.norm_mean, dtype=np.float64)
        ns = np.ascontiguousarray(decoder.norm_std, dtype=np.float64)
        check(self.lib.pp_set_vae_decoder(self._h, int(widths.size - 1), ptr(widths), ptr(params), ptr(nm), ptr(ns)))
        self._vae_latent = int(widths[0])

    def vae_decode(self, z) -> np.ndarray:
        """grades[S][B] = max(decoder(z) * norm_std + norm_mean, 0) on the device (vae.py:284-292)."""
        bm = self._need_bm()
        zz = np.ascontiguousarray(np.atleast_2d(z), dtype=np.float64)
        if zz.shape[1] != getattr(self, "_vae_latent", -1):
            raise ShapeMismatch("z must be [S][latent_dim] of the bound decoder")
        out = np.empty((zz.shape[0], bm.n_blocks), np.float64)
        check(self.lib.pp_vae_decode(self._h, zz.shape[0], ptr(zz), ptr(out), _lib.PP_MEM_HOST, None))
        return out

    def set_scenarios_vae(self, z, sigma=None):
        """Decode prior samples z[S][latent] on the device and bind the grades as the scenario set
        (the value table built there too; nothing returns to the host)."""
        bm = self._need_bm()
        zz = np.ascontiguousarray(np.atleast_2d(z), dtype=np.float64)
        if zz.shape[1] != getattr(self, "_vae_latent", -1):
            raise ShapeMismatch("z must be [S][latent_dim] of the bound decoder")
        S = zz.shape[0]
        sig = None
        if sigma is not None:
            sig = np.ascontiguousarray(sigma, dtype=np.float64)
            if sig.shape != (S, bm.n_periods):
                raise ShapeMismatch("sigma must be [S][T]")
        rec = np.ascontiguousarray(bm.recovery_by_mode, dtype=np.float64)
        pc = np.ascontiguousarray(bm.processing_cost_by_mode, dtype=np.float64)
        check(self.lib.pp_set_scenarios_vae(self._h, S, ptr(zz), int(bm.n_modes), float(bm.price), ptr(rec), rec.size,
                                            ptr(pc), pc.size, ptr(sig)))
        self.n_scenarios = int(S)
        self.has_sigma = sig is not None
        self._tables = None

    def scenario_table(self) -> np.ndarray:
        """vmax[S][B] of the bound scenario set (scenario_mode_values reduced over modes); read back
        from the device when the set was ingested from grades."""
        if getattr(self, "_tables", None) is None:
            if getattr(self, "n_scenarios", 0):  # a set decoded on the device (set_scenarios_vae)
                out = np.empty((self.n_scenarios, self._need_bm().n_blocks), np.float64)
                check(self.lib.pp_get_scenario_values(self._h, ptr(out)))
                return out
            raise InvalidArgs("set_scenarios first")
        if self._tables.vmax is None:
            out = np.empty((self.n_scenarios, self._need_bm().n_blocks), np.float64)
            check(self.lib.pp_get_scenario_values(self._h, ptr(out)))
            self._tables.vmax = out
        return self._tables.vmax

    def _need_bm(self) -> BlockModel:
        if self.bm is None:
            raise InvalidArgs("set_instance first")
        return self.bm

    # -- schedule --------------------------------------------------------------------
    def set_schedule(self, assign):
        """Host numpy array or a device int32 torch tensor."""
        if assign is not None and assign is self._sched_obj:  # the array of the previous call
            check(self.lib.pp_set_schedule(self._h, self._sched_ptr, _lib.PP_MEM_HOST, None))
            return
        bm = self._need_bm()
        if hasattr(assign, "data_ptr"):
            check(self.lib.pp_set_schedule(self._h, assign.data_ptr(), _lib.PP_MEM_DEVICE, None))
            return
        a = _i32(assign, bm.n_blocks, "assignment")  # range validated by pp_set_schedule
        p = ptr(a)
        if a is assign:
            self._sched_obj, self._sched_ptr = a, p
        check(self.lib.pp_set_schedule(self._h, p, _lib.PP_MEM_HOST, None))

    def set_schedule_device(self, assign_tensor, stream=None, borrow: bool = False):
        # borrow: read the device tensor in place (no copy) until the next set_schedule
        mem = _lib.PP_MEM_DEVICE_BORROW if borrow else _lib.PP_MEM_DEVICE
        check(self.lib.pp_set_schedule(self._h, assign_tensor.data_ptr(), mem, stream))

    def apply_moves(self, blocks, periods):
        b = _i32(blocks)
        t = _i32(periods, b.size, "periods")
        check(self.lib.pp_apply_moves(self._h, ptr(b), ptr(t), b.size, _lib.PP_MEM_HOST, None))

    def period_mass_device(self, out_tensor, stream=None):
        """Refresh (if stale) and copy the current period masses into a device f64[T] tensor."""
        check(self.lib.pp_get_schedule(self._h, None, ptr(out_tensor), _lib.PP_MEM_DEVICE, stream))

    def get_schedule(self):
        bm = self._need_bm()
        a = np.empty(bm.n_blocks, dtype=np.int32)
        pm = np.empty(bm.n_periods, dtype=np.float64)
        check(self.lib.pp_get_schedule(self._h, ptr(a), ptr(pm), _lib.PP_MEM_HOST, None))
        return a, pm

    # -- evaluation --------------------------------------------------------------------
    @staticmethod
    def flags(net=False, literal=False, use_sigma=True) -> int:
        f = 0
        if net:
            f |= _lib.PP_NET_MINING_COST
        if literal:
            f |= _lib.PP_LITERAL_VALUE
        if use_sigma:
            f |= _lib.PP_USE_SIGMA
        return f

    def eval_candidates(self, cand, scenario=None, *, net=False, literal=False, use_sigma=True,
                        trace=False, stats=False, scen=False, pairs=False, out: dict | None = None,
                        validate: bool = True, realism: bool = False) -> dict:
        """Host-buffer evaluation; returns numpy arrays (and `best` as a tuple or None).
        `out` may supply preallocated (e.g. pinned) host arrays for any output; page-locked
        arrays (PinnedPool) are written in place by one copy-out launch, and a repeated call
        with the same `out` arrays reuses the argument block (no per-call marshalling).
        pairs=True returns the statistics of the feasible moves only, as
        res["pairs"] = {"cand", "period", "exp", "cvar"} (unordered; capacity C*T).
        realism=True adds res["realism"]: lns_repair's fallback choice (hybrid.py:256-263), the
        feasible candidate with the highest geological consistency, lowest block on ties, as
        (block, period, spatial) or None.
        Candidate ids are range-checked by pp_eval_candidates (`validate` is kept for
        compatibility)."""
        bm = self._need_bm()
        if cand is self._cand_obj:
            c = cand
        else:
            c = cand if (isinstance(cand, np.ndarray) and cand.dtype == np.int32 and cand.flags.c_contiguous) \
                else _i32(cand)
            if c is cand:
                self._cand_obj, self._cand_ptr = c, c.ctypes.data
        C, T, S = c.size, bm.n_periods, self.n_scenarios
        key = None
        if out:
            key = (C, trace, stats, scen, pairs, realism) + tuple(map(id, out.values()))
            hit = self._eval_cache
            if hit is not None and hit[0] == key:
                _, _keep, res, pr, g, argblock = hit
                self._eval_call(c, C, scenario, net, literal, use_sigma, argblock)
                return self._eval_result(res, pr, g)
        out = out or {}
        res = {
            "best_t": out["best_t"] if "best_t" in out else np.empty(C, np.int32),
            "best_val": out["best_val"] if "best_val" in out else np.empty(C, np.float64),
            "feasible": out["feasible"] if "feasible" in out else np.empty(C, np.uint8),
        }
        if trace:
            res["trace_val"] = out["trace_val"] if "trace_val" in out else np.empty((C, T), np.float64)
            res["trace_feas"] = out["trace_feas"] if "trace_feas" in out else np.empty((C, T), np.uint8)
        if stats:
            res["exp_delta"] = out["exp_delta"] if "exp_delta" in out else np.empty((C, T), np.float64)
            res["cvar"] = out["cvar"] if "cvar" in out else np.empty((C, T), np.float64)
        if scen:
            res["scen_delta"] = out["scen_delta"] if "scen_delta" in out else np.empty((C, S, T), np.float32)
        pr = None
        if pairs:
            cap = max(C * T, 1)
            pr = {"cand": out["pair_cand"] if "pair_cand" in out else np.empty(cap, np.int32),
                  "period": out["pair_period"] if "pair_period" in out else np.empty(cap, np.int32),
                  "exp": out["pair_exp"] if "pair_exp" in out else np.empty(cap, np.float64),
                  "cvar": out["pair_cvar"] if "pair_cvar" in out else np.empty(cap, np.float64),
                  "n": out["n_pairs"] if "n_pairs" in out else np.zeros(1, np.int32)}
        g = (PPBest * 2)()  # [0] global best, [1] realism key
        argblock = PPCandOut(
            ptr(res["best_t"]), ptr(res["best_val"]), ptr(res["feasible"]),
            ptr(res.get("trace_val")), ptr(res.get("trace_feas")), ptr(res.get("exp_delta")),
            ptr(res.get("cvar")), ptr(res.get("scen_delta")), ctypes.addressof(g),
            *((ptr(pr["cand"]), ptr(pr["period"]), ptr(pr["exp"]), ptr(pr["cvar"]), ptr(pr["n"])) if pr else ()))
        if realism:
            argblock.realism = ctypes.addressof(g) + ctypes.sizeof(PPBest)
        if key is not None:  # the arrays are kept alive by the cache entry, so their ids stay valid
            self._eval_cache = (key, tuple(out.values()), res, pr, g, argblock)
        self._eval_call(c, C, scenario, net, literal, use_sigma, argblock)
        return self._eval_result(res, pr, g)

    def _eval_call(self, c, C, scenario, net, literal, use_sigma, argblock):
        sc = _lib.PP_SCENARIO_EXPECTED if scenario is None else int(scenario)
        cp = self._cand_ptr if c is self._cand_obj else c.ctypes.data
        check(self.lib.pp_eval_candidates(self._h, cp, C, sc, self.flags(net, literal, use_sigma),
                                          ctypes.byref(argblock), _lib.PP_MEM_HOST, None))

    @staticmethod
    def _eval_result(res, pr, gg):
        res = dict(res)
        g = gg[0]
        res["best"] = None if g.block < 0 else (int(g.block), int(g.period), float(g.value))
        r = gg[1]
        res["realism"] = None if r.block < 0 else (int(r.block), int(r.period), float(r.value))
        if pr is not None:
            n = int(pr["n"][0])
            res["pairs"] = {k: pr[k][:n] for k in ("cand", "period", "exp", "cvar")}
        return res

    def eval_candidates_device(self, cand, out: dict, scenario=None, *, net=False, literal=False,
                               use_sigma=True, stream=None):
        """Device-buffer evaluation: `cand` an int32 CUDA tensor, `out` a dict of CUDA
        tensors (best_t, best_val, feasible, global [16-byte], optional trace_val,
        trace_feas, exp_delta, cvar, scen_delta, or the sparse pair_cand / pair_period /
        pair_exp / pair_cvar [C*T] with n_pairs [1]).  Enqueues on `stream`."""
        o = PPCandOut(
            ptr(out["best_t"]), ptr(out["best_val"]), ptr(out["feasible"]),
            ptr(out.get("trace_val")), ptr(out.get("trace_feas")), ptr(out.get("exp_delta")),
            ptr(out.get("cvar")), ptr(out.get("scen_delta")), ptr(out["global"]),
            ptr(out.get("pair_cand")), ptr(out.get("pair_period")), ptr(out.get("pair_exp")),
            ptr(out.get("pair_cvar")), ptr(out.get("n_pairs")), ptr(out.get("realism")))
        sc = _lib.PP_SCENARIO_EXPECTED if scenario is None else int(scenario)
        check(self.lib.pp_eval_candidates(self._h, ptr(cand), int(cand.numel()), sc,
                                          self.flags(net, literal, use_sigma), ctypes.byref(o),
                                          _lib.PP_MEM_DEVICE, stream))

    def eval_moves(self, a, b, kind="reassign", scenario=None, *, net=False, literal=False,
                   use_sigma=True, stats=False, scen=False, out: dict | None = None) -> dict:
        """Host-buffer evaluation of explicit moves; `out` may supply preallocated (e.g. pinned,
        PinnedPool) output arrays, written in place."""
        bm = self._need_bm()
        av = _i32(a)
        bv = _i32(b, av.size, "move arrays")
        M, S = av.size, self.n_scenarios
        k = _lib.PP_MOVE_SWAP if kind == "swap" else _lib.PP_MOVE_REASSIGN
        out = out or {}

        def buf(name, shape, dt):
            v = out.get(name)
            if v is None:
                return np.empty(shape, dt)
            if v.dtype != np.dtype(dt) or v.size != int(np.prod(shape)) or not v.flags.c_contiguous:
                raise ShapeMismatch(f"out[{name!r}] must be a contiguous {np.dtype(dt)} array of {shape}")
            return v

        res = {"feasible": buf("feasible", M, np.uint8), "delta": buf("delta", M, np.float64)}
        if stats:
            res["exp_delta"] = buf("exp_delta", M, np.float64)
            res["cvar"] = buf("cvar", M, np.float64)
        if scen:
            res["scen_delta"] = buf("scen_delta", (M, S), np.float32)
        g = PPBest()
        out = PPMoveOut(ptr(res["feasible"]), ptr(res["delta"]), ptr(res.get("exp_delta")),
                        ptr(res.get("cvar")), ptr(res.get("scen_delta")), ctypes.addressof(g))
        sc = _lib.PP_SCENARIO_EXPECTED if scenario is None else int(scenario)
        check(self.lib.pp_eval_moves(self._h, k, ptr(av), ptr(bv), M, sc,
                                     self.flags(net, literal, use_sigma), ctypes.byref(out),
                                     _lib.PP_MEM_HOST, None))
        del bm
        res["best"] = None if g.block < 0 else (int(g.block), float(g.value))
        return res

    def eval_moves_device(self, a, b, out: dict, kind="reassign", scenario=None, *, net=False,
                          literal=False, use_sigma=True, stream=None):
        k = _lib.PP_MOVE_SWAP if kind == "swap" else _lib.PP_MOVE_REASSIGN
        o = PPMoveOut(ptr(out["feasible"]), ptr(out["delta"]), ptr(out.get("exp_delta")),
                      ptr(out.get("cvar")), ptr(out.get("scen_delta")), ptr(out["global"]))
        sc = _lib.PP_SCENARIO_EXPECTED if scenario is None else int(scenario)
        check(self.lib.pp_eval_moves(self._h, k, ptr(a), ptr(b), int(a.numel()), sc,
                                     self.flags(net, literal, use_sigma), ctypes.byref(o),
                                     _lib.PP_MEM_DEVICE, stream))

    def check_feasible(self, assign_batch) -> dict:
        bm = self._need_bm()
        a = np.ascontiguousarray(np.atleast_2d(np.asarray(assign_batch)), dtype=np.int32)
        if a.shape[1] != bm.n_blocks:
            raise ShapeMismatch("schedule length does not match the instance")
        P = a.shape[0]
        res = {
            "pred_count": np.empty(P, np.int64),
            "excess": np.empty(P, np.float64),
            "violation": np.empty(P, np.float64),
            "period_mass": np.empty((P, bm.n_periods), np.float64),
        }
        check(self.lib.pp_check_feasible(self._h, ptr(a), P, ptr(res["pred_count"]), ptr(res["excess"]),
                                         ptr(res["violation"]), ptr(res["period_mass"]),
                                         _lib.PP_MEM_HOST, None))
        return res

    def repair(self, assign_batch, mode="push", unmined=False):
        """Returns (repaired int32 [P][B], unmined flags [P][B] or None)."""
        bm = self._need_bm()
        a = np.array(np.atleast_2d(np.asarray(assign_batch)), dtype=np.int32, order="C")
        if a.shape[1] != bm.n_blocks:
            raise ShapeMismatch("schedule length does not match the instance")
        m = _lib.PP_REPAIR_UNMINE if mode == "unmine" else _lib.PP_REPAIR_PUSH_FORWARD
        u = np.empty(a.shape, np.uint8) if unmined else None
        check(self.lib.pp_repair(self._h, ptr(a), a.shape[0], m, ptr(u), _lib.PP_MEM_HOST, None))
        return a, u

    def set_plant(self, plant_hours=None, rate=None):
        """Plant hours per period and the single mode's throughput rate (relaxed NPV); defaults
        from the BlockModel."""
        bm = self._need_bm()
        h = np.ascontiguousarray(bm.plant_hours if plant_hours is None else plant_hours, dtype=np.float64)
        r = float(bm.mode_rates[0] if rate is None else rate)
        check(self.lib.pp_set_plant(self._h, ptr(h), r))
        self._plant = True

    def npv_relaxed(self, assign_batch, use_sigma=True, per_scenario=False):
        """ScheduleEvaluator.npv_relaxed (and per_scenario_npv) of P schedules (evaluate.py:222-258),
        single-mode fast path.  Returns npv[P] (and per_scenario [P][S])."""
        bm = self._need_bm()
        if not getattr(self, "_plant", False):
            if not bm.single_mode_fast:
                raise InvalidArgs("the device stage-2 path needs one mode, one rock type and a positive rate")
            self.set_plant()
        a = np.ascontiguousarray(np.atleast_2d(np.asarray(assign_batch)), dtype=np.int32)
        if a.shape[1] != bm.n_blocks:
            raise ShapeMismatch("schedule length does not match the instance")
        P = a.shape[0]
        npv = np.empty(P, np.float64)
        ps = np.empty((P, self.n_scenarios), np.float64) if per_scenario else None
        f = _lib.PP_USE_SIGMA if (use_sigma and self.has_sigma) else 0
        check(self.lib.pp_npv_relaxed(self._h, ptr(a), P, f, ptr(npv), ptr(ps), _lib.PP_MEM_HOST, None))
        return (npv, ps) if per_scenario else npv

    def stage2(self, assign_batch):
        """Stage-2 optima raw[P][T][S] (sigma = 1) and period mining-cost sums cost[P][T] of P schedules
        (ScheduleEvaluator.stage2_raw, evaluate.py:153-183)."""
        bm = self._need_bm()
        if not getattr(self, "_plant", False):
            if not bm.single_mode_fast:
                raise InvalidArgs("the device stage-2 path needs one mode, one rock type and a positive rate")
            self.set_plant()
        a = np.ascontiguousarray(np.atleast_2d(np.asarray(assign_batch)), dtype=np.int32)
        if a.shape[1] != bm.n_blocks:
            raise ShapeMismatch("schedule length does not match the instance")
        P = a.shape[0]
        raw = np.empty((P, bm.n_periods, self.n_scenarios), np.float64)
        cost = np.empty((P, bm.n_periods), np.float64)
        check(self.lib.pp_stage2(self._h, ptr(a), P, ptr(raw), ptr(cost), _lib.PP_MEM_HOST, None))
        return raw, cost

    def npv_moves(self, assign, blocks, periods, use_sigma=True):
        """Relaxed NPV of the schedules assign with blocks[m] moved to periods[m] (one move each),
        re-solving only the two periods a move changes; equal to npv_relaxed of each variant."""
        bm = self._need_bm()
        if not getattr(self, "_plant", False):
            if not bm.single_mode_fast:
                raise InvalidArgs("the device stage-2 path needs one mode, one rock type and a positive rate")
            self.set_plant()
        a = _i32(assign, bm.n_blocks, "assignment")
        b = _i32(blocks)
        t = _i32(periods, b.size, "periods")
        out = np.empty(b.size, np.float64)
        f = _lib.PP_USE_SIGMA if (use_sigma and self.has_sigma) else 0
        check(self.lib.pp_npv_moves(self._h, ptr(a), ptr(b), ptr(t), b.size, f, ptr(out), _lib.PP_MEM_HOST, None))
        return out

    def polish_sweep(self, assign32: np.ndarray, load: np.ndarray, cur_val: float, use_sigma=True,
                     chunk0: int = 64, chunk_max: int = 128):
        """One single-block sweep of polish_schedule (hybrid.py:357-385) in the C++ driver; assign32
        (int32) and load (f64[T]) are updated in place.  Returns (cur_val, improved, device calls)."""
        bm = self._need_bm()
        if not getattr(self, "_plant", False):
            self.set_plant()
        if assign32.dtype != np.int32 or not assign32.flags.c_contiguous or assign32.size != bm.n_blocks:
            raise ShapeMismatch("assign32 must be a contiguous int32 [B] array")
        if load.dtype != np.float64 or not load.flags.c_contiguous or load.size != bm.n_periods:
            raise ShapeMismatch("load must be a contiguous float64 [T] array")
        cv = ctypes.c_double(cur_val)
        imp = ctypes.c_int32(0)
        calls = ctypes.c_int64(0)
        f = _lib.PP_USE_SIGMA if (use_sigma and self.has_sigma) else 0
        check(self.lib.pp_polish_sweep(self._h, ptr(assign32), ptr(load), ctypes.byref(cv), f, int(chunk0),
                                       int(chunk_max), ctypes.byref(imp), ctypes.byref(calls)))
        return float(cv.value), bool(imp.value), int(calls.value)

    def price_greedy(self, score, cap, node_cap: int):
        """colgen.price_column's sequence greedy (colgen.py:236-254) on the device: score[B][T]
        f64, cap[T] = mining_capacity * capacity_slack; returns (assign int32[B], expansions)."""
        bm = self._need_bm()
        sc = np.ascontiguousarray(score, dtype=np.float64)
        if sc.shape != (bm.n_blocks, bm.n_periods):
            raise ShapeMismatch(f"score has shape {sc.shape}, expected {(bm.n_blocks, bm.n_periods)}")
        cp = np.ascontiguousarray(cap, dtype=np.float64)
        if cp.size != bm.n_periods:
            raise ShapeMismatch(f"cap has {cp.size} entries, expected {bm.n_periods}")
        a = np.empty(bm.n_blocks, np.int32)
        ex = ctypes.c_int64(0)
        check(self.lib.pp_price_greedy(self._h, ptr(sc), ptr(cp), int(node_cap), ptr(a), ctypes.addressof(ex)))
        return a, int(ex.value)

    def spatial(self) -> np.ndarray:
        """geological_consistency of every block (uncertainty.py:185-191), as computed on the device."""
        bm = self._need_bm()
        out = np.empty(bm.n_blocks, np.float64)
        check(self.lib.pp_get_spatial(self._h, ptr(out), _lib.PP_MEM_HOST, None))
        return out

    def eject(self, assign_batch, mean_grade, destroy_fraction=0.0):
        """lns_repair's over-capacity ejection (hybrid.py:213-235), after the unmine fixpoint.
        Returns (assign int32 [P][B], ejected flags uint8 [P][B])."""
        bm = self._need_bm()
        a = np.array(np.atleast_2d(np.asarray(assign_batch)), dtype=np.int32, order="C")
        if a.shape[1] != bm.n_blocks:
            raise ShapeMismatch("schedule length does not match the instance")
        g = np.ascontiguousarray(mean_grade, dtype=np.float64)
        if g.size != bm.n_blocks:
            raise ShapeMismatch("mean_grade length does not match the instance")
        e = np.empty(a.shape, np.uint8)
        check(self.lib.pp_eject(self._h, ptr(a), a.shape[0], ptr(g), float(destroy_fraction), ptr(e),
                                _lib.PP_MEM_HOST, None))
        return a, e

    def lns_destroy(self, assign_batch, mean_grade, destroy_fraction=0.0):
        """The destroy step of lns_repair (hybrid.py:199-235): unmine fixpoint, then ejection.
        Returns (assign [P][B], pool additions [P][B] (fixpoint-unmined or ejected))."""
        a, u = self.repair(assign_batch, mode="unmine", unmined=True)
        a, e = self.eject(a, mean_grade, destroy_fraction)
        return a, (u | e)

    def set_rook(self, rook_ptr, rook_idx):
        """lns_repair's rook neighbour map as a CSR (at most 7 neighbours per block), once per instance."""
        bm = self._need_bm()
        rp = np.ascontiguousarray(rook_ptr, dtype=np.int32)
        ri = np.ascontiguousarray(rook_idx, dtype=np.int32)
        if rp.size != bm.n_blocks + 1:
            raise ShapeMismatch("rook_ptr must have n_blocks + 1 entries")
        check(self.lib.pp_set_rook(self._h, ptr(rp), ptr(ri) if ri.size else None))

    def ensure_rook(self):
        """Upload the instance's rook neighbour map (rook_weights order) once."""
        if getattr(self, "_rook_set", False):
            return
        from .evaluate import _rook_csr
        from .model import rook_neighbor_map, rook_padded

        bm = self._need_bm()
        pad = rook_padded(rook_neighbor_map(bm), bm.n_blocks)
        if pad is None:
            raise ShapeMismatch("a block has 8 or more rook neighbours")
        self.set_rook(*_rook_csr(pad))
        self._rook_set = True

    def uncertainty_sigma(self, grades, kappa=0.1, psi_weights=(0.4, 0.35, 0.25), psi_min=0.5):
        """uncertainty_factors (uncertainty.py:276-321) on the device: (sigma[S][T], moran[S],
        local[S]); agrees with the reference to rounding (its Moran denominator is a BLAS dot)."""
        bm = self._need_bm()
        self.ensure_rook()
        g = np.ascontiguousarray(np.atleast_2d(grades), dtype=np.float64)
        if g.shape[1] != bm.n_blocks:
            raise ShapeMismatch("grades must be [S][n_blocks]")
        # psi_geological (uncertainty.py:173-182) and phi (uncertainty.py:292) on the host, as the reference
        diam = bm.diameter()
        w1, w2, w3 = psi_weights
        dn = np.clip(bm.dist_intrusion / diam, 0.0, 1.0) if diam > 0 else np.zeros_like(bm.dist_intrusion)
        raw = float(np.mean(w1 * bm.alteration + w2 * bm.structural + w3 * dn))
        psi = psi_min + (1.0 - psi_min) * min(max(raw, 0.0), 1.0)
        phi = np.exp(-kappa * np.arange(bm.n_periods))
        S = g.shape[0]
        sig = np.empty((S, bm.n_periods), np.float64)
        mo = np.empty(S, np.float64)
        lo = np.empty(S, np.float64)
        check(self.lib.pp_uncertainty_sigma(self._h, S, ptr(g), ptr(phi), float(psi), ptr(sig), ptr(mo), ptr(lo),
                                            _lib.PP_MEM_HOST, None))
        return sig, mo, lo

    def lns_insert(self, assign, pool, mean_grade, *, max_iters, candidate_width=16, realism_threshold=0.5,
                   only_positive=False, net=False, use_sigma=True):
        """lns_repair's insertion loop (hybrid.py:238-266) as one device-resident CUDA graph
        (pp_lns_insert).  Returns (assign int32 [B], pool uint8 [B], iterations, stalled)."""
        bm = self._need_bm()
        a = np.array(assign, dtype=np.int32, order="C")
        pl = np.array(pool, dtype=np.uint8, order="C")
        g = np.ascontiguousarray(mean_grade, dtype=np.float64)
        if a.size != bm.n_blocks or pl.size != bm.n_blocks or g.size != bm.n_blocks:
            raise ShapeMismatch("assign / pool / mean_grade length does not match the instance")
        it, stl = ctypes.c_int32(0), ctypes.c_int32(0)
        check(self.lib.pp_lns_insert(self._h, ptr(a), ptr(pl), ptr(g), int(max_iters), int(candidate_width),
                                     float(realism_threshold), int(bool(only_positive)),
                                     self.flags(net, False, use_sigma), ctypes.byref(it), ctypes.byref(stl)))
        return a, pl, int(it.value), bool(stl.value)

    def reduce_best_device(self, records, out, stream=None):
        """Ordered argmax over n 16-byte pp_best records (device tensors)."""
        n = records.numel() * records.element_size() // 16
        check(self.lib.pp_reduce_best(self._h, ptr(records), int(n), ptr(out), _lib.PP_MEM_DEVICE, stream))

    def reduce_best(self, recs):
        """Host version: recs = list of (value, block, period) with block < 0 meaning none."""
        arr = (PPBest * max(len(recs), 1))()
        for i, (v, b, t) in enumerate(recs):
            arr[i].value, arr[i].block, arr[i].period = float(v), int(b), int(t)
        g = PPBest()
        check(self.lib.pp_reduce_best(self._h, ctypes.addressof(arr), len(recs), ctypes.addressof(g),
                                      _lib.PP_MEM_HOST, None))
        return None if g.block < 0 else (int(g.block), int(g.period), float(g.value))

    def enpv_table(self, use_sigma=True, factored=False) -> np.ndarray:
        """enpv[B][T]: colgen.py:187-204 form, or hybrid.py:673-678 / saa.py:65-69 when factored."""
        bm = self._need_bm()
        out = np.empty((bm.n_blocks, bm.n_periods), np.float64)
        check(self.lib.pp_enpv_table(self._h, self.flags(use_sigma=use_sigma), int(bool(factored)), ptr(out),
                                     _lib.PP_MEM_HOST, None))
        return out

    def levels(self):
        bm = self._need_bm()
        n = ctypes.c_int32()
        lv = np.empty(bm.n_blocks, np.int32)
        check(self.lib.pp_get_levels(self._h, ctypes.byref(n), ptr(lv)))
        return int(n.value), lv

    # -- convenience -------------------------------------------------------------------
    @classmethod
    def from_tables(cls, bm: BlockModel, tables: ScenarioTables | None, assign=None, device=0,
                    psi_weights=DEFAULT_PSI_WEIGHTS) -> "Engine":
        eng = cls(device)
        eng.set_instance(bm)
        eng.set_geology(psi_weights)
        if tables is not None:
            eng.set_scenarios(tables)
        if assign is not None:
            eng.set_schedule(assign)
        return eng

    @property
    def cvar_k(self) -> int:
        return cvar_k(self.n_scenarios) if self.n_scenarios else 1
