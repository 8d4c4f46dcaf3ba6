"""Python front of the CPU oracle (oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
leg may import this module; the product package never does.

`Oracle(bm, vmax_sb, sigma_st)` takes the raw tables of an instance (any object with
the attributes of paper_2511_18296_b200.model.BlockModel: edges_i/edges_j, mass,
cost, capacity, discount_rate, coords, alteration, structural, dist_intrusion) and
derives everything else itself -- CSR adjacency in reference order
(blockmodel.py:180-184), discount table (evaluate.py:341), diameter
(evaluate.py:342-344), spatial factors (uncertainty.py:185-191), unit values and sigma
row (evaluate.py:291-303, 348-353), period masses (evaluate.py:334-337) -- before
calling the C restatement of the reference kernel.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

_P = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double

_SIGS = {
    "or_np_sum": (_f64, [_P, _i64]),
    "or_period_mass": (None, [_i32, _i32, _P, _P, _P]),
    "or_unit_values": (None, [_i32, _i32, _P, _i32, _i32, _P, _P]),
    "or_sig_row": (None, [_i32, _i32, _P, _i32, _P]),
    "or_spatial": (None, [_i32, _P, _P, _P, _f64, _f64, _f64, _f64, _P]),
    "or_eval_candidates": (None, [_i32, _i32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                  _i32, _P, _P, _P, _P, _P, _P, _P, _P, _i32]),
    "or_candidate_stats": (None, [_i32, _i32, _i32, _P, _P, _P, _P, _P, _P, _P, _i32, _P, _i32, _P, _P,
                                  _P, _i32]),
    "or_check_feasible": (None, [_i32, _i32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "or_topological_order": (ctypes.c_int, [_i32, _P, _P, _P, _P]),
    "or_precedence_repair": (None, [_i32, _P, _P, _P, _P]),
    "or_unmine_fixpoint": (None, [_i32, _i64, _P, _P, _P, _P]),
    "or_enpv_table": (None, [_i32, _i32, _i32, _P, _P, _P, _P, _i32, _P]),
    "or_eject": (None, [_i32, _i32, _P, _P, _P, _P, _P, _f64, _P, _P]),
    "or_price_greedy": (ctypes.c_int64, [_i32, _i32, _P, _P, _P, _P, _P, ctypes.c_int64, _P]),
    "or_npv_relaxed": (None, [_i32, _i32, _i32, _P, _P, _P, _P, _P, _P, _P, _f64, _P, _P]),
    "or_eval_moves": (None, [_i32, _i32, _i32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                             _P, _P, _P, _P, _i32, _i32, _i32, _P, _P, _P, _P, _P, _P, _P, _i32]),
}

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc, no FMA contraction, OpenMP) into oracle/liboracle.so."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-std=c11", "-o", LIB, SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        h = ctypes.CDLL(LIB)
        for name, (res, args) in _SIGS.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def np_sum(x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().or_np_sum(_p(x), x.size)


class Oracle:
    def __init__(self, bm, vmax_sb=None, sigma_st=None, psi_weights=(0.4, 0.35, 0.25)):
        L = lib()
        self.B, self.T = int(bm.n_blocks), int(bm.n_periods)
        B, T = self.B, self.T
        ei = np.ascontiguousarray(bm.edges_i, dtype=np.int32)
        ej = np.ascontiguousarray(bm.edges_j, dtype=np.int32)
        self.ei, self.ej = ei, ej
        # CSR in reference list order: preds[j] += [i], succs[i] += [j] per edge (blockmodel.py:180-184)
        self.pp = np.zeros(B + 1, np.int32)
        self.sp = np.zeros(B + 1, np.int32)
        self.pp[1:] = np.cumsum(np.bincount(ej, minlength=B))
        self.sp[1:] = np.cumsum(np.bincount(ei, minlength=B))
        self.pi = np.ascontiguousarray(ei[np.argsort(ej, kind="stable")], dtype=np.int32)
        self.si = np.ascontiguousarray(ej[np.argsort(ei, kind="stable")], dtype=np.int32)
        self.mass = np.ascontiguousarray(bm.mass, dtype=np.float64)
        self.cost = np.ascontiguousarray(bm.cost, dtype=np.float64).reshape(B, T)
        self.cap = np.ascontiguousarray(bm.capacity, dtype=np.float64)
        r = float(bm.discount_rate)
        self.disc = np.array([(1.0 + r) ** (-t) for t in range(T)], dtype=np.float64)
        coords = np.asarray(bm.coords, dtype=np.float64).reshape(B, 3)
        spans = coords.max(axis=0) - coords.min(axis=0)
        self.diameter = float(np.sqrt((spans**2).sum()))
        self.alt = np.ascontiguousarray(bm.alteration, dtype=np.float64)
        self.strc = np.ascontiguousarray(bm.structural, dtype=np.float64)
        self.dist = np.ascontiguousarray(bm.dist_intrusion, dtype=np.float64)
        self.set_params(psi_weights)
        self.vmax = None if vmax_sb is None else np.ascontiguousarray(vmax_sb, dtype=np.float64)
        self.S = 0 if self.vmax is None else int(self.vmax.shape[0])
        self.sigma = None if sigma_st is None else np.ascontiguousarray(sigma_st, dtype=np.float64)
        self.order = np.empty(B, np.int32)
        if L.or_topological_order(B, _p(self.pp), _p(self.sp), _p(self.si), _p(self.order)) != 0:
            raise ValueError("cycle in precedence graph")

    def set_params(self, psi_weights):
        w1, w2, w3 = (float(w) for w in psi_weights)
        self.spatial = np.empty(self.B, np.float64)
        lib().or_spatial(self.B, _p(self.alt), _p(self.strc), _p(self.dist), w1, w2, w3, self.diameter,
                         _p(self.spatial))

    # -- per-call tables ------------------------------------------------------------
    def period_mass(self, assign) -> np.ndarray:
        a = np.ascontiguousarray(assign, dtype=np.int32)
        pm = np.empty(self.T, np.float64)
        lib().or_period_mass(self.B, self.T, _p(a), _p(self.mass), _p(pm))
        return pm

    def unit(self, s=None, literal=False) -> np.ndarray:
        u = np.empty(self.B, np.float64)
        vm = self.vmax if self.vmax is not None else np.zeros((1, self.B))
        lib().or_unit_values(self.B, vm.shape[0], _p(vm), -1 if s is None else int(s), int(literal),
                             _p(self.mass), _p(u))
        return u

    def sig_row(self, s=None, use_sigma=True) -> np.ndarray:
        out = np.empty(self.T, np.float64)
        sig = self.sigma if use_sigma else None
        S = 0 if sig is None else sig.shape[0]
        lib().or_sig_row(self.T, S, _p(sig), -1 if s is None else int(s), _p(out))
        return out

    # -- evaluate_candidates_parallel (evaluate.py:306-430) ---------------------------
    def eval_candidates(self, assign, cand, s=None, *, net=False, literal=False, use_sigma=True,
                        trace=False, stats=False, scen=False, nthreads=1) -> dict:
        a = np.ascontiguousarray(assign, dtype=np.int32)
        c = np.ascontiguousarray(cand, dtype=np.int32)
        C, T = c.size, self.T
        pm = self.period_mass(a)
        unit = self.unit(s, literal)
        sig_row = self.sig_row(s, use_sigma)
        res = {"best_t": np.empty(C, np.int32), "best_val": np.empty(C, np.float64),
               "feasible": np.empty(C, np.uint8), "period_mass": pm}
        tv = np.empty((C, T), np.float64) if (trace or stats or scen) else None
        tf = np.empty((C, T), np.uint8) if (trace or stats or scen) else None
        gv, gb, gt = _f64(), _i32(), _i32()
        lib().or_eval_candidates(
            self.B, T, _p(self.pp), _p(self.pi), _p(self.sp), _p(self.si), _p(self.mass), _p(self.cap),
            _p(self.disc), _p(self.spatial), _p(unit), _p(sig_row), _p(self.cost) if net else None,
            _p(a), _p(pm), _p(c), C, _p(res["best_t"]), _p(res["best_val"]), _p(res["feasible"]),
            _p(tv), _p(tf), ctypes.addressof(gv), ctypes.addressof(gb), ctypes.addressof(gt), int(nthreads))
        res["best"] = None if gb.value < 0 else (int(gb.value), int(gt.value), float(gv.value))
        if trace:
            res["trace_val"], res["trace_feas"] = tv, tf
        if stats or scen:
            sig = self.sigma if use_sigma else None
            ed = np.empty((C, T), np.float64) if stats else None
            cv = np.empty((C, T), np.float64) if stats else None
            sd = np.empty((C, self.S, T), np.float32) if scen else None
            lib().or_candidate_stats(
                self.B, T, self.S, _p(self.vmax), _p(sig), _p(self.disc), _p(self.spatial),
                _p(self.cost) if net else None, _p(a), _p(c), C, _p(tf), cvar_k(self.S),
                _p(ed), _p(cv), _p(sd), int(nthreads))
            if stats:
                res["exp_delta"], res["cvar"] = ed, cv
            if scen:
                res["scen_delta"] = sd
        return res

    def eval_moves(self, assign, ma, mb, kind="reassign", s=None, *, net=False, literal=False,
                   use_sigma=True, stats=False, scen=False, nthreads=1) -> dict:
        a = np.ascontiguousarray(assign, dtype=np.int32)
        xa = np.ascontiguousarray(ma, dtype=np.int32)
        xb = np.ascontiguousarray(mb, dtype=np.int32)
        M = xa.size
        pm = self.period_mass(a)
        unit = self.unit(s, literal)
        sig_row = self.sig_row(s, use_sigma)
        sig = self.sigma if use_sigma else None
        res = {"feasible": np.empty(M, np.uint8), "delta": np.empty(M, np.float64)}
        ed = np.empty(M, np.float64) if stats else None
        cv = np.empty(M, np.float64) if stats else None
        sd = np.empty((M, self.S), np.float32) if scen else None
        want = stats or scen
        gv, gi = _f64(), _i32()
        lib().or_eval_moves(
            self.B, self.T, self.S if want else 0, _p(self.pp), _p(self.pi), _p(self.sp), _p(self.si),
            _p(self.mass), _p(self.cap), _p(self.disc), _p(self.spatial), _p(unit), _p(sig_row),
            _p(self.cost) if net else None, _p(self.vmax) if want else None, _p(sig), _p(a), _p(pm),
            _p(xa), _p(xb), M, int(kind == "swap"), cvar_k(max(self.S, 1)), _p(res["feasible"]),
            _p(res["delta"]), _p(ed), _p(cv), _p(sd), ctypes.addressof(gv), ctypes.addressof(gi),
            int(nthreads))
        res["best"] = None if gi.value < 0 else (int(gi.value), float(gv.value))
        if stats:
            res["exp_delta"], res["cvar"] = ed, cv
        if scen:
            res["scen_delta"] = sd
        return res

    # -- linear ENPV table (colgen.py:187-204; hybrid.py:673-678) -------------------------
    def enpv_table(self, use_sigma=True, factored=False) -> np.ndarray:
        out = np.empty((self.B, self.T), np.float64)
        sig = self.sigma if use_sigma else None
        lib().or_enpv_table(self.B, self.T, self.S, _p(self.vmax), _p(sig), _p(self.disc), _p(self.cost),
                            int(bool(factored)), _p(out))
        return out

    # -- check_feasible (evaluate.py:82-105) ------------------------------------------
    def check_feasible(self, assign):
        a = np.ascontiguousarray(assign, dtype=np.int32)
        pc, ex, vi = _i64(), _f64(), _f64()
        lib().or_check_feasible(self.B, self.T, _p(self.pp), _p(self.pi), _p(self.mass), _p(self.cap),
                                _p(a), ctypes.addressof(pc), ctypes.addressof(ex), ctypes.addressof(vi))
        return int(pc.value), float(ex.value), float(vi.value)

    # -- repair (hybrid.py:493-510, 199-211) --------------------------------------------
    def precedence_repair(self, assign) -> np.ndarray:
        a = np.array(assign, dtype=np.int32, order="C")
        lib().or_precedence_repair(self.B, _p(self.pp), _p(self.pi), _p(self.order), _p(a))
        return a

    def npv_relaxed(self, assign, plant_hours, rate, use_sigma=True):
        """ScheduleEvaluator.npv_relaxed / per_scenario_npv on the single-mode fast path
        (evaluate.py:166-183, 222-258) -> (npv, per_scenario[S])."""
        a = np.ascontiguousarray(assign, dtype=np.int32)
        h = np.ascontiguousarray(plant_hours, dtype=np.float64)
        out = np.zeros(1)
        ps = np.zeros(self.S)
        sig = self.sigma if (use_sigma and self.sigma is not None) else None
        lib().or_npv_relaxed(self.B, self.T, self.S, _p(a), _p(self.mass), _p(self.cost), _p(self.vmax),
                             _p(sig) if sig is not None else None, _p(self.disc), _p(h), float(rate),
                             _p(out), _p(ps))
        return float(out[0]), ps

    def eject(self, assign, mean_grade, destroy_fraction=0.0):
        """lns_repair's over-capacity ejection (hybrid.py:213-235) -> (assign, ejected mask)."""
        a = np.array(assign, dtype=np.int32, order="C")
        g = np.ascontiguousarray(mean_grade, dtype=np.float64)
        e = np.empty(self.B, np.uint8)
        lib().or_eject(self.B, self.T, _p(self.sp), _p(self.si), _p(self.mass), _p(self.cap), _p(g),
                       float(destroy_fraction), _p(a), _p(e))
        return a, e

    def price_greedy(self, score, cap, node_cap):
        """colgen.price_column's sequence greedy (colgen.py:236-254) -> (assign int32, expansions)."""
        sc = np.ascontiguousarray(score, dtype=np.float64)
        cp = np.ascontiguousarray(cap, dtype=np.float64)
        a = np.empty(self.B, np.int32)
        ex = lib().or_price_greedy(self.B, self.T, _p(self.pp), _p(self.pi), _p(self.mass), _p(sc), _p(cp),
                                   int(node_cap), _p(a))
        return a, int(ex)

    def unmine_fixpoint(self, assign):
        a = np.array(assign, dtype=np.int32, order="C")
        u = np.empty(self.B, np.uint8)
        lib().or_unmine_fixpoint(self.B, self.ei.size, _p(self.ei), _p(self.ej), _p(a), _p(u))
        return a, u


def cvar_k(n: int) -> int:
    """ceil(0.1 n) (saa.py:157)."""
    return max(1, math.ceil(0.1 * n))
