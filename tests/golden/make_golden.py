"""Generate tests/golden/*.npz by running the REFERENCE implementation (pitplan) in the
build container.  Run:  python tests/golden/make_golden.py

The reference checkout (/root/reference) is not available on the GPU box, so its
outputs are frozen here together with the inputs (small cases) or sha256 digests of
the inputs (large cases, rebuilt bit-identically by paper_2511_18296_b200.synth).
Every array below is produced by calling the reference's own functions:

  evaluate_candidates_parallel  evaluate.py:306-430   (moves, best, trace CSV)
  check_feasible                evaluate.py:82-105
  _precedence_repair_pass       hybrid.py:493-510
  lns_repair (max_iters=0)      hybrid.py:199-211 unmine fixpoint
  risk_metrics                  saa.py:150-166 (CVaR10 of per-scenario deltas)
  vae_generate                  vae.py:306-321 (python make_golden.py vae -> vae.npz)
"""

from __future__ import annotations

import csv
import hashlib
import os
import sys
import tempfile

import numpy as np

REF = os.environ.get("PITPLAN_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from pitplan.colgen import _enpv_adjusted  # noqa: E402
from pitplan.blockmodel import UNMINED, Block, Economics, GeoFeatures, Instance, OperatingMode, generate_synthetic  # noqa: E402
from pitplan.evaluate import Schedule, ScheduleEvaluator, check_feasible, evaluate_candidates_parallel  # noqa: E402
from pitplan.hybrid import _precedence_repair_pass, greedy_initialize, lns_repair, polish_schedule  # noqa: E402
from pitplan.rng import substream  # noqa: E402
from pitplan.saa import risk_metrics  # noqa: E402
from pitplan.scenarios import builtin_scenarios, sample_lognormal  # noqa: E402
from pitplan.uncertainty import uncertainty_factors  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def flat(inst: Instance, prefix: str) -> dict:
    """Raw tables of a reference Instance (no product code involved)."""
    prec = np.asarray(inst.precedence, dtype=np.int64).reshape(-1, 2)
    return {
        f"{prefix}n_blocks": np.int64(inst.n_blocks),
        f"{prefix}n_periods": np.int64(inst.n_periods),
        f"{prefix}edges": prec,
        f"{prefix}mass": inst.masses(),
        f"{prefix}cost": inst.mining_costs().reshape(inst.n_blocks, inst.n_periods),
        f"{prefix}capacity": np.asarray(inst.mining_capacity, dtype=np.float64),
        f"{prefix}discount_rate": np.float64(inst.discount_rate),
        f"{prefix}coords": inst.coords_array().reshape(inst.n_blocks, 3),
        f"{prefix}features": np.array([(b.features.alteration_intensity, b.features.structural_density,
                                        b.features.distance_to_intrusion) for b in inst.blocks]).reshape(-1, 3),
        f"{prefix}plant_hours": np.asarray(inst.plant_hours, dtype=np.float64),
        f"{prefix}mode_rates": np.array([m.rate for m in inst.modes], dtype=np.float64),
        f"{prefix}n_rock_types": np.int64(len(inst.rock_types)),
    }


def vmax_of(inst, scen) -> np.ndarray:
    from pitplan.evaluate import scenario_mode_values

    return scenario_mode_values(inst, scen).max(axis=2)


def full_greedy(inst) -> np.ndarray:
    """HybridSearch._full_greedy (hybrid.py:643-667) without building a HybridSearch."""
    masses = inst.masses()
    assign = np.full(inst.n_blocks, UNMINED, dtype=int)
    load = np.zeros(inst.n_periods)
    for b in inst.topological_order():
        t_min, ok = 0, True
        for p in inst.predecessors(b):
            if assign[p] == UNMINED:
                ok = False
                break
            t_min = max(t_min, assign[p])
        if not ok:
            continue
        for t in range(t_min, inst.n_periods):
            if load[t] + masses[b] <= inst.mining_capacity[t]:
                assign[b] = t
                load[t] += masses[b]
                break
    return assign


def run_kernel(inst, sched, cand, scen, s, sigma, **kw):
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "trace.csv")
        moves, best = evaluate_candidates_parallel(inst, sched, cand, scen, s, sigma, trace_path=path, **kw)
        rows = list(csv.reader(open(path)))[1:]
    T = inst.n_periods
    # trace rows are sorted by (candidate, period); re-key to input order [C][T]
    by_key = {(int(r[0]), int(r[1])): (int(r[2]), float(r[3])) for r in rows}
    tv = np.array([[by_key[(int(b), t)][1] for t in range(T)] for b in cand], dtype=np.float64).reshape(-1, T)
    tf = np.array([[by_key[(int(b), t)][0] for t in range(T)] for b in cand], dtype=np.uint8).reshape(-1, T)
    out = {
        "best_t": np.array([m.period for m in moves], dtype=np.int32),
        "best_val": np.array([m.improvement for m in moves], dtype=np.float64),
        "feasible": np.array([m.feasible for m in moves], dtype=np.uint8),
        "best": np.array([best.block, best.period, best.improvement] if best else [-1, -1, -np.inf]),
        "trace_val": tv,
        "trace_feas": tf,
    }
    return out


def put(store: dict, prefix: str, res: dict, keys=("best_t", "best_val", "feasible", "best", "trace_val", "trace_feas")):
    for k in keys:
        store[f"{prefix}{k}"] = res[k]


def scenario_stats(inst, sched, cand, scen, sigma, net=False):
    """Per-scenario deltas d_k(b,t) = kernel value with s=k at t minus at the current period,
    from the reference kernel's own trace; expected = np.mean over k, CVaR10 via risk_metrics."""
    S, T, C = scen.n_s, inst.n_periods, len(cand)
    vals = np.empty((S, C, T))
    for k in range(S):
        vals[k] = run_kernel(inst, sched, cand, scen, k, sigma, net_mining_cost=net)["trace_val"]
    a = sched.assignment
    d = np.empty((S, C, T))
    feas = np.isfinite(vals[0])
    for i, b in enumerate(cand):
        ab = a[b]
        for k in range(S):
            d[k, i] = vals[k, i] - vals[k, i, ab] if ab != UNMINED else vals[k, i]
    exp = np.full((C, T), -np.inf)
    cvar = np.full((C, T), -np.inf)
    for i in range(C):
        for t in range(T):
            if feas[i, t]:
                exp[i, t] = float(np.mean(d[:, i, t]))
                cvar[i, t] = risk_metrics(d[:, i, t]).cvar10
    d = np.where(feas[None], d, -np.inf)
    return np.transpose(d, (1, 0, 2)).astype(np.float32), exp, cvar


# ------------------------------------------------------------------------------------------
def small_cases(store):
    """The 20 TestKernelDeterminism cases (test_acceptance.py:140-165) plus variants."""
    for case in range(20):
        p = f"kd{case}_"
        inst = generate_synthetic(27, (3, 3, 3), 3, 1, seed=300 + case, n_rock_types=1)
        scen = sample_lognormal(inst, 2, 0.3, seed=400 + case)
        sigma = uncertainty_factors(inst, scen.grades)
        sched = greedy_initialize(inst, scen, sigma)
        drop = substream(500 + case, "kern").choice(27, size=6, replace=False)
        for b in drop:
            sched.assignment[b] = -1
        cand = [int(b) for b in drop]
        store.update(flat(inst, p))
        store[p + "vmax"] = vmax_of(inst, scen)
        store[p + "sigma"] = sigma.sigma
        store[p + "assign"] = sched.assignment.astype(np.int32)
        store[p + "cand"] = np.array(cand, dtype=np.int32)
        store[p + "enpv"] = _enpv_adjusted(inst, scen, sigma)
        store[p + "enpv_nosig"] = _enpv_adjusted(inst, scen, None)
        put(store, p + "s0_", run_kernel(inst, sched, cand, scen, 0, sigma))
        put(store, p + "sN_", run_kernel(inst, sched, cand, scen, None, sigma))
        put(store, p + "net_", run_kernel(inst, sched, cand, scen, None, sigma, net_mining_cost=True))
        put(store, p + "nosig_", run_kernel(inst, sched, cand, scen, 1, None))
        put(store, p + "lit_", run_kernel(inst, sched, cand, scen, 0, sigma, literal_kernel_value=True))
        # all-blocks candidates on the undamaged greedy schedule (mined candidates too)
        sched2 = greedy_initialize(inst, scen, sigma)
        allc = list(range(27))
        store[p + "assign2"] = sched2.assignment.astype(np.int32)
        put(store, p + "all_", run_kernel(inst, sched2, allc, scen, None, sigma, net_mining_cost=True))
        sd, ex, cv = scenario_stats(inst, sched2, allc, scen, sigma, net=True)
        store[p + "all_scen_delta"], store[p + "all_exp"], store[p + "all_cvar"] = sd, ex, cv
        # check_feasible / repair / unmine fixpoint on random assignments
        rng = np.random.default_rng(1000 + case)
        rand = rng.integers(-1, 3, size=(4, 27))
        store[p + "rand"] = rand.astype(np.int32)
        cf = [check_feasible(inst, Schedule(r)) for r in rand]
        store[p + "rand_pred"] = np.array([c.precedence_violations for c in cf], dtype=np.int64)
        store[p + "rand_excess"] = np.array([c.capacity_excess for c in cf])
        store[p + "rand_viol"] = np.array([c.violation for c in cf])
        rep = []
        for r in rand:
            a = r.copy()
            _precedence_repair_pass(inst, a)
            rep.append(a)
        store[p + "rand_repair"] = np.array(rep, dtype=np.int32)
        big = Instance(blocks=inst.blocks, precedence=inst.precedence, n_periods=inst.n_periods,
                       mining_capacity=tuple([1e12] * inst.n_periods), plant_hours=inst.plant_hours,
                       modes=inst.modes, rock_types=inst.rock_types, discount_rate=inst.discount_rate,
                       economics=inst.economics)
        fix = [lns_repair(big, Schedule(r), [], scen, None, max_iters=0).assignment for r in rand]
        store[p + "rand_unmine"] = np.array(fix, dtype=np.int32)
        # lns_repair's destroy step with the real capacities: unmine fixpoint + over-capacity
        # ejection (hybrid.py:199-235), destroy_fraction 0 and 0.3; a result equal to the input
        # while the fixpoint changed something would be the violation guard's revert (skipped)
        store[p + "mean_grade"] = scen.grades.mean(axis=0)
        store[p + "grades"] = scen.grades
        # relaxed NPV (stage-1 costs + stage-2 greedy knapsack per (s, t), evaluate.py:166-183,
        # 222-258) of the random schedules and of the greedy one, with and without sigma
        ev, ev0 = ScheduleEvaluator(inst, scen, sigma), ScheduleEvaluator(inst, scen, None)
        pop = [Schedule(r) for r in rand] + [Schedule(sched2.assignment.copy())]
        store[p + "npv_pop"] = np.array([x.assignment for x in pop], dtype=np.int32)
        store[p + "npv"] = np.array([ev.npv_relaxed(x) for x in pop])
        store[p + "npv_nosig"] = np.array([ev0.npv_relaxed(x) for x in pop])
        store[p + "npv_scen"] = np.array([ev.per_scenario_npv(x) for x in pop])
        # whole lns_repair runs (destroy + similarity-ranked insertions, hybrid.py:169-274)
        for tag, kw in (("a", dict(max_iters=50)),
                        ("b", dict(max_iters=50, destroy_fraction=0.3, net_mining_cost=True)),
                        ("c", dict(max_iters=50, realism_threshold=0.95, candidate_width=4))):
            outs = [lns_repair(inst, Schedule(r), [0, 5], scen, sigma, **kw).assignment.astype(np.int32)
                    for r in rand[:2]]
            store[p + f"lns_{tag}"] = np.array(outs)
        for tag, df in (("d0", 0.0), ("d3", 0.3)):
            outs = []
            for r in rand:
                out = lns_repair(inst, Schedule(r), [], scen, None, max_iters=0, destroy_fraction=df).assignment
                before = check_feasible(inst, Schedule(r)).violation
                after = check_feasible(inst, Schedule(out)).violation
                assert after <= before, "violation guard reverted a destroy step"
                outs.append(out)
            store[p + f"rand_destroy_{tag}"] = np.array(outs, dtype=np.int32)


def _feat(alt=0.5, struct=0.5, dist=1.0):
    return GeoFeatures(alteration_intensity=alt, structural_density=struct, distance_to_intrusion=dist)


def _block(bid, mass, coords, grade, n_periods, cost=0.0):
    return Block(id=bid, mass=float(mass), coords=tuple(float(c) for c in coords), base_grade=float(grade),
                 rock_type_by_scenario=(0,), features=_feat(),
                 mining_cost_by_period=tuple([float(cost)] * n_periods))


def _instance(blocks, precedence=(), n_periods=1, capacity=1e9):
    modes = [OperatingMode(id=0, rate=100.0, blend_fraction={"ore": 1.0},
                           value=tuple((100.0,) for _ in blocks))]
    return Instance(blocks=list(blocks), precedence=[tuple(e) for e in precedence], n_periods=n_periods,
                    mining_capacity=tuple([capacity] * n_periods), plant_hours=tuple([1e9] * n_periods),
                    modes=modes, rock_types=["ore"], discount_rate=0.08, economics=Economics())


def hand_cases(store):
    """Worked examples of test_evaluate.py:20-50 and 204-258."""
    cases = {
        # forced choice: block 1 fits only period 1 (test_evaluate.py:204-211)
        "forced": (_instance([_block(0, 100, (0, 0, 0), 1, 2), _block(1, 100, (0, 0, 1), 1, 2)], [(0, 1)], 2, 150.0),
                   [0, UNMINED], [1], 0, False),
        # earlier period wins under discounting (213-220)
        "early": (_instance([_block(0, 100, (0, 0, 0), 1, 2)], (), 2, 500.0), [UNMINED], [0], 0, False),
        # infeasible sentinel (238-245)
        "infeas": (_instance([_block(0, 100, (0, 0, 0), 1, 1), _block(1, 100, (0, 0, 1), 1, 1)], [(0, 1)], 1),
                   [UNMINED, UNMINED], [1], 0, False),
        # literal kernel value 100*100*factor = 11250 (247-258)
        "literal": (_instance([_block(0, 100, (0, 0, 0), 1, 1)], (), 1, 500.0), [UNMINED], [0], 0, True),
    }
    for name, (inst, assign, cand, s, lit) in cases.items():
        p = f"hand_{name}_"
        scen = builtin_scenarios(inst)
        sched = Schedule(np.array(assign))
        store.update(flat(inst, p))
        store[p + "vmax"] = vmax_of(inst, scen)
        store[p + "assign"] = np.array(assign, dtype=np.int32)
        store[p + "cand"] = np.array(cand, dtype=np.int32)
        store[p + "literal"] = np.int64(lit)
        put(store, p, run_kernel(inst, sched, cand, scen, s, None, literal_kernel_value=lit))
    feas = {
        "prec": (_instance([_block(0, 100, (0, 0, 0), 1, 2), _block(1, 100, (0, 0, 1), 1, 2)], [(0, 1)], 2), [1, 0]),
        "unmined_parent": (_instance([_block(0, 100, (0, 0, 0), 1, 2), _block(1, 100, (0, 0, 1), 1, 2)], [(0, 1)], 2),
                           [UNMINED, 0]),
        "same": (_instance([_block(0, 100, (0, 0, 0), 1, 2), _block(1, 100, (0, 0, 1), 1, 2)], [(0, 1)], 2), [0, 0]),
        "capacity": (_instance([_block(0, 600, (0, 0, 0), 1, 1), _block(1, 600, (1, 0, 0), 1, 1)], (), 1, 1000.0), [0, 0]),
        "empty": (generate_synthetic(8, (2, 2, 2), 3, 1, seed=11, n_rock_types=1), [UNMINED] * 8),
    }
    for name, (inst, assign) in feas.items():
        p = f"feas_{name}_"
        store.update(flat(inst, p))
        store[p + "assign"] = np.array(assign, dtype=np.int32)
        r = check_feasible(inst, Schedule(np.array(assign)))
        store[p + "out"] = np.array([r.precedence_violations, r.capacity_excess, r.violation])


def config_case(store, name, n, dims, T, S, C, cf=1.3, scen_subset=0):
    inst = generate_synthetic(n, dims, T, 1, seed=1, n_rock_types=1, capacity_factor=cf)
    scen = sample_lognormal(inst, S, 0.3, seed=2)
    sigma = uncertainty_factors(inst, scen.grades)
    cand = substream(3, "cand").integers(0, n, size=C).astype(np.int32)
    p = f"{name}_"
    f = flat(inst, "")
    store[p + "digest_instance"] = np.bytes_(digest(f["edges"].astype(np.int32), f["mass"], f["cost"], f["capacity"],
                                                    f["coords"], f["features"]))
    store[p + "digest_scen"] = np.bytes_(digest(vmax_of(inst, scen), sigma.sigma))
    store[p + "digest_vmax"] = np.bytes_(digest(vmax_of(inst, scen)))
    # sigma[S][T] depends on a BLAS dot product (Moran's I), whose rounding varies with the
    # host's thread count: freeze the small matrix itself
    store[p + "sigma"] = sigma.sigma
    store[p + "cand"] = cand
    if n <= 4000:
        store[p + "enpv"] = _enpv_adjusted(inst, scen, sigma)
    for sname, assign in (("full", full_greedy(inst)), ("greedy", greedy_initialize(inst, scen, sigma).assignment)):
        q = f"{p}{sname}_"
        sched = Schedule(assign)
        store[q + "digest_assign"] = np.bytes_(digest(assign.astype(np.int32)))
        keys = ("best_t", "best_val", "feasible", "best") + (("trace_val", "trace_feas") if n <= 4000 else ())
        put(store, q + "sN_", run_kernel(inst, sched, cand.tolist(), scen, None, sigma), keys)
        put(store, q + "net_", run_kernel(inst, sched, cand.tolist(), scen, None, sigma, net_mining_cost=True), keys)
        put(store, q + "s0_", run_kernel(inst, sched, cand.tolist(), scen, 0, sigma), keys)
        r = check_feasible(inst, sched)
        store[q + "feas"] = np.array([r.precedence_violations, r.capacity_excess, r.violation])
        if scen_subset and sname == "full":
            sub = cand[:scen_subset].tolist()
            sd, ex, cv = scenario_stats(inst, sched, sub, scen, sigma, net=True)
            store[q + "sub_scen_delta"], store[q + "sub_exp"], store[q + "sub_cvar"] = sd, ex, cv
    # repair pass on crossover-like damaged schedules (hybrid.py:716-722 shape)
    rng = np.random.default_rng(7)
    full = full_greedy(inst)
    emp = np.full(n, UNMINED)
    reps, srcs = [], []
    for k in range(3):
        cut = int(rng.integers(1, n))
        child = full.copy()
        child[cut:] = rng.integers(-1, T, size=n - cut) if k == 2 else emp[cut:]
        srcs.append(child.astype(np.int32))
        a = child.copy()
        _precedence_repair_pass(inst, a)
        reps.append(a.astype(np.int32))
    store[p + "repair_in"] = np.array(srcs)
    store[p + "repair_out"] = np.array(reps)
    if n <= 4000:  # lns_repair's destroy step (hybrid.py:199-235) on overloaded schedules
        store[p + "mean_grade"] = scen.grades.mean(axis=0)
        ins = []
        tm = int(full.max())  # the last period the full schedule uses
        for merge in (((tm, tm - 1),), ((tm - 1, tm - 2), (tm, tm - 2)), ((1, 0),)):
            a = full.copy()  # merging a period into an earlier one keeps precedence, overloads it
            for src, dst in merge:
                a[a == src] = dst
            ins.append(a.astype(np.int32))
        a = full.copy()  # plus a precedence-damaged one (the fixpoint runs first)
        mined = np.nonzero(a >= 0)[0]
        pick = rng.choice(mined, size=len(mined) // 10, replace=False)
        a[pick] = rng.integers(0, max(1, T // 3), size=pick.size)
        ins.append(a.astype(np.int32))
        store[p + "destroy_in"] = np.array(ins)
        for tag, df in (("d0", 0.0), ("d25", 0.25)):
            outs = [lns_repair(inst, Schedule(a.astype(int)), [], scen, None, max_iters=0,
                               destroy_fraction=df).assignment.astype(np.int32) for a in ins]
            store[p + f"destroy_{tag}"] = np.array(outs)
        # relaxed NPV of the config's schedules (evaluate.py:222-258)
        ev = ScheduleEvaluator(inst, scen, sigma)
        pop = [full.astype(np.int32), greedy_initialize(inst, scen, sigma).assignment.astype(np.int32)] + list(ins)
        store[p + "npv_pop"] = np.array(pop, dtype=np.int32)
        store[p + "npv"] = np.array([ev.npv_relaxed(Schedule(a.astype(int))) for a in pop])
        store[p + "npv_scen"] = np.array([ev.per_scenario_npv(Schedule(a.astype(int))) for a in pop])
        store[p + "plant_hours"] = np.asarray(inst.plant_hours, dtype=np.float64)
        store[p + "mode_rates"] = np.array([m.rate for m in inst.modes], dtype=np.float64)
        # a whole lns_repair run at 4k blocks (40 insertion rounds after the destroy step)
        store[p + "grades"] = scen.grades
        store[p + "lns"] = lns_repair(inst, Schedule(ins[0].astype(int)), [], scen, sigma, max_iters=40,
                                      destroy_fraction=0.1).assignment.astype(np.int32)


def polish_cases(store):
    """polish_schedule (hybrid.py:326-490) runs: 8 blocks (joint pair insertion), 27 blocks (pair
    swaps, 1-1 exchanges), 512 blocks (single-block sweeps only)."""
    for name, n, dims, T, S, sweeps in (("p8", 8, (2, 2, 2), 3, 3, 3), ("p27", 27, (3, 3, 3), 3, 2, 3),
                                        ("p512", 512, (8, 8, 8), 6, 4, 2)):
        inst = generate_synthetic(n, dims, T, 1, seed=70 + n, n_rock_types=1, capacity_factor=0.9)
        scen = sample_lognormal(inst, S, 0.3, seed=71 + n)
        sigma = uncertainty_factors(inst, scen.grades)
        p = f"{name}_"
        store.update(flat(inst, p))
        store[p + "vmax"] = vmax_of(inst, scen)
        store[p + "sigma"] = sigma.sigma
        ev = ScheduleEvaluator(inst, scen, sigma)
        starts = [greedy_initialize(inst, scen, sigma).assignment.copy()]
        rng = np.random.default_rng(n)
        a = starts[0].copy()
        a[rng.random(n) < 0.3] = UNMINED
        _precedence_repair_pass(inst, a)
        starts.append(a)
        store[p + "start"] = np.array(starts, dtype=np.int32)
        store[p + "out"] = np.array([polish_schedule(inst, ev, Schedule(x.copy()), max_sweeps=sweeps).assignment
                                     for x in starts], dtype=np.int32)
        store[p + "sweeps"] = np.int64(sweeps)


def price_cases(store):
    """colgen.price_column (colgen.py:207-293) runs: the score matrix is formed exactly as
    colgen.py:227-234 does (the reference's own _enpv_adjusted and substream), and the expected
    sequence is the reference's returned column (capacity_slack 1.0: no trim)."""
    from pitplan.colgen import DualPrices, price_column

    cases = (("q8", 8, (2, 2, 2), 3, 2, 0.0, 5000, "zero"), ("q27", 27, (3, 3, 3), 3, 3, 0.4, 5000, "zero"),
             ("q512", 512, (8, 8, 8), 6, 4, 0.0, 10 ** 7, "rand"), ("q512n", 512, (8, 8, 8), 6, 4, 0.3, 700, "rand"),
             ("qC1", 4000, (20, 20, 10), 10, 5, 0.0, 5000, "rand"), ("qC1big", 4000, (20, 20, 10), 10, 5, 0.2, 10 ** 7,
                                                                     "rand"))
    for name, n, dims, T, S, noise, node_cap, dk in cases:
        inst = generate_synthetic(n, dims, T, 1, seed=90 + n, n_rock_types=1, capacity_factor=0.6)
        scen = sample_lognormal(inst, S, 0.3, seed=91 + n)
        sigma = uncertainty_factors(inst, scen.grades)
        rng = np.random.default_rng(n + T)
        if dk == "zero":
            duals = DualPrices(block=np.zeros(n), capacity=np.zeros(T), convexity=np.zeros(1))
        else:
            enpv0 = _enpv_adjusted(inst, scen, sigma)
            duals = DualPrices(block=np.abs(rng.normal(0, 0.3, n)) * np.abs(enpv0).mean(),
                               capacity=np.abs(rng.normal(0, 0.5, T)) * np.abs(enpv0).mean() / inst.masses().mean(),
                               convexity=np.zeros(1))
        seed = (5, "price", n)
        col, rc = price_column(inst, duals, scen, sigma, 0, seed, node_cap=node_cap, noise=noise)
        # the score the greedy sees (colgen.py:226-234, same calls in the same order)
        srng = substream(seed[0], *seed[1:])
        enpv = _enpv_adjusted(inst, scen, sigma)
        score = enpv - duals.block[:, None] - np.outer(inst.masses(), duals.capacity)
        if noise > 0:
            scale = max(float(np.abs(score).max()), 1e-9)
            score = score + srng.normal(0.0, noise * scale, size=score.shape)
        p = f"{name}_"
        store.update(flat(inst, p))
        store[p + "score"] = score
        store[p + "cap"] = np.array([inst.mining_capacity[t] * 1.0 for t in range(T)], dtype=np.float64)
        store[p + "node_cap"] = np.int64(node_cap)
        store[p + "assign"] = (np.full(n, UNMINED) if col is None else col.assignment).astype(np.int32)
        store[p + "rc"] = np.float64(rc)


def stats_cases(store):
    """Per-scenario statistics with CVaR10 over k > 1 scenarios, from the reference kernel itself
    (run once per scenario with s=k) and saa.risk_metrics: a C2 subset (S = 20, k = 2) and a C3
    subset (S = 200, k = 20: the many-scenario warp-selection path).  Inputs are rebuilt by the
    package's synth module and checked against the digests stored here."""
    for name, cf, S, n_sub in (("C2", 1.3, 20, 300), ("C3", 0.3, 200, 60)):
        inst = generate_synthetic(50000, (50, 50, 20), 15, 1, seed=1, n_rock_types=1, capacity_factor=cf)
        scen = sample_lognormal(inst, S, 0.3, seed=2)
        sigma = uncertainty_factors(inst, scen.grades)
        cand = substream(3, "cand").integers(0, 50000, size=16667).astype(np.int32)
        p = f"{name}_"
        f = flat(inst, "")
        store[p + "digest_instance"] = np.bytes_(digest(f["edges"].astype(np.int32), f["mass"], f["cost"],
                                                        f["capacity"], f["coords"], f["features"]))
        store[p + "digest_vmax"] = np.bytes_(digest(vmax_of(inst, scen)))
        store[p + "sigma"] = sigma.sigma
        full = full_greedy(inst)
        store[p + "digest_assign"] = np.bytes_(digest(full.astype(np.int32)))
        # the subset: candidates with at least one precedence-feasible period, so the statistics
        # are exercised (a random draw is mostly unplaceable in a fully mined schedule)
        sub = cand[:n_sub].tolist()
        store[p + "sub"] = np.array(sub, dtype=np.int32)
        sd, ex, cv = scenario_stats(inst, Schedule(full), sub, scen, sigma, net=True)
        store[p + "sub_scen_delta"], store[p + "sub_exp"], store[p + "sub_cvar"] = sd, ex, cv
        print(name, "feasible moves in subset:", int(np.isfinite(ex).sum()), file=sys.stderr)


class _RecordingEvaluator:
    """Wraps a reference ScheduleEvaluator for polish_schedule: returns the base value for the
    unmodified schedule and -inf for every option, so no move is ever accepted and one sweep
    visits every block's option list against the same schedule; records each option as the
    difference between the evaluated assignment and the base (hybrid.py:357-403)."""

    def __init__(self, base):
        self.base = np.asarray(base).copy()
        self.reassign, self.swap, self.other = [], [], []

    def npv_relaxed(self, sched):
        a = np.asarray(sched.assignment)
        d = np.nonzero(a != self.base)[0]
        if d.size == 0:
            return 0.0
        if d.size == 1:
            self.reassign.append((int(d[0]), int(a[d[0]])))
        elif (d.size == 2 and a[d[0]] == self.base[d[1]] and a[d[1]] == self.base[d[0]]
              and self.base[d[0]] != UNMINED and self.base[d[1]] != UNMINED):  # not a 1-1 exchange
            self.swap.append((int(d[0]), int(d[1])))
        else:
            self.other.append(tuple(int(x) for x in d))
        return -np.inf


def move_cases(store):
    """The reference's own move generation of polish_schedule (hybrid.py:348-403): for a fixed
    schedule, every reassign / unmine option (window + capacity) and every feasible pair swap it
    evaluates, recorded through _RecordingEvaluator.  Pins pp_eval_moves' feasibility rules."""
    for name, n, dims, T, S, cf in (("m27", 27, (3, 3, 3), 3, 2, 0.9), ("m32", 32, (4, 4, 2), 4, 3, 0.7),
                                    ("m512", 512, (8, 8, 8), 6, 4, 0.9), ("mC1", 4000, (20, 20, 10), 10, 10, 1.3)):
        inst = generate_synthetic(n, dims, T, 1, seed=170 + n, n_rock_types=1, capacity_factor=cf)
        scen = sample_lognormal(inst, S, 0.3, seed=171 + n)
        sigma = uncertainty_factors(inst, scen.grades)
        p = f"{name}_"
        store.update(flat(inst, p))
        store[p + "vmax"] = vmax_of(inst, scen)
        store[p + "sigma"] = sigma.sigma
        scheds = [greedy_initialize(inst, scen, sigma).assignment.copy(), full_greedy(inst)]
        rng = np.random.default_rng(n + 1)
        a = scheds[1].copy()
        a[rng.random(n) < 0.25] = UNMINED
        _precedence_repair_pass(inst, a)
        scheds.append(a)
        for k, base in enumerate(scheds):
            rec = _RecordingEvaluator(base)
            polish_schedule(inst, rec, Schedule(base.copy()), max_sweeps=1, pair_swaps=n <= 32)
            q = f"{p}{k}_"
            store[q + "assign"] = base.astype(np.int32)
            store[q + "reassign"] = np.array(rec.reassign, dtype=np.int32).reshape(-1, 2)
            store[q + "swap"] = np.array(rec.swap, dtype=np.int32).reshape(-1, 2)
            print(name, k, len(rec.reassign), len(rec.swap), len(rec.other), file=sys.stderr)


def vae_cases(store: dict) -> None:
    """vae_generate (vae.py:306-321) from a VAE trained by the reference on a small instance
    (train_on_instance, vae.py:295-303, a few epochs): the decoder's layers and normalisation, the
    prior samples z of each scenario (the substream of vae.py:288-290) and the decoded grades."""
    from pitplan.vae import VaeConfig, train_on_instance, vae_generate

    for name, n, dims, T, n_s, widths in (("v1", 240, (8, 6, 5), 6, 12, (16, 32, 48)),
                                           ("v2", 900, (15, 12, 5), 8, 40, (64, 128, 256))):
        inst = generate_synthetic(n, dims, T, 1, seed=5, n_rock_types=1)
        cfg = VaeConfig(latent_dim=8 if name == "v1" else 16, encoder_widths=tuple(reversed(widths)),
                        decoder_widths=widths, epochs=3, batch_size=16, seed=3)
        model = train_on_instance(inst, cfg, n_fields=64)
        out = vae_generate(model, n_s, seed=11)
        p = name + "_"
        store.update(flat(inst, p))
        store[p + "widths"] = np.array([cfg.latent_dim, *widths, n], dtype=np.int32)
        for k, layer in enumerate(model.decoder.layers):
            store[p + f"W{k}"] = layer.W
            store[p + f"b{k}"] = layer.b
        store[p + "norm_mean"] = model.norm_mean
        store[p + "norm_std"] = model.norm_std
        store[p + "z"] = np.stack([substream(11, "vae-gen", i).standard_normal((1, cfg.latent_dim))[0]
                                   for i in range(n_s)])
        store[p + "grades"] = out.grades
        print(name, n, n_s, file=sys.stderr)


def main():
    if sys.argv[1:] == ["vae"]:  # the VAE decode fixture only
        store: dict = {"numpy_version": np.bytes_(np.__version__)}
        vae_cases(store)
        np.savez_compressed(os.path.join(OUT, "vae.npz"), **store)
        return
    if sys.argv[1:] == ["stats"]:  # the k > 1 statistics fixture only
        store: dict = {"numpy_version": np.bytes_(np.__version__)}
        stats_cases(store)
        np.savez_compressed(os.path.join(OUT, "stats.npz"), **store)
        return
    if sys.argv[1:] == ["moves"]:  # the polish move-generation fixture only
        store = {"numpy_version": np.bytes_(np.__version__)}
        move_cases(store)
        np.savez_compressed(os.path.join(OUT, "moves.npz"), **store)
        return
    if sys.argv[1:] == ["price"]:  # regenerate only the pricing fixture
        store: dict = {"numpy_version": np.bytes_(np.__version__)}
        price_cases(store)
        np.savez_compressed(os.path.join(OUT, "price.npz"), **store)
        return
    store = {}
    small_cases(store)
    hand_cases(store)
    polish_cases(store)
    np.savez_compressed(os.path.join(OUT, "small.npz"), **store)
    store = {"numpy_version": np.bytes_(np.__version__)}
    config_case(store, "C1", 4000, (20, 20, 10), 10, 10, 1000, scen_subset=200)
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **store)
    store = {"numpy_version": np.bytes_(np.__version__)}
    config_case(store, "C2", 50000, (50, 50, 20), 15, 20, 16667)
    np.savez_compressed(os.path.join(OUT, "c2.npz"), **store)


if __name__ == "__main__":
    main()
