"""Repeat the shape parity cases many times with several live contexts; report mismatches."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from tests.test_gpu_parity import _rand_instance
from tests._fixtures import bm_from, load, tables_from
from paper_2511_18296_b200 import synth, evaluate as ev
from paper_2511_18296_b200.engine import Engine
from paper_2511_18296_b200.model import ScenarioTables, Schedule
from oracle import oracle

st = load("small")
keep = []
for case in range(0, 20, 3):  # live engines like the drop-in cache leaves behind
    p = f"kd{case}_"
    ev.evaluate_candidates_parallel(bm_from(st, p), Schedule(st[p + "assign"].astype(int)),
                                    [int(b) for b in st[p + "cand"]], tables_from(st, p), 0, True)
cases = [(1, 1), (3, 7), (7, 9), (9, 20), (16, 64), (17, 129), (32, 200), (33, 40), (40, 300), (5, 1000)]
bad_total = 0
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
t0 = time.time()
for it in range(iters):
    for T, S in cases:
        bm, vmax, sigma = _rand_instance(11 + T + S, T=T, S=S)
        rng = np.random.default_rng(T * 1000 + S)
        assign = synth.full_greedy(bm)
        assign[rng.random(assign.size) < 0.2] = -1
        cand = rng.integers(0, bm.n_blocks, size=157).astype(np.int32)
        cand[:5] = cand[5]
        eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
        o = oracle.Oracle(bm, vmax, sigma)
        for s in (None, S - 1):
            for net in (False, True):
                got = eng.eval_candidates(cand, s, net=net, trace=True, stats=True, scen=True)
                ref = o.eval_candidates(assign, cand, s, net=net, trace=True, stats=True, scen=True)
                for k in ("best_t", "best_val", "feasible", "trace_val", "trace_feas", "exp_delta", "cvar", "scen_delta"):
                    x, y = got[k], ref[k]
                    badm = ~((x == y) | (np.isnan(x) & np.isnan(y))) if x.dtype.kind == 'f' else (x != y)
                    if badm.any():
                        bad_total += 1
                        idx = np.argwhere(badm)
                        _, pm = eng.get_schedule()
                        again = eng.eval_candidates(cand, s, net=net, trace=True, stats=True, scen=True)[k]
                        rep = bool(np.all((again == y) | (np.isnan(again) & np.isnan(y))))
                        sp_ok = np.array_equal(eng.spatial(), o.spatial)
                        eng.set_schedule(assign)
                        again2 = eng.eval_candidates(cand, s, net=net, trace=True, stats=True, scen=True)[k]
                        rep2 = bool(np.all((again2 == y) | (np.isnan(again2) & np.isnan(y))))
                        e2 = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
                        again3 = e2.eval_candidates(cand, s, net=net, trace=True, stats=True, scen=True)[k]
                        e2.close()
                        rep3 = bool(np.all((again3 == y) | (np.isnan(again3) & np.isnan(y))))
                        rows = np.unique(idx[:, 0])
                        print(f"   spatial ok {sp_ok}; after set_schedule correct={rep2}; fresh engine correct={rep3};"
                              f" bad rows {rows[:20].tolist()} (of {rows.size}) blocks {cand[rows[:20]].tolist()}", flush=True)
                        print(f"it{it} T={T} S={S} s={s} net={net} {k}: {badm.sum()} bad; first {idx[:3].tolist()}"
                              f" got {x[tuple(idx[0])]!r} ref {y[tuple(idx[0])]!r}; pm ok {np.array_equal(pm, o.period_mass(assign))};"
                              f" immediate rerun correct={rep}", flush=True)
                        break
        eng.close()
print(f"done {iters} iters, {bad_total} mismatching calls, {time.time()-t0:.1f}s")
