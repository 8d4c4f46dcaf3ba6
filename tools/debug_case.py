import sys, numpy as np
sys.path.insert(0, '.')
from tests.test_gpu_parity import _rand_instance
from paper_2511_18296_b200 import synth
from paper_2511_18296_b200.engine import Engine
from paper_2511_18296_b200.model import ScenarioTables
from oracle import oracle
T, S = int(sys.argv[1]), int(sys.argv[2])
bm, vmax, sigma = _rand_instance(11 + T + S, T=T, S=S)
rng = np.random.default_rng(T * 1000 + S)
assign = synth.full_greedy(bm)
assign[rng.random(assign.size) < 0.2] = -1
cand = rng.integers(0, bm.n_blocks, size=157).astype(np.int32)
cand[:5] = cand[5]
eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
o = oracle.Oracle(bm, vmax, sigma)
a, pm = eng.get_schedule()
print("pm equal", np.array_equal(pm, o.period_mass(assign)), pm[:5], o.period_mass(assign)[:5])
for s in (None, S - 1):
    for net in (False, True):
        for stats in (False, True, "scen"):
            got = eng.eval_candidates(cand, s, net=net, trace=True, stats=bool(stats), scen=stats == "scen")
            ref = o.eval_candidates(assign, cand, s, net=net, trace=True, stats=bool(stats), scen=stats == "scen")
            for k in ("best_t", "best_val", "feasible", "trace_val", "trace_feas") + (("exp_delta", "cvar") if stats else ()) + (("scen_delta",) if stats == "scen" else ()):
                x, y = got[k], ref[k]
                bad = ~((x == y) | (np.isnan(x) & np.isnan(y))) if x.dtype.kind == 'f' else (x != y)
                if bad.any():
                    idx = np.argwhere(bad)[:3]
                    print(f"s={s} net={net} stats={stats} {k}: {bad.sum()} bad, first {idx.tolist()} got {x[tuple(idx[0])]} ref {y[tuple(idx[0])]}")
print("done")
