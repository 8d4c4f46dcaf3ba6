import sys, numpy as np
sys.path.insert(0, '.')
from tests.test_gpu_parity import _rand_instance
from paper_2511_18296_b200 import synth
from paper_2511_18296_b200.engine import Engine
from paper_2511_18296_b200.model import ScenarioTables
from oracle import oracle
T, S, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
bm, vmax, sigma = _rand_instance(11 + T + S, T=T, S=S)
rng = np.random.default_rng(T * 1000 + S)
assign = synth.full_greedy(bm)
assign[rng.random(assign.size) < 0.2] = -1
cand = rng.integers(0, bm.n_blocks, size=157).astype(np.int32)
cand[:5] = cand[5]
o = oracle.Oracle(bm, vmax, sigma)
refs = {}
bad = 0
eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
for it in range(N):
    if it % 10 == 0:
        eng.close(); eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
    s = [None, S - 1][it % 2]; net = bool((it // 2) % 2); scen = bool((it // 4) % 2)
    key = (s, net, scen)
    if key not in refs:
        refs[key] = o.eval_candidates(assign, cand, s, net=net, stats=True, scen=scen)
    got = eng.eval_candidates(cand, s, net=net, stats=True, scen=scen)
    ref = refs[key]
    for k in ("exp_delta", "cvar") + (("scen_delta",) if scen else ()):
        x, y = got[k], ref[k]
        m = ~((x == y) | (np.isnan(x) & np.isnan(y)))
        if m.any():
            bad += 1
            idx = np.argwhere(m)
            print(f"it{it} key={key} {k}: {m.sum()} bad, rows {sorted(set(idx[:,0].tolist()))[:10]} first {idx[0].tolist()} got {x[tuple(idx[0])]!r} ref {y[tuple(idx[0])]!r}")
            break
print("bad calls", bad, "of", N)
