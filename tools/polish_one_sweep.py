"""One C2 polish sweep from the greedy start (a fixed workload for ncu launch lists)."""
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2511_18296_b200 import evaluate as dropin, synth
from paper_2511_18296_b200.model import ScenarioTables, scenario_values
c = synth.build_config("C2"); bm = c["bm"]
tb = ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"], grades=c["grades"])
a = synth.greedy_initialize(bm, c["grades"], c["sigma"]).astype(np.int64)
e = dropin._entry(bm); dropin._bind_scenarios(e, tb, True, None); eng = e.engine
cur = float(eng.npv_relaxed(a[None, :], use_sigma=True)[0])
load = np.array([bm.mass[a == t].sum() for t in range(bm.n_periods)])
a32 = a.astype(np.int32)
eng.polish_sweep(a32, load, cur, use_sigma=True, chunk0=64, chunk_max=128)
