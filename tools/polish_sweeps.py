"""Per-sweep cost of the native single-block polish sweep (pp_polish_sweep) at a synth config:
time, device evaluations (pp_npv_moves calls) and accepted moves per sweep, from the greedy start
until a sweep accepts nothing.

    python tools/polish_sweeps.py [C1|C2] [max_sweeps]
"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2511_18296_b200 import evaluate as dropin, synth
from paper_2511_18296_b200.model import ScenarioTables, scenario_values

which = sys.argv[1] if len(sys.argv) > 1 else "C2"
nsw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
c = synth.build_config(which)
bm = c["bm"]
tb = ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"], grades=c["grades"])
a = synth.greedy_initialize(bm, c["grades"], c["sigma"]).astype(np.int64)
ev = dropin.ScheduleEvaluator(bm, tb, True)
e = dropin._entry(bm)
dropin._bind_scenarios(e, tb, True, None)
eng = e.engine
cur = float(eng.npv_relaxed(a[None, :], use_sigma=True)[0])
load = np.array([bm.mass[a == t].sum() for t in range(bm.n_periods)])
a32 = a.astype(np.int32)
for k in range(nsw):
    before = a32.copy()
    t0 = time.perf_counter()
    cur, improved, calls = eng.polish_sweep(a32, load, cur, use_sigma=True, chunk0=dropin._POLISH_CHUNK,
                                            chunk_max=dropin._POLISH_CHUNK_MAX)
    dt = time.perf_counter() - t0
    print(f"sweep {k}: {dt:.3f} s, {calls} device evaluations, {int(np.sum(before != a32))} blocks moved, "
          f"npv {cur:.6f}", flush=True)
    if not improved:
        break
