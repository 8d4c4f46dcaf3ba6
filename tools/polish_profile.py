"""cProfile of the polish_schedule drop-in: p512 (golden fixture) or a synth config (C1/C2).

    python tools/polish_profile.py [p512|C1|C2] [sweeps]
"""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2511_18296_b200 import evaluate as dropin, synth
from paper_2511_18296_b200.model import ScenarioTables, Schedule, scenario_values

which = sys.argv[1] if len(sys.argv) > 1 else "p512"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if which == "p512":
    from tests._fixtures import bm_from, load, tables_from
    sm = load("small"); p = "p512_"
    bm = bm_from(sm, p); tb = tables_from(sm, p)
    start = sm[p + "start"][0].astype(np.int64)
else:
    c = synth.build_config(which)
    bm = c["bm"]
    tb = ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"], grades=c["grades"])
    start = synth.greedy_initialize(bm, c["grades"], c["sigma"]).astype(np.int64)
ev = dropin.ScheduleEvaluator(bm, tb, True)
run = lambda: dropin.polish_schedule(bm, ev, Schedule(start.copy()), max_sweeps=sweeps)
run()
t0 = time.perf_counter(); out = run(); print(f"[polish] {which}: {time.perf_counter() - t0:.3f} s for {sweeps} sweep(s), "
                                           f"changed {int(np.sum(out.assignment != start))}")
pr = cProfile.Profile(); pr.enable(); run(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
