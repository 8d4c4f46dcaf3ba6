"""cProfile of the polish_schedule drop-in on p512."""
import cProfile, pstats, sys
sys.path.insert(0, '.')
from tests._fixtures import bm_from, load, tables_from
from paper_2511_18296_b200 import evaluate as dropin
from paper_2511_18296_b200.model import Schedule
sm = load("small"); p = "p512_"
bm = bm_from(sm, p); tb = tables_from(sm, p)
ev = dropin.ScheduleEvaluator(bm, tb, True)
run = lambda: dropin.polish_schedule(bm, ev, Schedule(sm[p + "start"][0].copy()), max_sweeps=int(sm[p + "sweeps"]))
run()
pr = cProfile.Profile(); pr.enable(); run(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
