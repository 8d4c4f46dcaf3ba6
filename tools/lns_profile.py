"""cProfile of the lns_repair drop-in on C1 (destroy + 40 insertion rounds)."""
import cProfile, pstats, sys
import numpy as np
sys.path.insert(0, '.')
from tests._fixtures import config, load
from paper_2511_18296_b200 import evaluate as dropin
from paper_2511_18296_b200.model import ScenarioTables, Schedule
st = load("c1"); c = config("C1")
tables = ScenarioTables(c["vmax"], c["sigma"], grades=st["C1_grades"])
a0 = st["C1_destroy_in"][0]
run = lambda: dropin.lns_repair(c["bm"], Schedule(a0.copy()), [], tables, True, max_iters=40, destroy_fraction=0.1)
run()
pr = cProfile.Profile(); pr.enable(); run(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
