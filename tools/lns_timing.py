"""lns_repair at C2 (50k blocks): the device-resident graph loop (pp_lns_insert) against the
host-driven loop of the same drop-in (one evaluation call per round).  The greedy schedule's last
(half-full) period is unmined and its ~2,300 blocks are the unassigned pool.

    python tools/lns_timing.py [iters]
"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2511_18296_b200 import evaluate as dropin, synth
from paper_2511_18296_b200.model import ScenarioTables, Schedule, scenario_values

iters = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 300
c = synth.build_config("C2")
bm = c["bm"]
tables = ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"], grades=c["grades"])
a = np.asarray(c["assign"], dtype=np.int64).copy()
last = int(a.max())  # the greedy's last period, half full: its blocks go back to the pool
chunk = np.nonzero(a == last)[0]
a[chunk] = -1
run = lambda: dropin.lns_repair(bm, Schedule(a.copy()), chunk.tolist(), tables, True, max_iters=iters)
out_g = run()
ts = []
for _ in range(3):
    t0 = time.perf_counter(); out_g = run(); ts.append(time.perf_counter() - t0)
tg = min(ts)
dropin._LNS_GRAPH_WMAX = 0
out_h = run()
ts = []
for _ in range(3):
    t0 = time.perf_counter(); out_h = run(); ts.append(time.perf_counter() - t0)
th = min(ts)
assert np.array_equal(out_g.assignment, out_h.assignment)
rounds = int(np.sum((a < 0) & (out_g.assignment >= 0)))  # one pool block inserted per round
print(f"C2 lns_repair, pool {chunk.size}, max_iters {iters}, {rounds} rounds run: graph {tg * 1e3:.1f} ms ({tg / max(rounds, 1) * 1e6:.1f} us/round), "
      f"host loop {th * 1e3:.1f} ms ({th / max(rounds, 1) * 1e6:.1f} us/round), identical result")
