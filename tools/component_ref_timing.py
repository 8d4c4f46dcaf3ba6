"""Reference (pure Python) time of the widened components on the golden-fixture inputs.

Runs only where the reference source exists (the build container): lns_repair on C1 (destroy +
40 insertion rounds), polish_schedule on the 512-block case, price_column on the 4,000-block
pricing case.  The device drop-ins are timed on the same inputs by tools/component_timing.py."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden"))
import make_golden as mg  # puts the reference on sys.path; its helpers build the fixture inputs
from pitplan.colgen import DualPrices, price_column, _enpv_adjusted
from pitplan.evaluate import Schedule, ScheduleEvaluator
from pitplan.hybrid import _precedence_repair_pass, greedy_initialize, lns_repair, polish_schedule

def best_of(fn, n=2):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return min(ts)

# lns_repair, C1 (tests/golden/make_golden.py config_case: destroy_in[0], 40 rounds)
inst = mg.generate_synthetic(4000, (20, 20, 10), 10, 1, seed=1, n_rock_types=1, capacity_factor=1.3)
scen = mg.sample_lognormal(inst, 10, 0.3, seed=2)
sigma = mg.uncertainty_factors(inst, scen.grades)
full = mg.full_greedy(inst)
tm = int(full.max())
a = full.copy(); a[a == tm] = tm - 1
t = best_of(lambda: lns_repair(inst, Schedule(a.copy()), [], scen, sigma, max_iters=40, destroy_fraction=0.1), 1)
print(f"lns_repair C1 (4,000 blocks, 40 rounds): {t:.3f} s")

# polish_schedule, p512 (make_golden.py polish_cases)
inst = mg.generate_synthetic(512, (8, 8, 8), 6, 1, seed=70 + 512, n_rock_types=1, capacity_factor=0.9)
scen = mg.sample_lognormal(inst, 4, 0.3, seed=71 + 512)
sigma = mg.uncertainty_factors(inst, scen.grades)
ev = ScheduleEvaluator(inst, scen, sigma)
s0 = greedy_initialize(inst, scen, sigma).assignment.copy()
t = best_of(lambda: polish_schedule(inst, ev, Schedule(s0.copy()), max_sweeps=2), 1)
print(f"polish_schedule p512 (512 blocks, 2 sweeps, greedy start): {t:.3f} s")

# price_column, qC1big (make_golden.py price_cases)
n, T = 4000, 10
inst = mg.generate_synthetic(n, (20, 20, 10), T, 1, seed=90 + n, n_rock_types=1, capacity_factor=0.6)
scen = mg.sample_lognormal(inst, 5, 0.3, seed=91 + n)
sigma = mg.uncertainty_factors(inst, scen.grades)
rng = np.random.default_rng(n + T)
enpv0 = _enpv_adjusted(inst, scen, sigma)
duals = DualPrices(block=np.abs(rng.normal(0, 0.3, n)) * np.abs(enpv0).mean(),
                   capacity=np.abs(rng.normal(0, 0.5, T)) * np.abs(enpv0).mean() / inst.masses().mean(),
                   convexity=np.zeros(1))
t = best_of(lambda: price_column(inst, duals, scen, sigma, 0, (5, "price", n), node_cap=10 ** 7, noise=0.2), 1)
print(f"price_column qC1big (4,000 blocks, 1,093 picks): {t:.3f} s")
