"""Time the reference's own evaluate_candidates_parallel (pure Python) on the C2 batch.

Runs only where the reference source exists (the build container, not the GPU box); the
numbers are recorded in DESIGN.md beside the device and oracle-port timings."""
import os, sys, time
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
from pitplan.blockmodel import generate_synthetic
from pitplan.evaluate import ScheduleEvaluator, Schedule, evaluate_candidates_parallel
from pitplan.hybrid import HybridSearch
from pitplan.rng import substream
from pitplan.scenarios import sample_lognormal
from pitplan.uncertainty import uncertainty_factors

t0 = time.perf_counter()
inst = generate_synthetic(50000, (50, 50, 20), 15, 1, seed=1, n_rock_types=1, capacity_factor=1.3)
scen = sample_lognormal(inst, 20, 0.3, seed=2)
sigma = uncertainty_factors(inst, scen.grades)
print(f"instance + scenarios: {time.perf_counter() - t0:.1f} s")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18296_b200 import synth
assign = synth.full_greedy(synth.build_config("C2")["bm"]).astype(int)
cand = substream(3, "cand").integers(0, 50000, size=16667).tolist()
sched = Schedule(assign)
for w in (1, os.cpu_count()):
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        evaluate_candidates_parallel(inst, sched, cand, scen, None, sigma, worker_count=w, net_mining_cost=True)
        ts.append(time.perf_counter() - t0)
    print(f"reference evaluate_candidates_parallel, worker_count={w}: best of 2 = {min(ts):.3f} s per 250k-move batch")
ev = ScheduleEvaluator(inst, scen, sigma)
t0 = time.perf_counter(); ev.npv_relaxed(sched); t1 = time.perf_counter()
print(f"reference ScheduleEvaluator.npv_relaxed (cold cache): {t1 - t0:.3f} s")
