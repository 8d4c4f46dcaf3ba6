"""polish_schedule drop-in at C2 scale: speculative chunk sizes give the same schedule; time per
sweep for each.  Needs the reference's pip install under baseline/_ref (greedy start, evaluator).

    python tools/polish_chunk.py --blocks 50000 --dims 50 50 20 --periods 15 --scen 20
"""
import argparse, hashlib, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import pitplan.hybrid as H  # noqa: E402
from pitplan.blockmodel import generate_synthetic  # noqa: E402
from pitplan.scenarios import sample_lognormal  # noqa: E402
from pitplan.uncertainty import uncertainty_factors  # noqa: E402
from paper_2511_18296_b200 import evaluate as ev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=4000)
ap.add_argument("--dims", type=int, nargs=3, default=(20, 20, 10))
ap.add_argument("--periods", type=int, default=10)
ap.add_argument("--scen", type=int, default=10)
ap.add_argument("--sweeps", type=int, default=1)
ap.add_argument("--chunks", type=int, nargs="+", default=[1, 16, 64])
a = ap.parse_args()
inst = generate_synthetic(a.blocks, tuple(a.dims), a.periods, 1, seed=1, n_rock_types=1)
scen = sample_lognormal(inst, a.scen, 0.3, seed=2)
sigma = uncertainty_factors(inst, scen.grades)
start = H.greedy_initialize(inst, scen, sigma, 0)
E = ev.ScheduleEvaluator(inst, scen, sigma)
ref = None
for c in a.chunks:
    ev._POLISH_CHUNK = c
    ev._POLISH_CHUNK_MAX = max(c, ev._POLISH_CHUNK_MAX) if c > 1 else 1
    t0 = time.perf_counter()
    out = ev.polish_schedule(inst, E, start.copy(), max_sweeps=a.sweeps)
    dt = time.perf_counter() - t0
    d = hashlib.sha256(np.asarray(out.assignment, "<i8").tobytes()).hexdigest()[:16]
    ref = ref or d
    changed = int(np.sum(np.asarray(out.assignment) != np.asarray(start.assignment)))
    print(f"[polish] chunk {c}: {dt:.2f} s for {a.sweeps} sweep(s), changed {changed} blocks, digest {d}, same {d == ref}")
    ev._POLISH_CHUNK_MAX = 128
