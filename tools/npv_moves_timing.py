"""Per-call time of pp_npv_moves at C2 in the polish pattern: a base that drifts by one accepted
move per call, M one-block variants per call.  Prints the host wall time per call (median)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2511_18296_b200 import synth
from paper_2511_18296_b200.engine import Engine
from paper_2511_18296_b200.model import ScenarioTables, scenario_values

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = synth.build_config(cfg)
bm = c["bm"]
eng = Engine.from_tables(bm, ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"]))
a = synth.greedy_initialize(bm, c["grades"], c["sigma"]).astype(np.int32)
rng = np.random.default_rng(0)
B, T = bm.n_blocks, bm.n_periods
for M in (16, 100, 400):
    ts = []
    for it in range(30):
        blocks = np.repeat(rng.integers(0, B, M // 8 + 1), 8)[:M].astype(np.int32)
        periods = rng.integers(-1, T, M).astype(np.int32)
        t0 = time.perf_counter()
        eng.npv_moves(a, blocks, periods)
        ts.append(time.perf_counter() - t0)
        b = int(rng.integers(0, B))
        a[b] = int(rng.integers(-1, T))  # one accepted move
    print(f"M={M}: median {1e3 * np.median(ts[3:]):.3f} ms per call, min {1e3 * min(ts[3:]):.3f} ms")
