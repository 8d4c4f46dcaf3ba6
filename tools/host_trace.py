"""PP_TRACE_HOST=1 python tools/host_trace.py: per-phase host time of the C2 e2e calls."""
import os, sys, time, numpy as np
sys.path.insert(0, '.')
from bench import build_inputs
from paper_2511_18296_b200.engine import Engine, PinnedPool
c = build_inputs("C2")
eng = Engine.from_tables(c["bm"], c["tables"], c["assign"])
C, T = c["C"], c["T"]
pool = PinnedPool()
ha = pool.empty(c["bm"].n_blocks, np.int32); ha[:] = c["assign"]
hc = pool.empty(C, np.int32); hc[:] = c["cand"]
ho = {"best_t": pool.empty(C, np.int32), "best_val": pool.empty(C, np.float64), "feasible": pool.empty(C, np.uint8),
      "pair_cand": pool.empty(C * T, np.int32), "pair_period": pool.empty(C * T, np.int32),
      "pair_exp": pool.empty(C * T, np.float64), "pair_cvar": pool.empty(C * T, np.float64), "n_pairs": pool.empty(1, np.int32)}
for i in range(30):
    if i == 27: print("---- traced ----", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    eng.set_schedule(ha)
    t1 = time.perf_counter()
    eng.eval_candidates(hc, None, net=True, pairs=True, out=ho, validate=False)
    t2 = time.perf_counter()
    if i >= 27: print(f"python: set_schedule {1e6*(t1-t0):.1f} us, eval {1e6*(t2-t1):.1f} us", file=sys.stderr, flush=True)
