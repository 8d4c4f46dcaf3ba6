"""Fixed cost of pp_lns_insert / lns_repair calls at C2 (per-call graph build vs rounds)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2511_18296_b200 import evaluate as dropin, synth
from paper_2511_18296_b200.model import ScenarioTables, Schedule, scenario_values, rook_neighbor_map, rook_padded
c = synth.build_config("C2"); bm = c["bm"]
tables = ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"], grades=c["grades"])
a = np.asarray(c["assign"], dtype=np.int64).copy()
last = int(a.max()); chunk = np.nonzero(a == last)[0]; a[chunk] = -1
e = dropin._entry(bm); dropin._bind_scenarios(e, tables, True, None)
eng = e.engine
eng.set_rook(*dropin._rook_csr(rook_padded(rook_neighbor_map(bm), bm.n_blocks)))
mg = np.asarray(c["grades"]).mean(axis=0)
pool = np.zeros(bm.n_blocks, np.uint8); pool[chunk] = 1
for it in (1, 1, 1, 10, 10, 100):
    t0 = time.perf_counter(); out = eng.lns_insert(a, pool, mg, max_iters=it); t1 = time.perf_counter()
    print(f"lns_insert max_iters={it}: {1e3*(t1-t0):.2f} ms, rounds {out[2]}")
for it in (1, 10):
    t0 = time.perf_counter(); dropin.lns_repair(bm, Schedule(a.copy()), chunk.tolist(), tables, True, max_iters=it); t1 = time.perf_counter()
    print(f"lns_repair max_iters={it}: {1e3*(t1-t0):.2f} ms")
