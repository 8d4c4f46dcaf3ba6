"""Device drop-in time of the widened components on the golden-fixture inputs (the reference's
Python times on the same inputs come from tools/component_ref_timing.py)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from tests._fixtures import bm_from, config, load, tables_from
from paper_2511_18296_b200 import evaluate as dropin
from paper_2511_18296_b200.engine import Engine
from paper_2511_18296_b200.model import ScenarioTables, Schedule

def best_of(fn, n=3):
    fn()  # warm (context, tables)
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return min(ts)

st = load("c1"); c = config("C1")
tables = ScenarioTables(c["vmax"], c["sigma"], grades=st["C1_grades"])
a0 = st["C1_destroy_in"][0]
out = None
def lns():
    global out
    out = dropin.lns_repair(c["bm"], Schedule(a0.copy()), [], tables, True, max_iters=40, destroy_fraction=0.1)
t = best_of(lns)
print(f"lns_repair C1 (4,000 blocks, 40 rounds): {t * 1e3:.1f} ms  (matches reference: {np.array_equal(out.assignment, st['C1_lns'])})")

sm = load("small"); p = "p512_"
bm = bm_from(sm, p); tb = tables_from(sm, p)
ev = dropin.ScheduleEvaluator(bm, tb, True)
def pol():
    global out
    out = dropin.polish_schedule(bm, ev, Schedule(sm[p + "start"][0].copy()), max_sweeps=int(sm[p + "sweeps"]))
t = best_of(pol)
print(f"polish_schedule p512 (512 blocks, 2 sweeps, greedy start): {t * 1e3:.1f} ms  (matches reference: {np.array_equal(out.assignment, sm[p + 'out'][0])})")

pr = load("price"); p = "qC1big_"
eng = Engine.from_tables(bm_from(pr, p), None)
res = None
def price():
    global res
    res = eng.price_greedy(pr[p + "score"], pr[p + "cap"], int(pr[p + "node_cap"]))
t = best_of(price)
print(f"price_column greedy qC1big (4,000 blocks, 1,093 picks): {t * 1e3:.2f} ms  (matches reference: {np.array_equal(res[0], pr[p + 'assign'])})")
dropin.clear_cache()
