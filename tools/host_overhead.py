"""Host-side cost of the C-ABI calls (C2), to see where the end-to-end time goes."""
import sys, time, ctypes, numpy as np, torch
sys.path.insert(0, '.')
from bench import build_inputs
from paper_2511_18296_b200.engine import Engine, PinnedPool
from paper_2511_18296_b200 import _lib
c = build_inputs("C2")
eng = Engine.from_tables(c["bm"], c["tables"], c["assign"])
C, T = c["C"], c["T"]
pool = PinnedPool()
ha = pool.empty(c["bm"].n_blocks, np.int32); ha[:] = c["assign"]
hc = pool.empty(C, np.int32); hc[:] = c["cand"]
ho = {"best_t": pool.empty(C, np.int32), "best_val": pool.empty(C, np.float64), "feasible": pool.empty(C, np.uint8),
      "pair_cand": pool.empty(C * T, np.int32), "pair_period": pool.empty(C * T, np.int32),
      "pair_exp": pool.empty(C * T, np.float64), "pair_cvar": pool.empty(C * T, np.float64), "n_pairs": pool.empty(1, np.int32)}
lib = _lib.load()
def med(fn, n=300):
    ts = []
    for i in range(n + 20):
        t0 = time.perf_counter(); fn(); t1 = time.perf_counter()
        if i >= 20: ts.append(t1 - t0)
    return np.median(ts) * 1e6
print("ctypes pp_abi_version      %.1f us" % med(lambda: lib.pp_abi_version()))
print("pp_synchronize (idle)      %.1f us" % med(lambda: lib.pp_synchronize(eng._h, None)))
print("set_schedule (pinned)      %.1f us" % med(lambda: eng.set_schedule(ha)))
print("set_schedule+sync          %.1f us" % med(lambda: (eng.set_schedule(ha), lib.pp_synchronize(eng._h, None))))
print("eval best only (no pm)     %.1f us" % med(lambda: eng.eval_candidates(hc, None, net=True, out=ho, validate=False)))
print("eval pairs (no pm)         %.1f us" % med(lambda: eng.eval_candidates(hc, None, net=True, pairs=True, out=ho, validate=False)))
print("set+eval pairs (bench)     %.1f us" % med(lambda: (eng.set_schedule(ha), eng.eval_candidates(hc, None, net=True, pairs=True, out=ho, validate=False))))
x = torch.empty(C * 13 // 8 + 1, dtype=torch.float64, device="cuda"); hx = torch.from_numpy(pool.empty(x.numel(), np.float64))
print("raw D2H 217KB + sync       %.1f us" % med(lambda: (hx.copy_(x, non_blocking=True), torch.cuda.synchronize())))
y = torch.empty(20000 * 3, dtype=torch.float64, device="cuda"); hy = torch.from_numpy(pool.empty(y.numel(), np.float64))
print("raw D2H 480KB + sync       %.1f us" % med(lambda: (hy.copy_(y, non_blocking=True), torch.cuda.synchronize())))
