"""Where the end-to-end (host-buffer) time of one C2 batch goes."""
import sys, time, numpy as np, torch
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
      "exp_delta": pool.empty((C, T), np.float64), "cvar": pool.empty((C, T), np.float64)}
flush = torch.empty(256 << 18, dtype=torch.int32, device="cuda")
def med(fn, n=200):
    ts = []
    for i in range(n + 10):
        flush.fill_(i); torch.cuda.synchronize()
        t0 = time.perf_counter(); fn(); t1 = time.perf_counter()
        if i >= 10: ts.append(t1 - t0)
    return np.median(ts) * 1e6
print("set_schedule            %.1f us" % med(lambda: eng.set_schedule(ha)))
print("set_schedule(noval)     %.1f us" % med(lambda: eng.set_schedule(ha, validate=False) if 'validate' in Engine.set_schedule.__code__.co_varnames else eng.set_schedule(ha)))
print("eval best only          %.1f us" % med(lambda: eng.eval_candidates(hc, None, net=True, out=ho, validate=False)))
print("eval + stats            %.1f us" % med(lambda: eng.eval_candidates(hc, None, net=True, stats=True, out=ho, validate=False)))
print("both (bench e2e)        %.1f us" % med(lambda: (eng.set_schedule(ha), eng.eval_candidates(hc, None, net=True, stats=True, out=ho, validate=False))))
x = torch.empty(C * T * 2, dtype=torch.float64, device="cuda"); hx = pool.empty(C * T * 2, np.float64)
hxt = torch.from_numpy(hx)
print("raw D2H 4MB             %.1f us" % med(lambda: (hxt.copy_(x, non_blocking=True), torch.cuda.synchronize())))
