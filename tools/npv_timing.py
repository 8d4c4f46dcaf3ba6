"""Relaxed NPV (population fitness) timing at C2: device vs the oracle port."""
import sys, time, numpy as np
sys.path.insert(0, '.')
from bench import build_inputs
from paper_2511_18296_b200.engine import Engine
from oracle import oracle
c = build_inputs("C2")
bm = c["bm"]
eng = Engine.from_tables(bm, c["tables"])
rng = np.random.default_rng(0)
base = c["assign"]
for P in (1, 16, 64):
    pop = np.stack([base] * P)
    for k in range(1, P):  # perturbed copies: some blocks moved to a neighbouring period
        idx = rng.choice(bm.n_blocks, 200, replace=False)
        pop[k, idx] = np.clip(pop[k, idx] + rng.integers(-1, 2, 200), -1, bm.n_periods - 1)
    eng.npv_relaxed(pop)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); eng.npv_relaxed(pop); ts.append(time.perf_counter() - t0)
    print(f"device npv_relaxed P={P}: {1e3 * min(ts):.3f} ms ({1e3 * min(ts) / P:.3f} ms/schedule)")
oracle.build()
o = oracle.Oracle(bm, c["tables"].vmax, c["tables"].sigma)
t0 = time.perf_counter(); o.npv_relaxed(base, bm.plant_hours, bm.mode_rates[0]); t1 = time.perf_counter()
print(f"oracle port (1 core) npv_relaxed: {1e3 * (t1 - t0):.1f} ms/schedule")
# exact move values: one block's options, two periods re-solved per option
blk = int(np.nonzero(base >= 0)[0][0])
opts = np.array([t for t in range(-1, bm.n_periods) if t != base[blk]], dtype=np.int32)
eng.npv_moves(base, np.full(opts.size, blk), opts)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); eng.npv_moves(base, np.full(opts.size, blk), opts); ts.append(time.perf_counter() - t0)
print(f"device npv_moves ({opts.size} options of one block, incl. the base schedule): {1e3 * min(ts):.3f} ms")
