import sys; sys.path.insert(0, '.')
import numpy as np
from tests._fixtures import bm_from, load, tables_from
from paper_2511_18296_b200.engine import Engine
st = load("moves")
for name in sys.argv[1:]:
    p = f"{name}_"
    bm = bm_from(st, p)
    eng = Engine.from_tables(bm, tables_from(st, p))
    B, T = bm.n_blocks, bm.n_periods
    for k in range(3):
        q = f"{p}{k}_"
        eng.set_schedule(st[q + "assign"])
        bb = np.repeat(np.arange(B), T + 1).astype(np.int32)
        tt = np.tile(np.arange(-1, T), B).astype(np.int32)
        r = eng.eval_moves(bb, tt, "reassign", net=True)
        f = r["feasible"] == 1
        bad = np.nonzero(f & ~np.isfinite(r["delta"]))[0]
        print(name, k, "feasible", int(f.sum()), "nonfinite feasible deltas", bad.size, bad[:5].tolist(), r["delta"][bad[:5]].tolist())
        r2 = eng.eval_moves(bb, tt, "reassign", net=True)
        print("   repeat identical:", np.array_equal(r2["delta"], r["delta"], equal_nan=True))
    eng.close()
