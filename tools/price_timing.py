"""pp_price_greedy timing on the golden pricing cases (and the oracle's sequential scan beside it)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from tests._fixtures import bm_from, load
from paper_2511_18296_b200.engine import Engine
from oracle import oracle
st = load("price")
for name in ("qC1", "qC1big"):
    p = f"{name}_"
    bm = bm_from(st, p)
    eng = Engine.from_tables(bm, None)
    args = (st[p + "score"], st[p + "cap"], int(st[p + "node_cap"]))
    eng.price_greedy(*args)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); a, ex = eng.price_greedy(*args); ts.append(time.perf_counter() - t0)
    o = oracle.Oracle(bm)
    t0 = time.perf_counter(); ar, exr = o.price_greedy(*args); to = time.perf_counter() - t0
    print(f"{name}: B={bm.n_blocks} picks={int((a >= 0).sum())} expansions={ex}: device {np.median(ts) * 1e3:.2f} ms, "
          f"oracle (C, 1 core) {to * 1e3:.2f} ms, equal={np.array_equal(a, ar) and ex == exr}")
    eng.close()
