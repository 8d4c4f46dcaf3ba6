"""Feasible (candidate, period) pairs and precedence-feasible pairs per config (sizing the statistics work)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from bench import build_inputs
from paper_2511_18296_b200.engine import Engine
for name in sys.argv[1:] or ["C2", "C3"]:
    c = build_inputs(name)
    eng = Engine.from_tables(c["bm"], c["tables"], c["assign"])
    r = eng.eval_candidates(c["cand"], None, net=True, trace=True)
    feas = int(r["trace_feas"].sum())
    print(name, "C", c["C"], "T", c["T"], "S", c["S"], "feasible pairs", feas, "feasible cands", int(r["feasible"].sum()), flush=True)
    eng.close()
