import ctypes, sys, numpy as np
sys.path.insert(0, '.')
from paper_2511_18296_b200 import _lib
lib = _lib.load(sys.argv[1]); _lib._lib = lib
lib.pp_debug_npv_probe.argtypes = [ctypes.c_void_p]
from bench import build_inputs
from paper_2511_18296_b200.engine import Engine
c = build_inputs("C2")
eng = Engine.from_tables(c["bm"], c["tables"])
for _ in range(3):
    eng.npv_relaxed(c["assign"])
pr = np.zeros(8, np.uint64); lib.pp_debug_npv_probe(pr.ctypes.data); pr = pr.astype(np.int64)
print("phases (us): compaction %.1f, cost+sort+prep %.1f, greedy %.1f" % ((pr[1] - pr[0]) / 1e3, (pr[3] - pr[1]) / 1e3, (pr[4] - pr[3]) / 1e3))
