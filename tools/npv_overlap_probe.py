"""Kernel spans of pp_npv_moves calls in the polish pattern (a base drifting by one accepted move
per call, so each call starts with the one-block update k_s2_apply_one): per call the earliest
start / latest end of k_s2_apply_one, k_s2_varcost, k_s2_chain and the final accumulation, from
globaltimer probes (library built with -DPP_EVAL_PROBE: tools/build_probe.sh).

    python tools/npv_overlap_probe.py tools/libprobe.so
"""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2511_18296_b200 import _lib
lib = _lib.load(sys.argv[1]); _lib._lib = lib
lib.pp_debug_kspan.argtypes = [ctypes.c_void_p, ctypes.c_int]
from paper_2511_18296_b200 import synth
from paper_2511_18296_b200.engine import Engine
from paper_2511_18296_b200.model import ScenarioTables, scenario_values
c = synth.build_config("C2"); bm = c["bm"]
eng = Engine.from_tables(bm, ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"]))
a = synth.greedy_initialize(bm, c["grades"], c["sigma"]).astype(np.int32)
rng = np.random.default_rng(0)
B, T = bm.n_blocks, bm.n_periods
rows = []
buf = np.zeros(16, np.uint64)
for it in range(60):
    b0 = int(rng.integers(0, B - 8))
    blocks = np.repeat(np.arange(b0, b0 + 4, dtype=np.int32), T)
    periods = np.tile(np.arange(-1, T - 1, dtype=np.int32), 4)
    lib.pp_debug_kspan(None, 1)
    eng.npv_moves(a, blocks, periods)
    lib.pp_debug_kspan(buf.ctypes.data, 0)
    sp = buf.reshape(8, 2).astype(np.int64)
    if it >= 5 and sp[0, 1] > 0:
        t0 = sp[0, 0]
        rows.append([(sp[k, 0] - t0) / 1e3 if sp[k, 1] > 0 else np.nan for k in range(4)] +
                    [(sp[k, 1] - t0) / 1e3 if sp[k, 1] > 0 else np.nan for k in range(4)])
    b = int(rng.integers(0, B)); a[b] = int(rng.integers(-1, T))  # one accepted move
r = np.nanmedian(np.array(rows), axis=0)
names = ["apply_one", "varcost", "chain", "final"]
for k, nm in enumerate(names):
    print(f"{nm:10s} start {r[k]:7.2f}  end {r[4 + k]:7.2f} us (median over {len(rows)} calls, from the update's start)")
