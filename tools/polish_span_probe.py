"""Kernel spans of every pp_npv_moves evaluation of one native C2 polish sweep (library built
with -DPP_EVAL_PROBE: tools/build_probe.sh): earliest start / latest end of k_s2_apply_one,
k_s2_varcost, k_s2_chain and the final accumulation per call, medians over the calls that
started with the one-block update.

    python tools/polish_span_probe.py tools/libprobe.so
"""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2511_18296_b200 import _lib
lib = _lib.load(sys.argv[1]); _lib._lib = lib
lib.pp_debug_kspan_log.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
from paper_2511_18296_b200 import evaluate as dropin, synth
from paper_2511_18296_b200.model import ScenarioTables, scenario_values
c = synth.build_config("C2"); bm = c["bm"]
tb = ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"], grades=c["grades"])
a = synth.greedy_initialize(bm, c["grades"], c["sigma"]).astype(np.int64)
e = dropin._entry(bm); dropin._bind_scenarios(e, tb, True, None); eng = e.engine
cur = float(eng.npv_relaxed(a[None, :], use_sigma=True)[0])
load = np.array([bm.mass[a == t].sum() for t in range(bm.n_periods)])
n = ctypes.c_int64(0)
lib.pp_debug_kspan_log(None, 0, ctypes.byref(n))  # clear
a32 = a.astype(np.int32)
eng.polish_sweep(a32, load, cur, use_sigma=True, chunk0=64, chunk_max=128)
buf = np.zeros(20000 * 16, np.uint64)
lib.pp_debug_kspan_log(buf.ctypes.data, 20000, ctypes.byref(n))
sp = buf[: min(int(n.value), 20000) * 16].reshape(-1, 8, 2).astype(np.int64)
upd = sp[:, 0, 1] > 0  # calls with the one-block update
names = ["apply_one", "varcost", "chain", "final"]
t0 = np.where(upd, sp[:, 0, 0], sp[:, 2, 0])
print(f"{len(sp)} evaluations, {int(upd.sum())} with the one-block update")
for k, nm in enumerate(names):
    ok = upd & (sp[:, k, 1] > 0)
    st = (sp[ok, k, 0] - t0[ok]) / 1e3
    en = (sp[ok, k, 1] - t0[ok]) / 1e3
    print(f"{nm:10s} start {np.median(st):7.2f}  end {np.median(en):7.2f}  (p90 end {np.percentile(en, 90):7.2f}) us")
