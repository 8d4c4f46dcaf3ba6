"""Per-CTA stage timeline of k_eval_staged (library built with -DPP_EVAL_PROBE)."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_18296_b200 import _lib
lib = _lib.load(sys.argv[1]); _lib._lib = lib
lib.pp_debug_eval_probe.argtypes = [ctypes.c_void_p]
from bench import build_inputs
from paper_2511_18296_b200.engine import Engine
c = build_inputs("C2")
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); sp = st.cuda_stream
eng = Engine.from_tables(c["bm"], c["tables"], c["assign"])
C, T = c["C"], c["T"]
assign_d = torch.from_numpy(c["assign"].astype(np.int32)).to(dev)
cand_d = torch.from_numpy(c["cand"]).to(dev)
out = {"best_t": torch.empty(C, dtype=torch.int32, device=dev), "best_val": torch.empty(C, dtype=torch.float64, device=dev),
       "feasible": torch.empty(C, dtype=torch.uint8, device=dev), "exp_delta": torch.empty(C, T, dtype=torch.float64, device=dev),
       "cvar": torch.empty(C, T, dtype=torch.float64, device=dev), "global": torch.empty(2, dtype=torch.float64, device=dev)}
pm = torch.empty(T, dtype=torch.float64, device=dev)
flush = torch.empty(256 << 18, dtype=torch.int32, device=dev)
grid = (C + 31) // 32
for mode in ("cold", "warm", "step"):
    for rep in range(3):
        if mode == "cold": flush.fill_(rep)
        if mode == "step":
            flush.fill_(rep); eng.set_schedule_device(assign_d, stream=sp, borrow=True)
        else:
            eng.set_schedule_device(assign_d, stream=sp, borrow=True); eng.period_mass_device(pm, stream=sp); st.synchronize()
        eng.eval_candidates_device(cand_d, out, None, net=True, stream=sp); st.synchronize()
    a = np.zeros((4096, 8), np.uint64); lib.pp_debug_eval_probe(a.ctypes.data)
    a = a[:grid].astype(np.int64); t0 = a[:, 0].min()
    r = a - t0
    print(f"[{mode}] kernel span {(a[:,7].max()-t0)/1000:.2f} us; CTA start spread {r[:,0].max()/1000:.2f} us")
    names = ["start", "ids", "rows(cp.async)", "window", "pm-wait", "capacity", "stats", "out+argmax+exit"]
    for k in range(1, 8):
        d = (a[:, k] - a[:, k-1]) / 1000
        print(f"   {names[k]:16s} median {np.median(d):6.2f} us  p90 {np.percentile(d,90):6.2f}  max {d.max():6.2f}")
