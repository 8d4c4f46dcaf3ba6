"""Per-warp phase timeline of k_eval_warp (library built with -DPP_EVAL_PROBE: tools/build_probe.sh).
    python tools/warp_timeline.py tools/libprobe.so [C2]
Phases (lane 0 of every warp): 0 start, 1 loads done, 2 pool barrier passed, 3 own statistics
done, 4 statistics barrier passed, 5 values+ranks done, 6 period masses loaded, 7 selection done,
8 outputs done, 9 epilogue done."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_18296_b200 import _lib
lib = _lib.load(sys.argv[1]); _lib._lib = lib
lib.pp_debug_warp_probe.argtypes = [ctypes.c_void_p]
from bench import build_inputs
from paper_2511_18296_b200.engine import Engine
CFG = next((a for a in sys.argv[2:] if a in ("C1", "C2", "C3", "C4")), "C2")
c = build_inputs(CFG)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); sp = st.cuda_stream
eng = Engine.from_tables(c["bm"], c["tables"], c["assign"])
C, T = c["C"], c["T"]
assign_d = torch.from_numpy(c["assign"].astype(np.int32)).to(dev)
cand_d = torch.from_numpy(c["cand"]).to(dev)
out = {"best_t": torch.empty(C, dtype=torch.int32, device=dev), "best_val": torch.empty(C, dtype=torch.float64, device=dev),
       "feasible": torch.empty(C, dtype=torch.uint8, device=dev), "global": torch.empty(2, dtype=torch.float64, device=dev),
       "pair_cand": torch.empty(C * T, dtype=torch.int32, device=dev), "pair_period": torch.empty(C * T, dtype=torch.int32, device=dev),
       "pair_exp": torch.empty(C * T, dtype=torch.float64, device=dev), "pair_cvar": torch.empty(C * T, dtype=torch.float64, device=dev),
       "n_pairs": torch.zeros(1, dtype=torch.int32, device=dev)}
flush = torch.empty(256 << 18, dtype=torch.int32, device=dev)
g = torch.cuda.CUDAGraph()
for _ in range(3):
    eng.set_schedule_device(assign_d, stream=sp, borrow=True); eng.eval_candidates_device(cand_d, out, None, net=True, stream=sp)
st.synchronize()
with torch.cuda.graph(g):
    cs = torch.cuda.current_stream().cuda_stream
    eng.set_schedule_device(assign_d, stream=cs, borrow=True); eng.eval_candidates_device(cand_d, out, None, net=True, stream=cs)
for rep in range(3):
    flush.fill_(rep); st.synchronize(); g.replay(); st.synchronize()
w = np.zeros((1024, 8, 12), np.uint64); lib.pp_debug_warp_probe(w.ctypes.data); w = w.astype(np.int64)
grid = min((C + 31) // 32, 1024)
w = w[:grid]
t0 = w[:, :, 0].min()
f = lambda x: (x - t0) / 1000.0
names = ["start", "loads", "pool bar", "own stats", "stats bar", "values", "pm loaded", "selection", "outputs", "end"]
print(f"{CFG}: {grid} CTAs x 8 warps; times in us from the first warp start")
for k, nm in enumerate(names):
    v = f(w[:, :, k].ravel())
    print(f"  {k} {nm:10s} p10 {np.percentile(v, 10):6.2f}  median {np.median(v):6.2f}  p90 {np.percentile(v, 90):6.2f}  max {v.max():6.2f}")
print("phase durations per warp (median / p90 us):")
for k in range(1, len(names)):
    d = (w[:, :, k] - w[:, :, k - 1]).ravel() / 1000.0
    print(f"  {names[k - 1]:10s} -> {names[k]:10s} {np.median(d):6.2f} / {np.percentile(d, 90):6.2f}")

cyc = w[:, :, 10].ravel()
cyc = cyc[(cyc > 0) & (cyc < 10**9)]
if cyc.size:
    print("statistics loop, SM cycles per warp: median %d p90 %d max %d" % (np.median(cyc), np.percentile(cyc, 90), cyc.max()))
