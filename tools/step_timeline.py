"""Timeline of one evaluation step (P1, P2, eval CTAs) from globaltimer probes."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_18296_b200 import _lib
lib = _lib.load(sys.argv[1]); _lib._lib = lib
lib.pp_debug_eval_probe.argtypes = [ctypes.c_void_p]; lib.pp_debug_pm_probe.argtypes = [ctypes.c_void_p]
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
       "feasible": torch.empty(C, dtype=torch.uint8, device=dev), "exp_delta": torch.empty(C, T, dtype=torch.float64, device=dev),
       "cvar": torch.empty(C, T, dtype=torch.float64, device=dev), "global": torch.empty(2, dtype=torch.float64, device=dev)}
pm_out = torch.empty(T, dtype=torch.float64, device=dev)
flush = torch.empty(256 << 18, dtype=torch.int32, device=dev)
grid = (C + 31) // 32  # k_eval_warp: 32 candidates per CTA
g = torch.cuda.CUDAGraph()
for _ in range(3):
    eng.set_schedule_device(assign_d, stream=sp, borrow=True); eng.eval_candidates_device(cand_d, out, None, net=True, stream=sp)
    eng.period_mass_device(pm_out, stream=sp)
st.synchronize()
with torch.cuda.graph(g):
    cs = torch.cuda.current_stream().cuda_stream
    eng.set_schedule_device(assign_d, stream=cs, borrow=True)
    if "pmonly" in sys.argv:  # the period-mass kernel alone (no concurrent evaluation CTAs)
        eng.period_mass_device(pm_out, stream=cs)
    else:
        eng.eval_candidates_device(cand_d, out, None, net=True, stream=cs)
lib.pp_debug_stamp.argtypes = [ctypes.c_void_p, ctypes.c_int]; lib.pp_debug_stamps.argtypes = [ctypes.c_void_p]
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
for rep in range(4):
    if "noflush" not in sys.argv: flush.fill_(rep)
    lib.pp_debug_stamp(sp, 0)
    if "noevents" not in sys.argv: e0.record(st)
    if "eager" in sys.argv:
        eng.set_schedule_device(assign_d, stream=sp, borrow=True); eng.eval_candidates_device(cand_d, out, None, net=True, stream=sp)
    else:
        g.replay()
    if "noevents" not in sys.argv: e1.record(st)
    lib.pp_debug_stamp(sp, 1)
    st.synchronize()
stamps = np.zeros(8, np.uint64); lib.pp_debug_stamps(stamps.ctypes.data); stamps = stamps.astype(np.int64)
print(f"event elapsed {e0.elapsed_time(e1) * 1000 if 'noevents' not in sys.argv else 0:.2f} us; stamp-to-stamp {(stamps[1] - stamps[0]) / 1000:.2f} us")
ev = np.zeros((4096, 12), np.uint64); lib.pp_debug_eval_probe(ev.ctypes.data); ev = ev[:grid].astype(np.int64)
if "pmonly" in sys.argv:
    ev[:] = ev.max()
pm = np.zeros((2, 512, 2), np.uint64); lib.pp_debug_pm_probe(pm.ctypes.data); pm = pm.astype(np.int64)
nr = int((pm[0, :16, 0] > 0).sum())
cl = nr >= 8
if cl:  # cluster path: 8 CTAs, [0][r] = (start, scatter done), [1][r][1] = trees done
    t0 = min(pm[0, :nr, 0].min(), ev[:, 0].min())
    f = lambda x: (x - t0) / 1000
    for k, nm in enumerate(["loaded", "ranked+bar", "offsets", "leaves", "pre-leaf", "leaf-t0", "leaf-addr", "leaf-sum", "leaf-tail"]):
        v = pm[1, 16 + 16 * k:32 + 16 * k, 0]
        v = v[v > 0]
        print(f"  pm {nm:8s} {f(v.min()):.2f}..{f(v.max()):.2f} us" + ("   per CTA: " + " ".join(f"{f(x):.1f}" for x in v) if "percta" in sys.argv else ""))
    print(f"PM cluster ({nr} CTAs): start {f(pm[0,:nr,0].min()):.2f}..{f(pm[0,:nr,0].max()):.2f}  scattered {f(pm[0,:nr,1].min()):.2f}..{f(pm[0,:nr,1].max()):.2f}  trees done {f(pm[1,:nr,1].min()):.2f}..{f(pm[1,:nr,1].max()):.2f} us")
else:
    nch = (c["bm"].n_blocks + 511) // 512
    p1, p2 = pm[0, :nch], pm[1, :T]
    t0 = min(p1[:, 0].min(), ev[:, 0].min())
    f = lambda x: (x - t0) / 1000
    print(f"P1 ({nch} CTAs): start {f(p1[:,0].min()):.2f}..{f(p1[:,0].max()):.2f}  end {f(p1[:,1].min()):.2f}..{f(p1[:,1].max()):.2f} us")
    print(f"P2 ({T} CTAs): after-wait {f(p2[:,0].min()):.2f}..{f(p2[:,0].max()):.2f}  end {f(p2[:,1].min()):.2f}..{f(p2[:,1].max()):.2f} us")
names = ["start", "loads", "values", "pm-wait", "moves", "outputs", "end", "stats", "pooled"]
for k in range(len(names)):
    print(f"eval {names[k]:9s} min {f(ev[:,k].min()):6.2f}  median {f(np.median(ev[:,k])):6.2f}  max {f(ev[:,k].max()):6.2f} us")
d = (ev[:, 6] - ev[:, 0]) / 1000
print("eval CTA duration us: p10 %.2f median %.2f p90 %.2f max %.2f" % tuple(np.percentile(d, [10, 50, 90, 100])))
print(f"stamp before the step {f(stamps[0]):.2f} us, after {f(stamps[1]):.2f} us (relative to the first kernel start)")
if "corr" in sys.argv:  # stats-phase duration per CTA against the CTA's capacity-feasible moves
    r = eng.eval_candidates(c["cand"], None, net=True, trace=True)
    per = np.add.reduceat(r["trace_feas"].sum(axis=1), np.arange(0, C, 32))
    dur = (ev[:, 4] - ev[:, 3]) / 1000
    dd = lambda a, b: np.median((ev[:, b] - ev[:, a])[ev[:, 9] > 0]) / 1000
    print("pm-wait->okm barrier %.2f" % dd(3, 8)); print("first move of warp 0: pm-wait->computed %.2f, ->leaves %.2f, ->k-smallest %.2f us (median)" % (dd(3, 9), dd(9, 10), dd(10, 11)))
    print("moves/CTA: mean %.1f max %d" % (per.mean(), per.max()))
    for lo, hi in ((0, 4), (4, 8), (8, 12), (12, 16), (16, 24), (24, 33), (33, 1000)):
        m = (per >= lo) & (per < hi)
        if m.any():
            print(f"  {lo:3d}-{hi:3d} moves: {m.sum():4d} CTAs, stats phase median {np.median(dur[m]):6.2f} max {dur[m].max():6.2f} us")
