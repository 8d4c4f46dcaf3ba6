"""Event-timed k_eval (and the pm pair) with and without an L2 flush between launches."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from bench import build_inputs
from paper_2511_18296_b200.engine import Engine
c = build_inputs(sys.argv[1] if len(sys.argv) > 1 else "C2")
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
def timeit(fn, flush_on, n=50):
    ts = []
    for i in range(n):
        if flush_on: flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); st.synchronize(); ts.append(a.elapsed_time(b) * 1000)
    return np.median(ts[5:])
def eval_only():
    eng.eval_candidates_device(cand_d, out, None, net=True, stream=sp)
def pm_only():
    eng.set_schedule_device(assign_d, stream=sp, borrow=True); eng.period_mass_device(pm, stream=sp)
def step():
    eng.set_schedule_device(assign_d, stream=sp, borrow=True); eng.eval_candidates_device(cand_d, out, None, net=True, stream=sp)
eng.set_schedule_device(assign_d, stream=sp, borrow=True); eng.period_mass_device(pm, stream=sp)
for name, fn in (("eval_only", eval_only), ("pm_only", pm_only), ("step(pm+eval,PDL)", step)):
    print(f"{name:20s} cold {timeit(fn, True):8.2f} us   warm {timeit(fn, False):8.2f} us")
# eval with stats off and trace only
def eval_nostats():
    o2 = {k: out[k] for k in ("best_t", "best_val", "feasible", "global")}
    eng.eval_candidates_device(cand_d, o2, None, net=True, stream=sp)
print(f"{'eval_nostats':20s} cold {timeit(eval_nostats, True):8.2f} us   warm {timeit(eval_nostats, False):8.2f} us")
