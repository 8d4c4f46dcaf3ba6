"""cProfile of the reference's hybrid_optimize with the drop-ins installed (C5 at a given size)."""
import cProfile, os, pstats, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import pitplan.hybrid as H
from pitplan.blockmodel import generate_synthetic
from pitplan.scenarios import sample_lognormal
from pitplan.uncertainty import uncertainty_factors
from paper_2511_18296_b200.install import install

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
dims = {4000: (20, 20, 10), 50000: (50, 50, 20)}[n]
T, S = (10, 10) if n == 4000 else (15, 20)
inst = generate_synthetic(n, dims, T, 1, seed=1, n_rock_types=1)
scen = sample_lognormal(inst, S, 0.3, seed=2)
sigma = uncertainty_factors(inst, scen.grades)
cfg = H.HybridConfig(population=12, t_max=1, g_max=1, neighborhoods=2, init_multistarts=2, repair_iters=10, seed=0)
install()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
H.hybrid_optimize(inst, scen, sigma, cfg)
pr.disable()
print(f"total {time.perf_counter() - t0:.2f} s")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
pstats.Stats(pr).sort_stats("cumtime").print_stats("lns_repair|lns_insert|polish_schedule|_measure|_member")
