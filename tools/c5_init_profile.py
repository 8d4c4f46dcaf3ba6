"""cProfile of HybridSearch.__init__ (the C5 set-up: evaluator, greedy multistarts, the initial
population) at C2 with the drop-ins installed."""
import cProfile, os, pstats, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import pitplan.hybrid as H
from pitplan.blockmodel import generate_synthetic
from pitplan.scenarios import sample_lognormal
from pitplan.uncertainty import uncertainty_factors
from paper_2511_18296_b200.install import install

inst = generate_synthetic(50000, (50, 50, 20), 15, 1, seed=1, n_rock_types=1)
scen = sample_lognormal(inst, 20, 0.3, seed=2)
sigma = uncertainty_factors(inst, scen.grades)
cfg = H.HybridConfig(population=12, t_max=3, g_max=1, neighborhoods=2, init_multistarts=2, repair_iters=10, seed=0)
install()
import torch; torch.cuda.init()  # (context creation outside the profile)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
H.HybridSearch(inst, scen, sigma, cfg)
pr.disable()
print(f"init {time.perf_counter() - t0:.2f} s")
pstats.Stats(pr).sort_stats("cumtime").print_stats(30)
