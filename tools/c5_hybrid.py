"""C5: the reference's full hybrid GA+LNS+SA loop driving the device engine.

Runs the UNMODIFIED reference `hybrid_optimize` (hybrid.py:1015-1026) from the pip install
under baseline/_ref (or /root/reference/pkg/src in the build container), once on its own CPU
path and/or once with `paper_2511_18296_b200.install()` rebinding its evaluator entry points
(install.py). With --mode both the two runs must agree bit for bit: the same best schedule
(sha256 of the `<i8` assignment, evaluate.py:54-55) and the same per-iteration trace rows
(hybrid.py:514-534, `repr` of every float).

    python tools/c5_hybrid.py --blocks 4000 --dims 20 20 10 --periods 10 --scen 10 --mode both
    python tools/c5_hybrid.py --blocks 50000 --dims 50 50 20 --periods 15 --scen 20 --mode device
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "pitplan")):
        sys.path.insert(0, cand)
        break

import pitplan.hybrid as H  # noqa: E402
from pitplan.blockmodel import generate_synthetic  # noqa: E402
from pitplan.scenarios import sample_lognormal  # noqa: E402
from pitplan.uncertainty import uncertainty_factors  # noqa: E402


def digest(a) -> str:
    return hashlib.sha256(np.asarray(a, dtype="<i8").tobytes()).hexdigest()


def run_once(inst, scen, sigma, cfg, label):
    timings = []
    t_iter = [time.perf_counter()]

    def control(it, search):
        now = time.perf_counter()
        timings.append(now - t_iter[0])
        t_iter[0] = now
        return None

    t0 = time.perf_counter()
    search = H.HybridSearch(inst, scen, sigma, cfg)
    t_init = time.perf_counter() - t0
    t_iter[0] = time.perf_counter()
    best, trace = search.run(control)
    total = time.perf_counter() - t0
    rows = [r.as_list() for r in trace]
    return {
        "label": label,
        "init_s": t_init,
        "iter_s": timings,
        "total_s": total,
        "best_digest": digest(best.assignment),
        "best_npv": float(search.best_npv),
        "mined": int(np.sum(np.asarray(best.assignment) >= 0)),
        "trace": rows,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=4000)
    ap.add_argument("--dims", type=int, nargs=3, default=(20, 20, 10))
    ap.add_argument("--periods", type=int, default=10)
    ap.add_argument("--scen", type=int, default=10)
    ap.add_argument("--population", type=int, default=12)
    ap.add_argument("--t-max", type=int, default=3)
    ap.add_argument("--g-max", type=int, default=1)
    ap.add_argument("--neighborhoods", type=int, default=2)
    ap.add_argument("--multistarts", type=int, default=2)
    ap.add_argument("--repair-iters", type=int, default=10)
    ap.add_argument("--no-polish", action="store_true")
    ap.add_argument("--mode", choices=("reference", "device", "both"), default="both")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    t0 = time.perf_counter()
    inst = generate_synthetic(a.blocks, tuple(a.dims), a.periods, 1, seed=1, n_rock_types=1)
    scen = sample_lognormal(inst, a.scen, 0.3, seed=2)
    sigma = uncertainty_factors(inst, scen.grades)
    t_build = time.perf_counter() - t0
    cfg = H.HybridConfig(population=a.population, t_max=a.t_max, g_max=a.g_max,
                         neighborhoods=a.neighborhoods, init_multistarts=a.multistarts,
                         repair_iters=a.repair_iters, polish=not a.no_polish, seed=0)
    res = {"config": {"blocks": a.blocks, "dims": list(a.dims), "periods": a.periods,
                      "scenarios": a.scen, "population": a.population, "t_max": a.t_max,
                      "g_max": a.g_max, "neighborhoods": a.neighborhoods,
                      "init_multistarts": a.multistarts, "repair_iters": a.repair_iters,
                      "polish": not a.no_polish},
           "instance_build_s": t_build}
    runs = {}
    if a.mode in ("reference", "both"):
        runs["reference"] = run_once(inst, scen, sigma, cfg, "reference")
    if a.mode in ("device", "both"):
        from paper_2511_18296_b200 import evaluate as ev
        from paper_2511_18296_b200.install import install, uninstall
        patched = install()
        try:
            runs["device"] = run_once(inst, scen, sigma, cfg, "device")
        finally:
            uninstall()
            ev.clear_cache()
        runs["device"]["patched"] = patched
    res["runs"] = runs
    if len(runs) == 2:
        r, d = runs["reference"], runs["device"]
        res["identical"] = r["best_digest"] == d["best_digest"] and r["trace"] == d["trace"]
        res["speedup_total"] = r["total_s"] / d["total_s"]
    for k, v in runs.items():
        print(f"[c5] {k}: init {v['init_s']:.2f} s, iterations {[round(x, 2) for x in v['iter_s']]} s, "
              f"total {v['total_s']:.2f} s, best NPV {v['best_npv']!r}, mined {v['mined']}, "
              f"digest {v['best_digest'][:16]}")
    if "identical" in res:
        print(f"[c5] identical best schedule and trace: {res['identical']}; speed-up {res['speedup_total']:.1f}x")
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
    if res.get("identical") is False:
        sys.exit(1)


if __name__ == "__main__":
    main()
