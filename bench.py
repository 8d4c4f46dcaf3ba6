"""Benchmark of the B200 move-evaluation engine (BASELINE.json metric).

One step = one evaluator batch of the headline configuration C2:
50,000-block model, 15 periods, 20 scenarios, 16,667 candidate blocks x 15 periods =
250,005 candidate moves, each evaluated under all 20 scenarios:

  k_pm_cluster: period masses of the current schedule (bit-exact numpy pairwise tree,
    one 8-CTA cluster)
  + k_eval_warp (launched with programmatic dependent launch so its gathers and the
    per-scenario statistics overlap k_pm_cluster): precedence window, capacity test,
    kernel value (ref parity key), per-scenario deltas -> expected delta and CVaR10 of
    every feasible move (sparse output), per-candidate argmax, grid argmax (1 kernel)
  [+ N>1: NCCL all-gather of the 16-byte per-GPU best and an ordered reduce kernel]

`value` is device-timed (CUDA events, inputs resident in HBM, L2 flushed by a 256 MiB
write between timed steps); `e2e` is the same batch through the C ABI with host
buffers (pinned), host<->device copies inside the timed region.
`--impl reference` times the CPU restatement of the reference path (oracle/oracle.c, OpenMP,
all host cores; the reference is pure Python, so there is no compiled oracle/_ref) and, beside
it, the reference itself -- pitplan's own evaluate_candidates_parallel from its pip install
under baseline/_ref, worker_count 1 and os.cpu_count(), best of 3.

Roofline: `achieved` = SURVEY §8(d)'s algorithmic bytes of one batch
(M·(80 + 8·d̄) + 8·M·S, f64 values) / the k_eval_warp launch time measured with CUDA events
around a graph holding only that launch; the compulsory bytes (each candidate's rows once) and
ncu's measured DRAM bytes of the same config are reported beside it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "move×scenario evals/sec and ms per 250k-move batch (50k blocks); % HBM roofline"
UNIT = "move-scenario evals/s"
L2_FLUSH_BYTES = 256 << 20


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


STRONG = ("C4",)  # C4: one 1M-move list split over the GPUs; the others: C candidates per GPU


def build_inputs(config: str, rank: int = 0, world: int = 1):
    """The config's inputs plus this rank's shard of ONE global candidate list:
    weak scaling (C1-C3) draws world x C candidates from the config's stream and gives rank r the
    contiguous range [r C, (r+1) C) -- at world = 1 exactly the config's list; strong scaling (C4)
    splits the config's list into contiguous balanced shards."""
    from paper_2511_18296_b200 import synth
    from paper_2511_18296_b200.distributed import shard_bounds
    from paper_2511_18296_b200.model import ScenarioTables, scenario_values

    c = synth.build_config(config)
    if config == "C3":
        # BASELINE's C3 names 200 VAE-sampled scenarios: the reference's VAE architecture (VaeConfig
        # defaults: latent 16, decoder 64-128-256-B) with random-init weights (no trained model can
        # be fetched here), normalised as vae_train does over a 256-field lognormal corpus of the
        # instance, decoded from standard-normal prior samples
        from paper_2511_18296_b200.model import VaeDecoder

        corpus = synth.sample_lognormal(c["bm"], 256, 0.3, seed=9)
        dec = VaeDecoder.random_init(c["bm"].n_blocks, corpus.mean(axis=0), corpus.std(axis=0) + 1e-8, seed=7)
        z = np.random.default_rng(8).standard_normal((c["S"], dec.latent_dim))
        c["grades"] = dec.decode_host(z)
        c["sigma"] = synth.uncertainty_sigma(c["bm"], c["grades"])
        c["vae"] = (dec, z)
    if config in STRONG:
        c["cand_global"] = c["cand"]
    else:
        c["cand_global"] = c["cand"] if world == 1 else synth.candidate_blocks(c["bm"].n_blocks, c["C"] * world)
    lo, hi = shard_bounds(c["cand_global"].size, world, rank)
    c["cand"] = np.ascontiguousarray(c["cand_global"][lo:hi])
    c["C"] = int(c["cand"].size)
    c["tables"] = ScenarioTables(scenario_values(c["bm"], c["grades"]), c["sigma"])
    return c


def _ncu_traffic(config: str):
    """(dram__bytes_read.sum + dram__bytes_write.sum of one k_eval_warp launch, source file) from the
    committed `ncu --set full` capture of the same --config (profiles/r02_ncu_<config>.json, or the
    round-1 C2 capture for C2), or (None, None)."""
    prof = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    cands = [f"r02_ncu_{config.lower()}.json"] + (["r01_ncu_full.json"] if config == "C2" else [])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for name in cands:
        try:
            m = json.load(open(os.path.join(prof, name)))["k_eval_warp"]
        except (OSError, KeyError, ValueError):
            continue
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = m[k]
            tot += float(v) * scale.get(u, 1)
        return tot, f"profiles/{name}"
    return None, None


def precedence_feasible_moves(c) -> int:
    """Moves whose precedence window admits the period (evaluate.py:361-372): the moves that reach
    the per-scenario statistics (scen_evals_performed = this x S)."""
    bm, a, cand, T = c["bm"], c["assign"], c["cand"], c["T"]
    pp_, pi_, sp_, si_ = bm.csr()
    tot = 0
    for b in cand.tolist():
        pa = a[pi_[pp_[b]:pp_[b + 1]]]
        if pa.size and np.any(pa < 0):
            continue
        lo = int(pa.max()) if pa.size else 0
        sa = a[si_[sp_[b]:sp_[b + 1]]]
        sa = sa[sa >= 0]
        hi = int(sa.min()) if sa.size else T - 1
        tot += max(0, min(hi, T - 1) - max(lo, 0) + 1)
    return tot


def python_reference_timing(config: str, cand: np.ndarray, assign: np.ndarray, repeats: int = 3) -> dict | None:
    """The reference itself: pitplan.evaluate.evaluate_candidates_parallel from its pip install under
    baseline/_ref, on inputs built by the reference's own generators (identical to synth's, digests
    checked in tests), worker_count 1 and os.cpu_count(), best of `repeats`."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "pitplan")):
        return None
    if ref not in sys.path:
        sys.path.append(ref)
    from pitplan.blockmodel import generate_synthetic
    from pitplan.evaluate import Schedule, evaluate_candidates_parallel
    from pitplan.scenarios import sample_lognormal
    from pitplan.uncertainty import uncertainty_factors

    from paper_2511_18296_b200 import synth

    spec = {"C1": (4000, (20, 20, 10), 10, 10, 1.3), "C2": (50000, (50, 50, 20), 15, 20, 1.3),
            "C3": (50000, (50, 50, 20), 15, 200, 0.3), "C4": (200000, (100, 100, 20), 20, 50, 1.3)}[config]
    n, dims, T, S, cf = spec
    t0 = time.perf_counter()
    inst = generate_synthetic(n, dims, T, 1, seed=1, n_rock_types=1, capacity_factor=cf)
    scen = sample_lognormal(inst, S, 0.3, seed=2)
    sigma = uncertainty_factors(inst, scen.grades)
    build_s = time.perf_counter() - t0
    sched = Schedule(np.asarray(assign, dtype=np.int64).copy())
    cl = [int(b) for b in cand]
    out = {"kind": "reference", "impl": "pitplan.evaluate.evaluate_candidates_parallel (baseline/_ref)",
           "inputs_build_s": build_s, "moves": len(cl) * T, "scenarios": S}
    for w in sorted({1, os.cpu_count() or 1}):
        ts = []
        for _ in range(repeats):
            t1 = time.perf_counter()
            evaluate_candidates_parallel(inst, sched, cl, scen, None, sigma, worker_count=w, net_mining_cost=True)
            ts.append(time.perf_counter() - t1)
        best = min(ts)
        out[f"W{w}"] = {"s_per_batch": best, "value": len(cl) * T * S / best, "unit": UNIT, "cores": w,
                        "moves_per_s": len(cl) * T / best}
    return out


def algorithmic_bytes(c, deg_mean: float, n_pairs: int) -> dict:
    """Compulsory bytes of one k_eval_warp launch: every candidate's inputs
    once, its best move, and one (candidate, period, expected delta, CVaR10) record per
    feasible move (sparse statistics output)."""
    C, T, S = c["C"], c["T"], c["S"]
    per_cand = (4 + 32 + 4 + 8 + 8 * deg_mean   # cand id, BlockRow, assign[b], unit_mean[b], adjacency ids+assign
                + 8 * T + 8 * ((S + 3) & ~3)      # mining-cost row, vmax row (fp64, padded to 4)
                + 13)                             # best (t, value, flag)
    per_pair = 4 + 4 + 8 + 8
    M = C * T
    survey = M * (80 + 8 * deg_mean) + 8 * M * S  # SURVEY §8(d) per-move figure, fp64 vmax, no reuse
    return {"per_candidate": per_cand, "per_pair": per_pair,
            "per_launch": per_cand * C + per_pair * n_pairs, "survey_uncached": survey}


def workload_config(args, c) -> dict:
    """The `config` object of both arms (identical, so the driver compares like with like)."""
    C, T, S = c["C"], c["T"], c["S"]
    G = int(c["cand_global"].size)
    return {
        "workload": ("C2: 50k-block model (50x50x20), 15 periods, 20 lognormal scenarios with sigma, "
                     "16,667 candidate blocks x 15 periods = 250,005 moves per GPU per step, "
                     "net mining cost, per-move expected delta + CVaR10, argmax")
        if args.config == "C2" else args.config,
        "blocks": c["bm"].n_blocks, "periods": T, "scenarios": S,
        "candidates_global": G, "moves_global_per_step": G * T,
        "candidates_per_gpu": C, "moves_per_gpu_per_step": C * T,
        "sharding": ("one global candidate list, contiguous per-GPU ranges; "
                     + ("strong scaling (fixed 1M-move list)" if args.config in STRONG
                        else "weak scaling (C candidates per GPU)")),
        "l2": "256 MiB flush write between timed GPU steps",
        "scenario_source": SCENARIO_SOURCE.get(args.config, "sample_lognormal"),
    }


# where each configuration's scenario grades come from (the value table the kernels consume is the
# same function of the grades either way)
SCENARIO_SOURCE = {
    "C1": "sample_lognormal (scenarios.py), shock 0.3",
    "C2": "sample_lognormal (scenarios.py), shock 0.3",
    "C3": ("200 scenarios decoded by a VAE of the reference's architecture (vae.py VaeConfig defaults: latent "
           "16, decoder 64-128-256-B, random-init weights, vae_train's normalisation over a 256-field "
           "lognormal corpus), standard-normal prior samples"),
    "C4": "sample_lognormal (scenarios.py), shock 0.3",
}


def cpu_reference(c, seconds: float = 3.0, nthreads: int | None = None, max_batches: int | None = None):
    """Time the oracle port on the same batch (period mass + evaluation + scenario stats)."""
    from oracle import oracle

    oracle.build()
    o = oracle.Oracle(c["bm"], c["tables"].vmax, c["tables"].sigma)
    nthreads = nthreads or os.cpu_count() or 1
    o.eval_candidates(c["assign"], c["cand"], None, net=True, stats=True, nthreads=nthreads)  # warm
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or not times:
        t0 = time.perf_counter()
        o.eval_candidates(c["assign"], c["cand"], None, net=True, stats=True, nthreads=nthreads)
        times.append(time.perf_counter() - t0)
        if max_batches and len(times) >= max_batches:
            break
    return times, nthreads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    c = build_inputs(args.config, 0, world)
    cfg = workload_config(args, c)
    c["cand"] = np.ascontiguousarray(c["cand_global"])  # the whole job's list, on the host cores
    c["C"] = int(c["cand"].size)
    M, S = c["C"] * c["T"], c["S"]
    from oracle import oracle

    oracle.build()
    o = oracle.Oracle(c["bm"], c["tables"].vmax, c["tables"].sigma)
    nth = os.cpu_count() or 1
    t0 = time.perf_counter()
    o.eval_candidates(c["assign"], c["cand"], None, net=True, stats=True, nthreads=nth)
    one = time.perf_counter() - t0
    budget = 150.0
    frac = 1.0
    if (args.steps + args.warmup) * one > budget:
        frac = max(budget / ((args.steps + args.warmup) * one), 0.02)
    n_c = max(1, int(round(c["C"] * frac)))
    cand = c["cand"][:n_c]
    for _ in range(args.warmup):
        o.eval_candidates(c["assign"], cand, None, net=True, stats=True, nthreads=nth)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.eval_candidates(c["assign"], cand, None, net=True, stats=True, nthreads=nth)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    value = n_c * c["T"] * S / t
    sample = (f"{n_c} of {c['C']} candidates x {c['T']} periods x {S} scenarios per step "
              f"({'full batch' if n_c == c['C'] else 'bounded sample'}), incl. period masses")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "ms_per_250k_batch": t * 1e3 * (M / (n_c * c["T"])), "higher_is_better": True,
        "scaling": "strong" if args.config in STRONG else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nth, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_baseline_reference": None if args.no_python_ref else python_reference_timing(args.config, c["cand"],
                                                                                        c["assign"]),
    }
    print(json.dumps(line))
    return 0


def run_gpu(args):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PP_BENCH_DIST") == "gloo" and torch.cuda.device_count() <= local:
        local = 0  # the one-GPU functional check: every rank on device 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # NCCL over NVLink/NVSwitch; PP_BENCH_DIST=gloo is a functional multi-rank check on one GPU
        # (host-staged exchange, not a measurement)
        backend = os.environ.get("PP_BENCH_DIST", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def all_gather_dev(dst, src):
        if dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(dst, src)
        else:
            parts = [torch.empty_like(src, device="cpu") for _ in range(world)]
            dist.all_gather(parts, src.cpu())
            dst.copy_(torch.cat(parts))

    def all_reduce_max(t):
        if dist.get_backend() == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        return h
    from paper_2511_18296_b200.engine import Engine, PinnedPool

    c = build_inputs(args.config, rank, world)
    bm, T, S, C = c["bm"], c["T"], c["S"], c["C"]
    M = C * T
    M_global = c["cand_global"].size * T
    dev = torch.device("cuda", local)
    eng = Engine.from_tables(bm, c["tables"], c["assign"], device=local)
    ingest = None
    if "vae" in c:  # C3: the scenario set decoded and tabulated on the device (outside the timed step)
        dec, z = c["vae"]
        eng.set_vae_decoder(dec)
        g_dev = eng.vae_decode(z)
        rel = float(np.max(np.abs(g_dev - c["grades"]) / np.maximum(np.abs(c["grades"]), 1.0)))
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            eng.set_scenarios_vae(z, c["sigma"])
            ts.append(time.perf_counter() - t0)
        w = dec.widths
        flop = 2.0 * S * sum(w[k] * w[k + 1] for k in range(len(w) - 1))
        ingest = {"what": f"VAE decode of {S} scenarios (decoder {'-'.join(map(str, w))}, f64 tiled GEMMs) + "
                          "value table, on the device (pp_set_scenarios_vae), host call time",
                  "ms": float(np.median(ts[1:])) * 1e3, "decode_gflop": flop / 1e9,
                  "max_rel_diff_vs_numpy_decode": rel}
        eng.set_scenarios(c["tables"])  # both arms evaluate the numpy-decoded grades (identical inputs)
    deg_mean = 2.0 * bm.n_edges / bm.n_blocks
    # a dedicated stream: handle 0 (torch's legacy default stream) would mean "the engine
    # context's own stream" to the C ABI, and events recorded on it would not order the kernels
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    assert sptr != 0

    assign_d = torch.from_numpy(c["assign"].astype(np.int32)).to(dev)
    cand_d = torch.from_numpy(c["cand"]).to(dev)
    out = {
        "best_t": torch.empty(C, dtype=torch.int32, device=dev),
        "best_val": torch.empty(C, dtype=torch.float64, device=dev),
        "feasible": torch.empty(C, dtype=torch.uint8, device=dev),
        "global": torch.empty(2, dtype=torch.float64, device=dev),
        # sparse statistics of the feasible moves (pp_cand_out.pair_*)
        "pair_cand": torch.empty(C * T, dtype=torch.int32, device=dev),
        "pair_period": torch.empty(C * T, dtype=torch.int32, device=dev),
        "pair_exp": torch.empty(C * T, dtype=torch.float64, device=dev),
        "pair_cvar": torch.empty(C * T, dtype=torch.float64, device=dev),
        "n_pairs": torch.zeros(1, dtype=torch.int32, device=dev),
    }
    gathered = torch.empty(2 * world, dtype=torch.float64, device=dev)
    final = torch.empty(2, dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    pm_copy = torch.empty(T, dtype=torch.float64, device=dev)

    def step():
        # the schedule is read in place; the call enqueues k_pm_cluster + k_eval_warp (PDL)
        eng.set_schedule_device(assign_d, stream=sptr, borrow=True)
        eng.eval_candidates_device(cand_d, out, None, net=True, stream=sptr)
        if world > 1:
            all_gather_dev(gathered, out["global"])
            eng.reduce_best_device(gathered, final, stream=sptr)

    for _ in range(max(args.warmup, 3)):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()

    graph = None
    if world == 1 and not args.no_graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                cs = torch.cuda.current_stream().cuda_stream
                eng.set_schedule_device(assign_d, stream=cs, borrow=True)
                eng.eval_candidates_device(cand_d, out, None, net=True, stream=cs)
            g.replay()
            torch.cuda.synchronize()
            graph = g
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] graph capture failed, eager launches: {exc}", file=sys.stderr)
            graph = None

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kstarts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        time.sleep(0.05)
        for i in range(args.steps):
            flush.fill_(i)  # 256 MiB write: nothing of the previous step stays in the 126 MB L2
            starts[i].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        time.sleep(0.05)
    if dist is not None:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_local = float(np.mean(step_ms))
    t_max = t_local
    if dist is not None:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        t_max = float(all_reduce_max(tt).item())

    # dominant kernel alone: k_eval_warp in its own CUDA graph (period masses refreshed beforehand,
    # so the captured call launches only the evaluation kernel and its output-init copy), timed
    # with events on its stream, L2 flushed between replays
    eng.set_schedule_device(assign_d, stream=sptr, borrow=True)
    eng.period_mass_device(pm_copy, stream=sptr)
    torch.cuda.synchronize()
    kgraph = None
    if not args.no_graph:
        try:
            kg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(kg):
                eng.eval_candidates_device(cand_d, out, None, net=True, stream=torch.cuda.current_stream().cuda_stream)
            kg.replay()
            torch.cuda.synchronize()
            kgraph = kg
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] kernel graph capture failed, eager launch: {exc}", file=sys.stderr)
    nk = min(args.steps, 200)
    for i in range(nk):
        flush.fill_(i)
        kstarts[i].record(stream)
        if kgraph is not None:
            kgraph.replay()
        else:
            eng.eval_candidates_device(cand_d, out, None, net=True, stream=sptr)
        kends[i].record(stream)
    torch.cuda.synchronize()
    kms = [s.elapsed_time(e) for s, e in zip(kstarts[:nk], kends[:nk])]
    k_ms = float(np.median(kms))

    # e2e through the C ABI with host (pinned) buffers on every rank: H2D schedule + candidates,
    # both kernels, D2H of the best moves and the sparse statistics; for N > 1 also the 16-byte
    # per-rank best through NCCL (all-gather + ordered reduce) and back to the host
    pool = PinnedPool()
    h_assign = pool.empty(bm.n_blocks, np.int32)
    h_assign[:] = c["assign"]
    h_cand = pool.empty(C, np.int32)
    h_cand[:] = c["cand"]
    h_out = {"best_t": pool.empty(C, np.int32), "best_val": pool.empty(C, np.float64),
             "feasible": pool.empty(C, np.uint8), "pair_cand": pool.empty(C * T, np.int32),
             "pair_period": pool.empty(C * T, np.int32), "pair_exp": pool.empty(C * T, np.float64),
             "pair_cvar": pool.empty(C * T, np.float64), "n_pairs": pool.empty(1, np.int32)}
    h_best = pool.empty(2, np.float64)
    h_best_t = torch.from_numpy(h_best)
    d_best = torch.empty(2, dtype=torch.float64, device=dev)
    e2e = []
    r = None
    for i in range(args.warmup + min(args.steps, 300)):
        flush.fill_(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.set_schedule(h_assign)
        r = eng.eval_candidates(h_cand, None, net=True, pairs=True, out=h_out, validate=False)
        if world > 1:
            bb, bt, bv = r["best"] if r["best"] is not None else (-1, -1, -np.inf)  # (block, period, value)
            h_best[0] = bv
            h_best.view(np.int32)[2:4] = (bb, bt)
            d_best.copy_(h_best_t, non_blocking=True)
            all_gather_dev(gathered, d_best)
            eng.reduce_best_device(gathered, final, stream=sptr)
            h_best_t.copy_(final)  # synchronising D2H of the global best
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e.append(t1 - t0)
    e2e_t = float(np.median(e2e))
    if dist is not None:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        e2e_t = float(all_reduce_max(tt).item())
    h2d = h_assign.nbytes + h_cand.nbytes
    npairs = int(h_out["n_pairs"][0])
    d2h = (h_out["best_t"].nbytes + h_out["best_val"].nbytes + h_out["feasible"].nbytes + 16 + 4
           + npairs * (4 + 4 + 8 + 8))
    # parity spot check of the timed configuration against the device run
    assert r["best"] is not None
    g = out["global"].cpu().numpy()
    gi = g.view(np.int32)
    assert (int(gi[2]), int(gi[3]), float(g[0])) == r["best"], "device/host paths disagree"
    argmax_check = None
    if world > 1:  # the all-gathered argmax of the shards == one GPU evaluating the whole global list
        glob = (int(h_best.view(np.int32)[2]), int(h_best.view(np.int32)[3]), float(h_best[0]))
        if rank == 0:
            eng.set_schedule(c["assign"])
            whole = eng.eval_candidates(np.ascontiguousarray(c["cand_global"], dtype=np.int32), None, net=True)["best"]
            argmax_check = {"sharded": list(glob), "whole_list_on_rank0": list(whole), "equal": whole == glob}
            assert whole == glob, ("sharded argmax differs from the whole-list evaluation", glob, whole)
    pool.close()

    result = None
    if rank == 0:
        hbm, peak_kind = _peaks()
        ab = algorithmic_bytes(c, deg_mean, int(out["n_pairs"].item()))
        # roofline numerator (the contract's): SURVEY §8(d)'s algorithmic bytes of the batch, which
        # count every (b, t) move as reading its rows and its scenario row; the kernel reads each
        # candidate's rows once for all its periods, so the compulsory bytes and ncu's DRAM bytes
        # are reported beside it
        ks = k_ms * 1e-3
        achieved = ab["survey_uncached"] / ks / 1e9
        achieved_comp = ab["per_launch"] / ks / 1e9
        traffic, traffic_src = (args.ncu_traffic, "--ncu-traffic") if args.ncu_traffic is not None \
            else _ncu_traffic(args.config)
        value = M_global * S / (t_max * 1e-3)
        n_prec = precedence_feasible_moves(c)

        cpu = None
        pyref = None
        if world == 1 and not args.no_cpu_baseline:
            ts, nth = cpu_reference(c, seconds=args.cpu_seconds)
            t_cpu = float(np.median(ts))
            cpu = {"value": M * S / t_cpu, "unit": UNIT, "cores": nth, "kind": "port",
                   "sample": f"{len(ts)} full batches ({M} moves x {S} scenarios each, incl. period masses), "
                             f"oracle/oracle.c with OpenMP, median"}
            if not args.no_python_ref:
                pyref = python_reference_timing(args.config, c["cand"], c["assign"])
        launches_per_step = 2 + (1 if world > 1 else 0)  # k_pm_cluster + k_eval_warp [+ k_reduce_best]
        result = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_max,
            "ms_per_250k_batch": t_max * (250000.0 / M),
            "higher_is_better": True,
            "scaling": "strong" if args.config in STRONG else "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(args, c),
            "argmax_check": argmax_check,
            "cuda_graph": graph is not None,
            "roofline": {
                "bound": "hbm",
                "achieved": achieved,
                "peak": hbm,
                "unit": "GB/s",
                "frac": achieved / hbm,
                "traffic": traffic,
                "traffic_source": traffic_src,
                "kernel": "k_eval_warp",
                "kernel_ms": k_ms,
                "kernel_timing": "median CUDA-event time of a graph holding only the k_eval_warp launch, L2 flushed",
                "algorithmic_bytes_per_launch": ab["survey_uncached"],
                "algorithmic_basis": "SURVEY §8(d): M*(80 + 8*deg) + 8*M*S (f64 scenario values), M = moves per batch",
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "compulsory_bytes_per_launch": ab["per_launch"],
                "compulsory_basis": "per candidate 4+32+4+8+8*deg+8*T+8*Sp+13 B, per feasible pair 24 B",
                "compulsory_achieved": achieved_comp,
                "compulsory_frac": achieved_comp / hbm,
                "dram_achieved": (traffic / ks / 1e9) if traffic else None,
                "dram_frac": (traffic / ks / 1e9 / hbm) if traffic else None,
            },
            "moves_per_step": M,
            "scen_evals_nominal_per_step": M * S,
            "precedence_feasible_moves_per_step": n_prec,
            "scen_evals_performed_per_step": n_prec * S,
            "e2e": {"value": M_global * S / e2e_t, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_t * 1e3,
                    "api": "Engine.set_schedule + Engine.eval_candidates (pp_set_schedule/pp_eval_candidates, "
                           "PP_MEM_HOST, pinned)" + (" + NCCL all-gather/reduce of the per-rank best" if world > 1 else ""),
                    "note": "per rank; max over ranks" if world > 1 else None},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "cpu_baseline_reference": pyref,
            "best_move": {"block": r["best"][0], "period": r["best"][1], "value": r["best"][2]},
        }
        if ingest is not None:
            result["ingestion"] = ingest
        print(json.dumps(result))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()
    return 0


def run_moves(args):
    """Explicit moves (north_star (1)): M reassign (b, t_new) pairs or M swaps
    (b1, b2) per step at the config's scale, evaluated by k_moves_warp (a warp per move) with the
    per-scenario statistics; one GPU.  Device-timed (graph: period masses + the moves kernel, L2
    flushed), e2e through Engine.eval_moves with host buffers, and the oracle port on all host
    cores for the same moves."""
    import torch

    from oracle import oracle
    from paper_2511_18296_b200 import synth
    from paper_2511_18296_b200.engine import Engine

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    c = build_inputs(args.config)
    bm, T, S = c["bm"], c["T"], c["S"]
    M = args.moves
    rng = synth.substream(3, "moves", args.workload)
    a = rng.integers(0, bm.n_blocks, M).astype(np.int32)
    b = (rng.integers(-1, T, M) if args.workload == "reassign" else rng.integers(0, bm.n_blocks, M)).astype(np.int32)
    eng = Engine.from_tables(bm, c["tables"], c["assign"])
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    assign_d = torch.from_numpy(c["assign"].astype(np.int32)).to(dev)
    a_d, b_d = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    out = {"feasible": torch.empty(M, dtype=torch.uint8, device=dev),
           "delta": torch.empty(M, dtype=torch.float64, device=dev),
           "exp_delta": torch.empty(M, dtype=torch.float64, device=dev),
           "cvar": torch.empty(M, dtype=torch.float64, device=dev),
           "global": torch.empty(2, dtype=torch.float64, device=dev)}
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    def step(sp):
        eng.set_schedule_device(assign_d, stream=sp, borrow=True)
        eng.eval_moves_device(a_d, b_d, out, args.workload, None, net=True, stream=sp)

    for _ in range(max(args.warmup, 3)):
        step(stream.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(torch.cuda.current_stream().cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(0) as clocks:
        for i in range(args.steps):
            flush.fill_(i)
            ev[i][0].record(stream)
            g.replay()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    t_ms = float(np.mean([x.elapsed_time(y) for x, y in ev]))
    # e2e: page-locked host arrays through the C ABI (upload schedule + moves, kernels, download
    # of all outputs into page-locked arrays)
    from paper_2511_18296_b200.engine import PinnedPool
    pool = PinnedPool()
    ha, hb, hs = pool.empty(M, np.int32), pool.empty(M, np.int32), pool.empty(bm.n_blocks, np.int32)
    ha[:], hb[:], hs[:] = a, b, c["assign"]
    hout = {"feasible": pool.empty(M, np.uint8), "delta": pool.empty(M, np.float64),
            "exp_delta": pool.empty(M, np.float64), "cvar": pool.empty(M, np.float64)}
    e2e = []
    res = None
    for i in range(args.warmup + min(args.steps, 100)):
        flush.fill_(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.set_schedule(hs)
        res = eng.eval_moves(ha, hb, args.workload, None, net=True, stats=True, out=hout)
        if i >= args.warmup:
            e2e.append(time.perf_counter() - t0)
    e2e_t = float(np.median(e2e))
    ref = None
    if not args.no_cpu_baseline:
        oracle.build()
        o = oracle.Oracle(bm, c["tables"].vmax, c["tables"].sigma)
        n_cpu = min(M, 50000)
        t0 = time.perf_counter()
        r = o.eval_moves(c["assign"], a[:n_cpu], b[:n_cpu], args.workload, None, net=True, stats=True)
        t_cpu = time.perf_counter() - t0
        ref = {"value": n_cpu * S / t_cpu, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{n_cpu} of {M} moves x {S} scenarios, oracle/oracle.c eval_moves, one core"}
        assert np.array_equal(r["feasible"], res["feasible"][:n_cpu]) and np.array_equal(
            r["delta"], res["delta"][:n_cpu]), "oracle parity on the bench moves"
    deg = 2.0 * bm.n_edges / bm.n_blocks
    nblk = 1 if args.workload == "reassign" else 2
    survey = M * nblk * (80 + 8 * deg) + 8 * M * nblk * S
    hbm, peak_kind = _peaks()
    print(json.dumps({
        "metric": METRIC, "workload": f"explicit {args.workload} moves", "value": M * S / (t_ms * 1e-3),
        "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
        "higher_is_better": True, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {M} explicit {args.workload} moves x {S} scenarios per step, "
                               "net mining cost, per-move delta + expected delta + CVaR10, argmax",
                   "blocks": bm.n_blocks, "periods": T, "scenarios": S, "moves_per_step": M,
                   "l2": "256 MiB flush write between timed GPU steps"},
        "feasible_moves": int(res["feasible"].sum()),
        "roofline": {"bound": "hbm", "achieved": survey / (t_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": survey / (t_ms * 1e-3) / 1e9 / hbm, "traffic": None,
                     "algorithmic_basis": "SURVEY §8(d) per move and block: 80 + 8*deg + 8*S (f64 values); "
                                          "step time (period masses + moves kernel)",
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
        "e2e": {"value": M * S / e2e_t, "unit": UNIT, "ms_per_step": e2e_t * 1e3,
                "h2d_bytes_per_step": int(c["assign"].size * 4 + 8 * M),
                "d2h_bytes_per_step": int(M * (1 + 8 + 8 + 8) + 16),
                "api": "Engine.set_schedule + Engine.eval_moves (PP_MEM_HOST, pinned)"},
        # period masses + (k_block_windows when the batch holds >= 2 moves per block) + k_moves_warp
        "gpu_launches": (3 if M >= 2 * bm.n_blocks else 2) * args.steps, "clocks": clocks.summary(),
        "cpu_baseline": ref, "best_move": res["best"]}))
    eng.close()
    pool.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=5.0)
    ap.add_argument("--no-python-ref", action="store_true", help="skip timing pitplan itself (baseline/_ref)")
    ap.add_argument("--ncu-traffic", type=float, default=None,
                    help="dram bytes per k_eval_warp launch from the committed ncu capture")
    ap.add_argument("--workload", default="candidates", choices=["candidates", "reassign", "swap"],
                    help="candidates: the headline evaluate_candidates_parallel batch; reassign / swap: "
                         "explicit moves (one GPU, a separate line)")
    ap.add_argument("--moves", type=int, default=250000)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "candidates":
        return run_moves(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
