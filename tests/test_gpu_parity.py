"""GPU parity: the sm_100a engine through the C ABI versus the reference's golden
vectors and the CPU oracle, bit for bit (integer, flag and index outputs exactly;
float64 values exactly -- the kernels never contract a multiply-add)."""

import numpy as np
import pytest

from paper_2511_18296_b200.engine import Engine
from paper_2511_18296_b200.model import BlockModel, ScenarioTables
from tests._fixtures import bm_from, config, load, same, tables_from

pytestmark = pytest.mark.gpu

KD = range(20)


def _check(res, store, q, trace=True):
    assert same(res["best_t"], store[q + "best_t"]), q
    assert same(res["best_val"], store[q + "best_val"]), q
    assert same(res["feasible"], store[q + "feasible"]), q
    g = store[q + "best"]
    if g[0] < 0:
        assert res["best"] is None, q
    else:
        assert res["best"] == (int(g[0]), int(g[1]), float(g[2])), q
    if trace:
        assert same(res["trace_val"], store[q + "trace_val"]), q
        assert same(res["trace_feas"], store[q + "trace_feas"]), q


def _same_res(a, b, keys):
    for k in keys:
        if k in a or k in b:
            assert same(a[k], b[k]), k
    assert a["best"] == b["best"]


@pytest.fixture(scope="module")
def small():
    return load("small")


@pytest.mark.parametrize("case", KD)
def test_kernel_determinism_cases(small, case):
    st, p = small, f"kd{case}_"
    eng = Engine.from_tables(bm_from(st, p), tables_from(st, p), st[p + "assign"])
    c = st[p + "cand"]
    _check(eng.eval_candidates(c, 0, trace=True), st, p + "s0_")
    _check(eng.eval_candidates(c, None, trace=True), st, p + "sN_")
    _check(eng.eval_candidates(c, None, net=True, trace=True), st, p + "net_")
    _check(eng.eval_candidates(c, 1, use_sigma=False, trace=True), st, p + "nosig_")
    _check(eng.eval_candidates(c, 0, literal=True, trace=True), st, p + "lit_")
    # candidate-order invariance of the selected move (test_evaluate.py:231-236)
    rev = eng.eval_candidates(c[::-1].copy(), None, trace=True)
    assert rev["best"] == eng.eval_candidates(c, None)["best"]
    eng.set_schedule(st[p + "assign2"])
    r = eng.eval_candidates(np.arange(27), None, net=True, trace=True, stats=True, scen=True)
    _check(r, st, p + "all_")
    assert same(r["scen_delta"], st[p + "all_scen_delta"])
    assert same(r["exp_delta"], st[p + "all_exp"])
    assert same(r["cvar"], st[p + "all_cvar"])
    eng.close()


@pytest.mark.parametrize("case", KD)
def test_feasibility_and_repair_cases(small, case):
    st, p = small, f"kd{case}_"
    eng = Engine.from_tables(bm_from(st, p), None)
    rand = st[p + "rand"]
    r = eng.check_feasible(rand)
    assert np.array_equal(r["pred_count"], st[p + "rand_pred"])
    assert same(r["excess"], st[p + "rand_excess"])
    assert same(r["violation"], st[p + "rand_viol"])
    rep, _ = eng.repair(rand, mode="push")
    assert np.array_equal(rep, st[p + "rand_repair"])
    fix, unm = eng.repair(rand, mode="unmine", unmined=True)
    assert np.array_equal(fix, st[p + "rand_unmine"])
    assert np.array_equal(unm.astype(bool), (rand != -1) & (fix == -1))
    eng.close()


def test_hand_cases(small):
    st = small
    for name in ("forced", "early", "infeas", "literal"):
        p = f"hand_{name}_"
        eng = Engine.from_tables(bm_from(st, p), ScenarioTables(st[p + "vmax"], None), st[p + "assign"])
        r = eng.eval_candidates(st[p + "cand"], 0, literal=bool(st[p + "literal"]), use_sigma=False, trace=True)
        _check(r, st, p)
        eng.close()
    for name in ("prec", "unmined_parent", "same", "capacity", "empty"):
        p = f"feas_{name}_"
        eng = Engine.from_tables(bm_from(st, p), None)
        r = eng.check_feasible(st[p + "assign"])
        exp = st[p + "out"]
        assert (int(r["pred_count"][0]), float(r["excess"][0]), float(r["violation"][0])) == (
            int(exp[0]), float(exp[1]), float(exp[2])), name
        eng.close()


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_batches_match_reference(oracle_lib, name):
    st = load(name.lower())
    c = config(name)
    if not c["golden_ok"]:
        pytest.skip("this host's numpy rebuilds different input bits; oracle parity covers it")
    tables = ScenarioTables(c["vmax"], c["sigma"])
    eng = Engine.from_tables(c["bm"], tables)
    o = oracle_lib.Oracle(c["bm"], c["vmax"], c["sigma"])
    trace = name == "C1"
    for sname in ("full", "greedy"):
        a = c["assign"] if sname == "full" else c["greedy"]
        q = f"{name}_{sname}_"
        eng.set_schedule(a)
        _, pm = eng.get_schedule()
        assert same(pm, o.period_mass(a)), "period mass is not numpy-pairwise exact"
        _check(eng.eval_candidates(c["cand"], None, trace=trace), st, q + "sN_", trace)
        _check(eng.eval_candidates(c["cand"], None, net=True, trace=trace), st, q + "net_", trace)
        _check(eng.eval_candidates(c["cand"], 0, trace=trace), st, q + "s0_", trace)
        f = st[q + "feas"]
        r = eng.check_feasible(a)
        assert (int(r["pred_count"][0]), float(r["excess"][0]), float(r["violation"][0])) == (
            int(f[0]), float(f[1]), float(f[2]))
    eng.set_schedule(c["assign"])
    got = eng.eval_candidates(c["cand"], None, net=True, trace=True, stats=True, scen=True)
    ref = o.eval_candidates(c["assign"], c["cand"], None, net=True, trace=True, stats=True, scen=True,
                            nthreads=8)
    _same_res(got, ref, ("best_t", "best_val", "feasible", "trace_val", "trace_feas", "exp_delta", "cvar",
                         "scen_delta"))
    if name == "C1":
        sub = c["cand"][:200]
        r = eng.eval_candidates(sub, None, net=True, stats=True, scen=True)
        assert same(r["scen_delta"], st["C1_full_sub_scen_delta"])
        assert same(r["exp_delta"], st["C1_full_sub_exp"])
        assert same(r["cvar"], st["C1_full_sub_cvar"])
    rep, _ = eng.repair(st[f"{name}_repair_in"], mode="push")
    assert np.array_equal(rep, st[f"{name}_repair_out"])
    eng.close()


def _rand_instance(seed, n=(6, 5, 4), T=7, S=9, cf=0.5):
    from paper_2511_18296_b200 import synth
    from paper_2511_18296_b200.model import scenario_values

    nx, ny, nz = n
    bm = synth.generate_block_model(nx * ny * nz, n, T, 2, seed=seed, n_rock_types=1, capacity_factor=cf)
    grades = synth.sample_lognormal(bm, S, 0.4, seed=seed + 1)
    sigma = synth.uncertainty_sigma(bm, grades)
    return bm, scenario_values(bm, grades), sigma


@pytest.mark.parametrize("T,S", [(1, 1), (3, 7), (7, 9), (9, 20), (8, 25), (12, 35), (10, 45), (20, 55), (16, 64),
                                 (17, 129), (32, 200), (33, 40), (40, 300), (5, 1000)])
def test_shapes_against_oracle(oracle_lib, T, S):
    """Group widths 4..32, the multi-slot path (T > 32), single- and multi-leaf pairwise
    plans (S up to 1000), CVaR sample counts 1..100."""
    bm, vmax, sigma = _rand_instance(11 + T + S, T=T, S=S)
    rng = np.random.default_rng(T * 1000 + S)
    from paper_2511_18296_b200 import synth

    assign = synth.full_greedy(bm)
    assign[rng.random(assign.size) < 0.2] = -1  # ragged: some unmined blocks
    cand = rng.integers(0, bm.n_blocks, size=157).astype(np.int32)
    cand[:5] = cand[5]  # duplicates
    eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
    o = oracle_lib.Oracle(bm, vmax, sigma)
    keys = ("best_t", "best_val", "feasible", "trace_val", "trace_feas", "exp_delta", "cvar", "scen_delta")
    for s in (None, S - 1):
        for net in (False, True):
            got = eng.eval_candidates(cand, s, net=net, trace=True, stats=True, scen=True)
            ref = o.eval_candidates(assign, cand, s, net=net, trace=True, stats=True, scen=True)
            _same_res(got, ref, keys)
    got = eng.eval_candidates(cand, None, use_sigma=False, stats=True)
    ref = o.eval_candidates(assign, cand, None, use_sigma=False, stats=True)
    _same_res(got, ref, ("best_t", "best_val", "feasible", "exp_delta", "cvar"))
    eng.close()


def test_setup_uploads_ordered_before_first_eval(oracle_lib):
    """Fresh engines evaluated right after set_scenarios: the value table (tens of MB, pageable)
    must have landed before the first kernel on the context's non-blocking stream reads it."""
    from paper_2511_18296_b200 import synth

    bm, vmax, sigma = _rand_instance(3, n=(40, 30, 12), T=12, S=300)
    assign = synth.full_greedy(bm)
    cand = np.random.default_rng(1).integers(0, bm.n_blocks, size=4096).astype(np.int32)
    o = oracle_lib.Oracle(bm, vmax, sigma)
    ref = o.eval_candidates(assign, cand, None)
    for _ in range(8):
        eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
        got = eng.eval_candidates(cand, None)
        eng.close()
        _same_res(got, ref, ("best_t", "best_val", "feasible"))


def test_explicit_moves_against_oracle(oracle_lib):
    bm, vmax, sigma = _rand_instance(5, n=(12, 10, 6), T=9, S=20, cf=0.45)
    from paper_2511_18296_b200 import synth

    rng = np.random.default_rng(3)
    assign = synth.full_greedy(bm)
    eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
    o = oracle_lib.Oracle(bm, vmax, sigma)
    M = 5000
    b = rng.integers(0, bm.n_blocks, M).astype(np.int32)
    t = rng.integers(-1, bm.n_periods, M).astype(np.int32)
    keys = ("feasible", "delta", "exp_delta", "cvar", "scen_delta")
    for net in (False, True):
        for s in (None, 3):
            got = eng.eval_moves(b, t, "reassign", s, net=net, stats=True, scen=True)
            ref = o.eval_moves(assign, b, t, "reassign", s, net=net, stats=True, scen=True)
            _same_res(got, ref, keys)
    # M = 5000 >= 2 B takes the per-block windows (k_block_windows); M = 500 the per-move ones
    got = eng.eval_moves(b[:500].copy(), t[:500].copy(), "reassign", None, net=True, stats=True, scen=True)
    ref = o.eval_moves(assign, b[:500].copy(), t[:500].copy(), "reassign", None, net=True, stats=True, scen=True)
    _same_res(got, ref, keys)
    b2 = rng.integers(0, bm.n_blocks, M).astype(np.int32)
    got = eng.eval_moves(b, b2, "swap", None, net=True, stats=True, scen=True)
    ref = o.eval_moves(assign, b, b2, "swap", None, net=True, stats=True, scen=True)
    _same_res(got, ref, keys)
    assert got["feasible"].sum() > 0
    # swaps between neighbours (the partner seen at the other's period): every block with each of
    # its neighbours, through the per-block windows (M >= 2 B) and the per-move ones (M < 2 B)
    pp_, pi_, sp_, si_ = bm.csr()
    pa, pb = [], []
    for x in range(bm.n_blocks):
        for y in list(pi_[pp_[x]:pp_[x + 1]]) + list(si_[sp_[x]:sp_[x + 1]]):
            pa.append(x)
            pb.append(int(y))
    pa, pb = np.asarray(pa, np.int32), np.asarray(pb, np.int32)
    assert pa.size >= 2 * bm.n_blocks
    for lo_, hi_ in ((0, pa.size), (0, 400)):
        got = eng.eval_moves(pa[lo_:hi_].copy(), pb[lo_:hi_].copy(), "swap", None, net=True, stats=True)
        ref = o.eval_moves(assign, pa[lo_:hi_].copy(), pb[lo_:hi_].copy(), "swap", None, net=True, stats=True)
        _same_res(got, ref, ("feasible", "delta", "exp_delta", "cvar"))
    eng.close()


def test_population_feasibility_and_repair(oracle_lib):
    c = config("C1")
    eng = Engine.from_tables(c["bm"], None)
    o = oracle_lib.Oracle(c["bm"])
    rng = np.random.default_rng(9)
    pop = np.stack([c["assign"], c["greedy"]] + [rng.integers(-1, c["T"], c["bm"].n_blocks) for _ in range(6)])
    r = eng.check_feasible(pop)
    for k in range(pop.shape[0]):
        pc, ex, vi = o.check_feasible(pop[k])
        assert (int(r["pred_count"][k]), float(r["excess"][k]), float(r["violation"][k])) == (pc, ex, vi)
        assert same(r["period_mass"][k], o.period_mass(pop[k]))
    rep, _ = eng.repair(pop, mode="push")
    fix, unm = eng.repair(pop, mode="unmine", unmined=True)
    for k in range(pop.shape[0]):
        assert np.array_equal(rep[k], o.precedence_repair(pop[k]))
        f, u = o.unmine_fixpoint(pop[k])
        assert np.array_equal(fix[k], f)
        assert np.array_equal(unm[k], u)
    eng.close()


def test_apply_moves_and_period_mass(oracle_lib):
    c = config("C1")
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["greedy"])
    o = oracle_lib.Oracle(c["bm"], c["vmax"], c["sigma"])
    a = c["greedy"].copy()
    rng = np.random.default_rng(4)
    for _ in range(5):
        b = rng.integers(0, a.size, 7)
        t = rng.integers(-1, c["T"], 7)
        eng.apply_moves(b, t)
        for bb, tt in zip(b, t):
            a[bb] = tt
        got_a, pm = eng.get_schedule()
        assert np.array_equal(got_a, a)
        assert same(pm, o.period_mass(a))
        r = eng.eval_candidates(c["cand"], None, net=True)
        ref = o.eval_candidates(a, c["cand"], None, net=True)
        _same_res(r, ref, ("best_t", "best_val", "feasible"))
    eng.close()


def test_device_buffers_match_host_path():
    torch = pytest.importorskip("torch")
    c = config("C1")
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["assign"])
    host = eng.eval_candidates(c["cand"], None, net=True, trace=True, stats=True, scen=True)
    dev = torch.device("cuda:0")
    C, T, S = c["cand"].size, c["T"], c["S"]
    cand = torch.from_numpy(c["cand"]).to(dev)
    out = {
        "best_t": torch.empty(C, dtype=torch.int32, device=dev),
        "best_val": torch.empty(C, dtype=torch.float64, device=dev),
        "feasible": torch.empty(C, dtype=torch.uint8, device=dev),
        "trace_val": torch.empty(C, T, dtype=torch.float64, device=dev),
        "trace_feas": torch.empty(C, T, dtype=torch.uint8, device=dev),
        "exp_delta": torch.empty(C, T, dtype=torch.float64, device=dev),
        "cvar": torch.empty(C, T, dtype=torch.float64, device=dev),
        "scen_delta": torch.empty(C, S, T, dtype=torch.float32, device=dev),
        "global": torch.empty(2, dtype=torch.float64, device=dev),
    }
    stream = torch.cuda.Stream(dev).cuda_stream  # explicit stream (0 = the context's own)
    eng.set_schedule_device(torch.from_numpy(c["assign"].astype(np.int32)).to(dev), stream=stream)
    eng.eval_candidates_device(cand, out, None, net=True, stream=stream)
    torch.cuda.synchronize()
    for k in ("best_t", "best_val", "feasible", "trace_val", "trace_feas", "exp_delta", "cvar", "scen_delta"):
        assert same(out[k].cpu().numpy(), host[k]), k
    g = out["global"].cpu().numpy()
    gi = g.view(np.int32)
    assert (int(gi[2]), int(gi[3]), float(g[0])) == host["best"]
    eng.close()


def test_empty_and_degenerate_inputs(oracle_lib):
    c = config("C1")
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), np.full(c["bm"].n_blocks, -1))
    r = eng.eval_candidates(np.zeros(0, np.int32), None, stats=True)
    assert r["best"] is None and r["best_t"].size == 0
    # empty schedule: only surface blocks are placeable
    o = oracle_lib.Oracle(c["bm"], c["vmax"], c["sigma"])
    allc = np.arange(c["bm"].n_blocks, dtype=np.int32)
    got = eng.eval_candidates(allc, None, trace=True)
    ref = o.eval_candidates(np.full(c["bm"].n_blocks, -1), allc, None, trace=True)
    _same_res(got, ref, ("best_t", "best_val", "feasible", "trace_val", "trace_feas"))
    eng.close()


def test_errors_are_raised_not_fallen_back():
    from paper_2511_18296_b200.errors import InvalidArgs, PitplanError

    c = config("C1")
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["assign"])
    with pytest.raises(InvalidArgs):
        eng.eval_candidates(np.array([c["bm"].n_blocks]), None)
    with pytest.raises(InvalidArgs):
        eng.eval_candidates(np.array([0]), c["S"])
    # out-of-range periods: range-checked on the device, reported by the next host-mode call
    bad = np.full(c["bm"].n_blocks, c["T"])
    with pytest.raises(InvalidArgs):
        eng.set_schedule(bad)
        eng.eval_candidates(c["cand"], None, net=True)
    with pytest.raises(PitplanError):  # no schedule until the next set_schedule
        eng.eval_candidates(c["cand"], None)
    bad[:] = c["assign"]
    bad[17] = -2
    with pytest.raises(InvalidArgs):
        eng.set_schedule(bad)
        eng.get_schedule()
    eng.set_schedule(c["assign"])
    assert eng.eval_candidates(c["cand"], None, net=True)["best"] is not None
    fresh = Engine(0)
    with pytest.raises(PitplanError):
        fresh.eval_candidates(np.array([0]), None)
    fresh.close()
    eng.close()


def test_enpv_table_matches_reference(oracle_lib, small):
    for case in range(0, 20, 4):
        p = f"kd{case}_"
        eng = Engine.from_tables(bm_from(small, p), tables_from(small, p))
        assert same(eng.enpv_table(True), small[p + "enpv"])
        assert same(eng.enpv_table(False), small[p + "enpv_nosig"])
        eng.close()
    c = config("C1")
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]))
    assert same(eng.enpv_table(True), load("c1")["C1_enpv"])
    o = oracle_lib.Oracle(c["bm"], c["vmax"], c["sigma"])
    assert same(eng.enpv_table(True, factored=True), o.enpv_table(True, factored=True))
    eng.close()


def _flat_bm(B, T, seed):
    from paper_2511_18296_b200.model import BlockModel

    rng = np.random.default_rng(seed)
    z = np.zeros(B)
    return BlockModel(n_blocks=B, n_periods=T, edges_i=np.zeros(0, np.int32), edges_j=np.zeros(0, np.int32),
                      mass=rng.lognormal(8.0, 1.5, B), cost=np.zeros((B, T)), capacity=np.full(T, 1e30),
                      discount_rate=0.08, coords=np.zeros((B, 3)), alteration=z, structural=z,
                      dist_intrusion=z, base_grade=z)


@pytest.mark.parametrize("B,T", [(1, 1), (100, 3), (8192, 15), (8193, 16), (16385, 9), (50000, 15),
                                 (65536, 8), (65536, 16), (65537, 15), (70000, 17), (5000, 40),
                                 (131072, 20), (131073, 20), (200000, 20), (200000, 1), (245760, 32),
                                 (100000, 33), (245761, 15)])
def test_period_mass_paths(oracle_lib, B, T):
    """numpy-pairwise period masses on both device paths (the cluster path for B <= 245,760 and
    T <= 32 -- registers up to 8 blocks per lane, the count + scatter passes above; slots in
    shared memory or the global spill; the one-level pre-fold for periods above ~123k blocks --
    and the look-back path otherwise): uniform, skewed (one period holding almost every block,
    the deepest pairwise tree), all unmined, ragged tails."""
    bm = _flat_bm(B, T, B + T)
    rng = np.random.default_rng(B * 7 + T)
    pop = [rng.integers(-1, T, B), np.where(rng.random(B) < 0.97, T - 1, rng.integers(-1, T, B)),
           np.full(B, -1), np.full(B, 0), (np.arange(B) * 7919) % (T + 1) - 1]
    pop = np.stack(pop).astype(np.int32)
    eng = Engine.from_tables(bm, None)
    o = oracle_lib.Oracle(bm)
    r = eng.check_feasible(pop)
    for k in range(pop.shape[0]):
        assert same(r["period_mass"][k], o.period_mass(pop[k])), k
    for k in range(pop.shape[0]):  # single-schedule path (pm refresh behind set_schedule)
        eng.set_schedule(pop[k])
        _, pm = eng.get_schedule()
        assert same(pm, o.period_mass(pop[k])), k
    eng.close()


def _pairs_match_dense(pr, ref):
    """The sparse pair list equals the dense reference restricted to the feasible moves."""
    ci, ti = np.nonzero(ref["trace_feas"] == 1)
    order = np.lexsort((pr["period"], pr["cand"]))
    assert np.array_equal(pr["cand"][order], ci) and np.array_equal(pr["period"][order], ti)
    assert same(pr["exp"][order], ref["exp_delta"][ci, ti])
    assert same(pr["cvar"][order], ref["cvar"][ci, ti])


@pytest.mark.parametrize("T,S", [(7, 9), (15, 20), (40, 30), (9, 200)])
def test_sparse_pairs_against_oracle(oracle_lib, T, S):
    """pairs=True: the warp kernel (T <= 32, S <= 128) and the general kernel (T > 32 or
    S > 128) append every feasible move's expected delta and CVaR exactly once."""
    bm, vmax, sigma = _rand_instance(23 + T + S, n=(8, 7, 5), T=T, S=S)
    from paper_2511_18296_b200 import synth

    assign = synth.full_greedy(bm)
    rng = np.random.default_rng(T + S)
    assign[rng.random(assign.size) < 0.1] = -1
    cand = rng.integers(0, bm.n_blocks, size=301).astype(np.int32)
    eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
    o = oracle_lib.Oracle(bm, vmax, sigma)
    for net in (False, True):
        got = eng.eval_candidates(cand, None, net=net, pairs=True)
        ref = o.eval_candidates(assign, cand, None, net=net, trace=True, stats=True)
        _same_res(got, ref, ("best_t", "best_val", "feasible"))
        assert got["pairs"]["cand"].size == int(ref["trace_feas"].sum()) > 0
        _pairs_match_dense(got["pairs"], ref)
    eng.close()


def test_sparse_pairs_c2_and_device_mode(oracle_lib):
    import torch

    c = config("C2")
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["assign"])
    o = oracle_lib.Oracle(c["bm"], c["vmax"], c["sigma"])
    ref = o.eval_candidates(c["assign"], c["cand"], None, net=True, trace=True, stats=True, nthreads=8)
    got = eng.eval_candidates(c["cand"], None, net=True, pairs=True)
    _pairs_match_dense(got["pairs"], ref)
    C, T = c["C"], c["T"]
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    out = {"best_t": torch.empty(C, dtype=torch.int32, device=dev),
           "best_val": torch.empty(C, dtype=torch.float64, device=dev),
           "feasible": torch.empty(C, dtype=torch.uint8, device=dev),
           "global": torch.empty(2, dtype=torch.float64, device=dev),
           "pair_cand": torch.empty(C * T, dtype=torch.int32, device=dev),
           "pair_period": torch.empty(C * T, dtype=torch.int32, device=dev),
           "pair_exp": torch.empty(C * T, dtype=torch.float64, device=dev),
           "pair_cvar": torch.empty(C * T, dtype=torch.float64, device=dev),
           "n_pairs": torch.zeros(1, dtype=torch.int32, device=dev)}
    with torch.cuda.stream(st):
        cand_d = torch.from_numpy(c["cand"]).to(dev)
        eng.eval_candidates_device(cand_d, out, None, net=True, stream=st.cuda_stream)
    st.synchronize()
    n = int(out["n_pairs"].item())
    pr = {"cand": out["pair_cand"][:n].cpu().numpy(), "period": out["pair_period"][:n].cpu().numpy(),
          "exp": out["pair_exp"][:n].cpu().numpy(), "cvar": out["pair_cvar"][:n].cpu().numpy()}
    _pairs_match_dense(pr, ref)
    eng.close()


@pytest.mark.parametrize("case", [0, 5, 11, 19])
def test_destroy_step_small(small, case):
    """lns_repair's unmine fixpoint + over-capacity ejection (hybrid.py:199-235) against the
    reference's lns_repair(max_iters=0) on random schedules, destroy_fraction 0 and 0.3."""
    p = f"kd{case}_"
    eng = Engine.from_tables(bm_from(small, p), None)
    for tag, df in (("d0", 0.0), ("d3", 0.3)):
        out, _ = eng.lns_destroy(small[p + "rand"], small[p + "mean_grade"], df)
        assert np.array_equal(out, small[p + f"rand_destroy_{tag}"]), tag
    eng.close()


def test_destroy_step_c1(oracle_lib):
    st = load("c1")
    c = config("C1")
    eng = Engine.from_tables(c["bm"], None)
    o = oracle_lib.Oracle(c["bm"])
    ins = st["C1_destroy_in"]
    for tag, df in (("d0", 0.0), ("d25", 0.25)):
        out, pool = eng.lns_destroy(ins, st["C1_mean_grade"], df)  # all schedules in one batch
        assert np.array_equal(out, st[f"C1_destroy_{tag}"]), tag
        for k in range(ins.shape[0]):
            f, u = o.unmine_fixpoint(ins[k])
            ref, e = o.eject(f, st["C1_mean_grade"], df)
            assert np.array_equal(pool[k], (u | e)), (tag, k)
    eng.close()


@pytest.mark.parametrize("case", [0, 3, 8, 14, 19])
def test_lns_repair_dropin_small(small, case):
    """The whole lns_repair (hybrid.py:169-274) through the drop-in: device destroy step and
    insertion evaluations, restated similarity ranking; equal to the reference's runs."""
    from paper_2511_18296_b200 import evaluate as dropin
    from paper_2511_18296_b200.model import Schedule

    p = f"kd{case}_"
    bm = bm_from(small, p)
    tables = ScenarioTables(small[p + "vmax"], small[p + "sigma"], grades=small[p + "grades"])
    variants = {"a": dict(max_iters=50),
                "b": dict(max_iters=50, destroy_fraction=0.3, net_mining_cost=True),
                "c": dict(max_iters=50, realism_threshold=0.95, candidate_width=4)}
    for tag, kw in variants.items():
        for k in range(2):
            out = dropin.lns_repair(bm, Schedule(small[p + "rand"][k]), [0, 5], tables, True, **kw)
            assert np.array_equal(out.assignment, small[p + f"lns_{tag}"][k]), (tag, k)
    dropin.clear_cache()


def test_lns_repair_dropin_c1():
    from paper_2511_18296_b200 import evaluate as dropin
    from paper_2511_18296_b200.model import Schedule

    st = load("c1")
    c = config("C1")
    tables = ScenarioTables(c["vmax"], c["sigma"], grades=st["C1_grades"])
    out = dropin.lns_repair(c["bm"], Schedule(st["C1_destroy_in"][0]), [], tables, True, max_iters=40,
                            destroy_fraction=0.1)
    assert np.array_equal(out.assignment, st["C1_lns"])
    dropin.clear_cache()


@pytest.mark.parametrize("case", range(0, 20, 3))
def test_npv_relaxed_small(small, case):
    """ScheduleEvaluator.npv_relaxed / per_scenario_npv on the device (evaluate.py:166-183,
    222-258), bit-exact against the reference, population of 5 schedules in one call."""
    p = f"kd{case}_"
    bm = bm_from(small, p)
    eng = Engine.from_tables(bm, tables_from(small, p))
    pop = small[p + "npv_pop"]
    npv, ps = eng.npv_relaxed(pop, per_scenario=True)
    assert same(npv, small[p + "npv"])
    assert same(ps, small[p + "npv_scen"])
    assert same(eng.npv_relaxed(pop, use_sigma=False), small[p + "npv_nosig"])
    eng.close()


def test_npv_relaxed_c1(oracle_lib):
    st = load("c1")
    c = config("C1")
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]))
    npv, ps = eng.npv_relaxed(st["C1_npv_pop"], per_scenario=True)
    assert same(npv, st["C1_npv"])
    assert same(ps, st["C1_npv_scen"])
    eng.close()


def test_npv_relaxed_c2_against_oracle(oracle_lib):
    c = config("C2")
    bm = c["bm"]
    eng = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"]))
    o = oracle_lib.Oracle(bm, c["vmax"], c["sigma"])
    pop = np.stack([c["assign"], c["greedy"]])
    npv, ps = eng.npv_relaxed(pop, per_scenario=True)
    for k in range(2):
        v, pr = o.npv_relaxed(pop[k], bm.plant_hours, bm.mode_rates[0])
        assert npv[k] == v and np.array_equal(ps[k], pr), k
    eng.close()


def test_schedule_evaluator_dropin(small):
    """evaluate.ScheduleEvaluator (the drop-in class) on the device fast path, equal to the
    reference's npv_relaxed / per_scenario_npv."""
    from paper_2511_18296_b200 import evaluate as dropin
    from paper_2511_18296_b200.model import Schedule

    for case in (2, 9):
        p = f"kd{case}_"
        bm = bm_from(small, p)
        ev = dropin.ScheduleEvaluator(bm, tables_from(small, p), True)
        for k, a in enumerate(small[p + "npv_pop"]):
            assert ev.npv_relaxed(Schedule(a)) == small[p + "npv"][k]
            assert np.array_equal(ev.per_scenario_npv(Schedule(a)), small[p + "npv_scen"][k])
    dropin.clear_cache()


@pytest.mark.parametrize("name", ["p8", "p27", "p512"])
def test_polish_schedule_dropin(small, name):
    """polish_schedule (hybrid.py:326-490) through the drop-in: options batched on the device,
    same final schedule as the reference (joint insertion at 8 blocks, pair swaps and 1-1 exchanges
    at 27, single-block sweeps at 512)."""
    from paper_2511_18296_b200 import evaluate as dropin
    from paper_2511_18296_b200.model import Schedule

    p = f"{name}_"
    bm = bm_from(small, p)
    tables = tables_from(small, p)
    ev = dropin.ScheduleEvaluator(bm, tables, True)
    for k in range(small[p + "start"].shape[0]):
        out = dropin.polish_schedule(bm, ev, Schedule(small[p + "start"][k].copy()),
                                     max_sweeps=int(small[p + "sweeps"]))
        assert np.array_equal(out.assignment, small[p + "out"][k]), k
    dropin.clear_cache()


def test_npv_moves_equal_full_recompute():
    """pp_npv_moves (two periods re-solved per move) equals pp_npv_relaxed of each modified
    schedule bit for bit: reassign, unmine, mine, same-period moves."""
    c = config("C1")
    bm = c["bm"]
    eng = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"]))
    a = c["greedy"].copy()
    rng = np.random.default_rng(12)
    blocks = rng.integers(0, bm.n_blocks, 40).astype(np.int32)
    periods = rng.integers(-1, bm.n_periods, 40).astype(np.int32)
    periods[:3] = a[blocks[:3]]  # no-op moves
    for use_sigma in (True, False):
        got = eng.npv_moves(a, blocks, periods, use_sigma=use_sigma)
        batch = np.repeat(a[None, :], blocks.size, axis=0)
        batch[np.arange(blocks.size), blocks] = periods
        ref = eng.npv_relaxed(batch, use_sigma=use_sigma)
        assert same(got, ref)
    eng.close()


def test_npv_moves_base_cache_invalidation():
    """pp_npv_moves keeps the base schedule's stage-2 results between calls: a sequence of calls
    alternating bases, interleaved pp_npv_relaxed batches (which reuse the buffers) and a new
    plant table must each equal a full recompute."""
    c = config("C1")
    bm = c["bm"]
    eng = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"]))
    rng = np.random.default_rng(5)
    bases = [c["greedy"].copy(), c["assign"].copy()]

    def check(a, m=12):
        blocks = rng.integers(0, bm.n_blocks, m).astype(np.int32)
        periods = rng.integers(-1, bm.n_periods, m).astype(np.int32)
        got = eng.npv_moves(a, blocks, periods)
        batch = np.repeat(a[None, :], m, axis=0)
        batch[np.arange(m), blocks] = periods
        assert same(got, eng.npv_relaxed(batch))

    for k in (0, 0, 1, 0, 1, 1):
        check(bases[k])
        check(bases[k], m=3)  # same base, fewer moves: a cache hit
    a = bases[0].copy()
    a[np.flatnonzero(a >= 0)[:5]] = -1  # the same array object, new contents
    check(a)
    check(bases[0])
    hours = np.asarray(bm.plant_hours, dtype=np.float64) * 0.5
    eng.set_plant(hours)
    check(bases[0])
    eng.close()


@pytest.mark.parametrize("name", ("q8", "q27", "q512", "q512n", "qC1", "qC1big"))
def test_price_greedy_matches_reference(oracle_lib, name):
    """pp_price_greedy against the reference's price_column sequences (colgen.py:236-254)."""
    st = load("price")
    p = f"{name}_"
    bm = bm_from(st, p)
    eng = Engine.from_tables(bm, None)
    a, ex = eng.price_greedy(st[p + "score"], st[p + "cap"], int(st[p + "node_cap"]))
    eng.close()
    assert np.array_equal(a, st[p + "assign"])
    _, ex_ref = oracle_lib.Oracle(bm).price_greedy(st[p + "score"], st[p + "cap"], int(st[p + "node_cap"]))
    assert ex == ex_ref


def test_price_greedy_near_ties_against_oracle(oracle_lib):
    """Scores with exact ties, ties within the reference's 1e-12 tolerance and tiny magnitudes
    (where the tolerance is not absorbed by rounding) take the sequential replay."""
    bm, _, _ = _rand_instance(21, n=(10, 10, 8), T=5, S=2, cf=0.4)
    B, T = bm.n_blocks, bm.n_periods
    rng = np.random.default_rng(4)
    o = oracle_lib.Oracle(bm)
    eng = Engine.from_tables(bm, None)
    cap = np.asarray(bm.capacity, dtype=np.float64)
    for kind in range(4):
        if kind == 0:  # few distinct values: exact ties everywhere
            score = rng.integers(-2, 6, size=(B, T)).astype(np.float64)
        elif kind == 1:  # near-ties below the tolerance
            score = 1e-9 + rng.integers(0, 4, size=(B, T)) * 4e-13
        elif kind == 2:  # around the 1e-12 threshold itself
            score = rng.choice([0.0, 5e-13, 1e-12, 1.0000000001e-12, 2e-12, 3e-12], size=(B, T))
        else:  # distinct values, large node_cap
            score = rng.normal(0.0, 1.0, size=(B, T))
        for node_cap in (50, 10 ** 7):
            a, ex = eng.price_greedy(score, cap, node_cap)
            ar, exr = o.price_greedy(score, cap, node_cap)
            assert np.array_equal(a, ar), (kind, node_cap)
            assert ex == exr, (kind, node_cap)
    eng.close()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_configs_against_oracle(oracle_lib, name):
    """C3 (S = 200, the many-scenario statistics kernel, capacity binding) and C4 (200k
    blocks, 1M moves) at their full bench sizes: every per-candidate output, the dense
    statistics, the sparse pairs and the selected move against the oracle; the selected move
    is invariant under a permutation of the candidates (test_evaluate.py:231-236)."""
    c = config(name)
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["assign"])
    o = oracle_lib.Oracle(c["bm"], c["vmax"], c["sigma"])
    ref = o.eval_candidates(c["assign"], c["cand"], None, net=True, trace=True, stats=True, nthreads=8)
    got = eng.eval_candidates(c["cand"], None, net=True, trace=True, stats=True)
    _same_res(got, ref, ("best_t", "best_val", "feasible", "trace_val", "trace_feas", "exp_delta", "cvar"))
    _pairs_match_dense(eng.eval_candidates(c["cand"], None, net=True, pairs=True)["pairs"], ref)
    perm = np.random.default_rng(7).permutation(c["cand"].size)
    assert eng.eval_candidates(c["cand"][perm].copy(), None, net=True)["best"] == got["best"]
    eng.close()


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_pinned_copy_out_matches_pageable(name):
    """Page-locked outputs take the one-launch copy-out (k_copy_out, launched under programmatic
    dependent launch behind k_eval_warp, which triggers it from its epilogue): at C2 (one wave)
    and C4 (1,563 CTAs, several waves) every output and the sparse pairs equal the pageable
    path's cudaMemcpyAsync copies, over repeated calls with the same arrays (the cached argument
    block)."""
    from paper_2511_18296_b200.engine import PinnedPool
    c = config(name)
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["assign"])
    C, T = c["cand"].size, c["T"]
    ref = eng.eval_candidates(c["cand"], None, net=True, trace=True, stats=True, pairs=True)
    pool = PinnedPool()
    out = {"best_t": pool.empty(C, np.int32), "best_val": pool.empty(C, np.float64),
           "feasible": pool.empty(C, np.uint8), "trace_val": pool.empty((C, T), np.float64),
           "trace_feas": pool.empty((C, T), np.uint8), "exp_delta": pool.empty((C, T), np.float64),
           "cvar": pool.empty((C, T), np.float64), "pair_cand": pool.empty(C * T, np.int32),
           "pair_period": pool.empty(C * T, np.int32), "pair_exp": pool.empty(C * T, np.float64),
           "pair_cvar": pool.empty(C * T, np.float64), "n_pairs": pool.empty(1, np.int32)}
    hc = pool.empty(C, np.int32)  # page-locked ids: read in place by k_eval_warp (no copy-in)
    hc[:] = c["cand"]
    try:
        for rep in range(3):
            for v in out.values():
                v.view(np.uint8)[...] = 0xA5  # stale bytes must be overwritten
            got = eng.eval_candidates(hc if rep else c["cand"], None, net=True, trace=True, stats=True, pairs=True,
                                      out=out)
            _same_res(got, ref, ("best_t", "best_val", "feasible", "trace_val", "trace_feas", "exp_delta", "cvar"))
            assert got["best"] == ref["best"], rep
            n = ref["pairs"]["cand"].size
            assert got["pairs"]["cand"].size == n, rep
            ka = np.lexsort((ref["pairs"]["period"], ref["pairs"]["cand"]))
            kb = np.lexsort((got["pairs"]["period"], got["pairs"]["cand"]))
            for k in ("cand", "period", "exp", "cvar"):
                assert same(got["pairs"][k][kb], ref["pairs"][k][ka]), (rep, k)
        hc[C // 2] = c["bm"].n_blocks  # an out-of-range id in the page-locked list is still reported
        with pytest.raises(Exception, match="out of range"):
            eng.eval_candidates(hc, None, net=True, pairs=True, out=out)
        hc[C // 2] = c["cand"][C // 2]
        assert eng.eval_candidates(hc, None, net=True, trace=True, stats=True, pairs=True, out=out)["best"] == ref["best"]
    finally:
        eng.close()
        pool.close()


def test_repeated_host_calls_replay_graph_with_fresh_inputs():
    """A host-mode call repeated with the same page-locked arrays replays one cached graph: the
    schedule and the ids are re-read on every replay (two schedules alternating in one page-locked
    buffer, the ids changed in place), and freeing / re-allocating page-locked buffers invalidates
    the cached device mappings (the registry generation is part of the key)."""
    from paper_2511_18296_b200.engine import PinnedPool
    c = config("C1")
    bm = c["bm"]
    eng = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"]), c["assign"])
    C, T = c["cand"].size, c["T"]
    a0 = c["assign"].astype(np.int32)
    a1 = a0.copy()
    a1[(a1 >= 0) & (np.arange(a1.size) % 7 == 0)] = -1  # some blocks unmined: other windows, masses
    rng = np.random.default_rng(11)
    ids = [c["cand"].copy(), rng.permutation(c["cand"]).astype(np.int32)]
    refs = {}
    for ia, a in enumerate((a0, a1)):
        for ic, cd in enumerate(ids):
            eng.set_schedule(a)
            refs[ia, ic] = eng.eval_candidates(cd, None, net=True, stats=True, pairs=True)
    for round_ in range(2):
        pool = PinnedPool()
        hs = pool.empty(bm.n_blocks, np.int32)
        hc = pool.empty(C, np.int32)
        out = {"best_t": pool.empty(C, np.int32), "best_val": pool.empty(C, np.float64),
               "feasible": pool.empty(C, np.uint8), "exp_delta": pool.empty((C, T), np.float64),
               "cvar": pool.empty((C, T), np.float64), "pair_cand": pool.empty(C * T, np.int32),
               "pair_period": pool.empty(C * T, np.int32), "pair_exp": pool.empty(C * T, np.float64),
               "pair_cvar": pool.empty(C * T, np.float64), "n_pairs": pool.empty(1, np.int32)}
        for step in range(8):
            ia, ic = step % 2, (step // 2) % 2
            hs[:] = (a0, a1)[ia]
            hc[:] = ids[ic]
            eng.set_schedule(hs)
            got = eng.eval_candidates(hc, None, net=True, stats=True, pairs=True, out=out)
            ref = refs[ia, ic]
            _same_res(got, ref, ("best_t", "best_val", "feasible", "exp_delta", "cvar"))
            n = ref["pairs"]["cand"].size
            assert got["pairs"]["cand"].size == n, (round_, step)
        pool.close()  # the next round's buffers may reuse these addresses
    eng.close()


def test_eval_moves_into_pinned_outputs(oracle_lib):
    """Engine.eval_moves(out=...): page-locked move arrays and outputs, written in place, equal the
    oracle; a wrong-typed output array is rejected."""
    from paper_2511_18296_b200.engine import PinnedPool
    from paper_2511_18296_b200.errors import ShapeMismatch
    bm, vmax, sigma = _rand_instance(9, n=(12, 10, 6), T=9, S=20, cf=0.45)
    from paper_2511_18296_b200 import synth

    rng = np.random.default_rng(5)
    assign = synth.full_greedy(bm)
    eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
    o = oracle_lib.Oracle(bm, vmax, sigma)
    pool = PinnedPool()
    try:
        M = 4000
        for kind in ("reassign", "swap"):
            a = pool.empty(M, np.int32)
            b = pool.empty(M, np.int32)
            a[:] = rng.integers(0, bm.n_blocks, M)
            b[:] = rng.integers(-1, bm.n_periods, M) if kind == "reassign" else rng.integers(0, bm.n_blocks, M)
            out = {"feasible": pool.empty(M, np.uint8), "delta": pool.empty(M, np.float64),
                   "exp_delta": pool.empty(M, np.float64), "cvar": pool.empty(M, np.float64)}
            got = eng.eval_moves(a, b, kind, None, net=True, stats=True, out=out)
            assert got["delta"] is out["delta"]
            ref = o.eval_moves(assign, np.array(a), np.array(b), kind, None, net=True, stats=True)
            _same_res(got, ref, ("feasible", "delta", "exp_delta", "cvar"))
        with pytest.raises(ShapeMismatch):
            eng.eval_moves(a, b, "swap", None, net=True, stats=True, out={"delta": np.empty(M, np.float32)})
    finally:
        eng.close()
        pool.close()


def _big_period_population(c):
    """Schedules whose periods hold far more than the 6,144 blocks of k_stage2's on-chip buffers:
    the C2 schedule folded into 4 periods (~12.5k blocks each), everything in one period (n = B),
    and a ragged mix (one period of ~25k beside small ones) -- the large-period path
    (k_stage2_big: on-chip runs + merge rounds in global scratch) next to the on-chip one."""
    a = c["assign"].astype(np.int64)
    T = c["bm"].n_periods
    fold = np.where(a >= 0, a // 4, -1)
    one = np.zeros_like(a)
    rag = a.copy()
    rag[(a >= 0) & (a < 6)] = 2
    rag[np.arange(a.size) % 97 == 0] = -1
    assert fold.max() < T
    return np.stack([fold, one, rag, a])


def test_npv_relaxed_large_periods_against_oracle(oracle_lib):
    """Stage 2 (evaluate.py:166-183) of periods mining 12k-50k blocks runs on the device and equals
    the oracle bit for bit, with and without sigma, per scenario included."""
    c = config("C2")
    bm = c["bm"]
    eng = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"]))
    o = oracle_lib.Oracle(bm, c["vmax"], c["sigma"])
    pop = _big_period_population(c)
    for use_sigma in (True, False):
        npv, ps = eng.npv_relaxed(pop, per_scenario=True, use_sigma=use_sigma)
        for k in range(pop.shape[0]):
            v, pr = o.npv_relaxed(pop[k], bm.plant_hours, bm.mode_rates[0], use_sigma=use_sigma)
            assert npv[k] == v and same(ps[k], pr), (k, use_sigma)
    eng.close()


def test_npv_moves_large_periods_equal_full_recompute():
    """pp_npv_moves re-solving periods of ~12.5k blocks (the large-period path with the variant's
    moved block) equals pp_npv_relaxed of each modified schedule."""
    c = config("C2")
    bm = c["bm"]
    eng = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"]))
    a = _big_period_population(c)[0].astype(np.int32)
    rng = np.random.default_rng(3)
    blocks = rng.integers(0, bm.n_blocks, 24).astype(np.int32)
    periods = rng.integers(-1, 4, 24).astype(np.int32)
    got = eng.npv_moves(a, blocks, periods)
    batch = np.repeat(a[None, :], blocks.size, axis=0)
    batch[np.arange(blocks.size), blocks] = periods
    assert same(got, eng.npv_relaxed(batch))
    eng.close()


def test_npv_relaxed_c4_against_oracle(oracle_lib):
    """C4 (200k blocks, 20 periods of ~10k blocks, S = 50): every period is above the on-chip size."""
    c = config("C4")
    bm = c["bm"]
    eng = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"]))
    o = oracle_lib.Oracle(bm, c["vmax"], c["sigma"])
    npv, ps = eng.npv_relaxed(c["assign"][None, :], per_scenario=True)
    v, pr = o.npv_relaxed(c["assign"], bm.plant_hours, bm.mode_rates[0])
    assert npv[0] == v and same(ps[0], pr)
    eng.close()


@pytest.mark.parametrize("name", ["m27", "m32", "m512", "mC1"])
def test_explicit_moves_match_reference_polish_options(name):
    """pp_eval_moves' feasibility against the reference's own move generation: the reassign /
    unmine options and the pair swaps polish_schedule evaluates for a fixed schedule
    (hybrid.py:348-403, recorded by tests/golden/make_golden.py move_cases) are exactly the
    moves the engine reports feasible."""
    st = load("moves")
    p = f"{name}_"
    bm = bm_from(st, p)
    eng = Engine.from_tables(bm, tables_from(st, p))
    B, T = bm.n_blocks, bm.n_periods
    for k in range(3):
        q = f"{p}{k}_"
        eng.set_schedule(st[q + "assign"])
        bb = np.repeat(np.arange(B), T + 1).astype(np.int32)
        tt = np.tile(np.arange(-1, T), B).astype(np.int32)
        r = eng.eval_moves(bb, tt, "reassign", net=True)
        f = r["feasible"] == 1
        assert set(zip(bb[f].tolist(), tt[f].tolist())) == set(map(tuple, st[q + "reassign"].tolist())), k
        assert np.all(np.isfinite(r["delta"][f])) and np.all(r["delta"][~f] == -np.inf)
        if B <= 32:
            i, j = np.triu_indices(B, 1)
            r = eng.eval_moves(i.astype(np.int32), j.astype(np.int32), "swap", net=True)
            f = r["feasible"] == 1
            assert set(zip(i[f].tolist(), j[f].tolist())) == set(map(tuple, st[q + "swap"].tolist())), k
    eng.close()


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_scenario_stats_cvar_k_gt_1_match_reference(name):
    """Expected delta and CVaR10 over k > 1 scenarios (C2: S = 20, k = 2; C3: S = 200, k = 20, the
    warp-per-move selection path) and the per-scenario deltas, against the reference kernel run
    once per scenario plus saa.risk_metrics (tests/golden/make_golden.py stats_cases)."""
    from tests._fixtures import digest, instance_digest

    st = load("stats")
    c = config(name)
    assert instance_digest(c["bm"]) == st[f"{name}_digest_instance"].item().decode()
    assert digest(c["vmax"]) == st[f"{name}_digest_vmax"].item().decode()
    assert digest(c["assign"].astype(np.int32)) == st[f"{name}_digest_assign"].item().decode()
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], st[f"{name}_sigma"]), c["assign"])
    sub = st[f"{name}_sub"]
    got = eng.eval_candidates(sub, None, net=True, stats=True, scen=True)
    assert same(got["exp_delta"], st[f"{name}_sub_exp"])
    assert same(got["cvar"], st[f"{name}_sub_cvar"])
    assert same(got["scen_delta"], st[f"{name}_sub_scen_delta"])
    pr = eng.eval_candidates(sub, None, net=True, pairs=True)["pairs"]
    ex = st[f"{name}_sub_exp"]
    assert pr["cand"].size == int(np.isfinite(ex).sum())
    assert same(pr["exp"], ex[pr["cand"], pr["period"]]) and same(pr["cvar"], st[f"{name}_sub_cvar"][pr["cand"], pr["period"]])
    eng.close()


def _realism_ref(cand, best_t, spatial):
    """lns_repair's realism fallback (hybrid.py:256-263): feasible moves sorted by
    (-spatial[b], b), first one."""
    feas = [(int(b), int(t)) for b, t in zip(cand, best_t) if t >= 0]
    if not feas:
        return None
    b, t = sorted(feas, key=lambda m: (-spatial[m[0]], m[0]))[0]
    return (b, t, float(spatial[b]))


def test_realism_key_on_device(oracle_lib):
    """The second selection key (k_realism) equals the reference's sort of the feasible moves, with
    duplicated candidates, ties in geological consistency (a constant-feature instance), host and
    device buffers, both evaluation kernels (T <= 32 and T = 40)."""
    c = config("C1")
    rng = np.random.default_rng(9)
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["greedy"])
    sp = eng.spatial()
    for k in range(6):
        cand = rng.integers(0, c["bm"].n_blocks, size=int(rng.integers(1, 3000))).astype(np.int32)
        cand = np.concatenate([cand, cand[: cand.size // 3]])
        r = eng.eval_candidates(cand, None, net=bool(k % 2), realism=True)
        assert r["realism"] == _realism_ref(cand, r["best_t"], sp), k
    eng.close()
    # ties: every block has the same features, hence the same consistency -> lowest block wins
    bm = c["bm"]
    flat = BlockModel(n_blocks=bm.n_blocks, n_periods=bm.n_periods, edges_i=bm.edges_i, edges_j=bm.edges_j,
                      mass=bm.mass, cost=bm.cost, capacity=bm.capacity, discount_rate=bm.discount_rate,
                      coords=bm.coords, alteration=np.full(bm.n_blocks, 0.5), structural=np.full(bm.n_blocks, 0.5),
                      dist_intrusion=np.ones(bm.n_blocks), base_grade=np.zeros(bm.n_blocks))
    eng = Engine.from_tables(flat, ScenarioTables(c["vmax"], c["sigma"]), c["greedy"])
    sp = eng.spatial()
    assert np.all(sp == sp[0])
    cand = rng.permutation(bm.n_blocks)[:1500].astype(np.int32)
    r = eng.eval_candidates(cand, None, realism=True)
    assert r["realism"] == _realism_ref(cand, r["best_t"], sp)
    eng.close()
    # T = 40: the general evaluation kernel
    from paper_2511_18296_b200 import synth
    from paper_2511_18296_b200.model import scenario_values

    bm40 = synth.generate_block_model(2000, (20, 10, 10), 40, 1, seed=4, n_rock_types=1)
    g = synth.sample_lognormal(bm40, 7, 0.3, seed=5)
    eng = Engine.from_tables(bm40, ScenarioTables(scenario_values(bm40, g), synth.uncertainty_sigma(bm40, g)),
                             synth.full_greedy(bm40))
    sp = eng.spatial()
    cand = rng.integers(0, 2000, size=900).astype(np.int32)
    r = eng.eval_candidates(cand, None, realism=True)
    assert r["realism"] == _realism_ref(cand, r["best_t"], sp)
    eng.close()


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_npv_moves_incremental_base_sequence(name):
    """pp_npv_moves keeps the base schedule's per-(scenario, period) greedy structure and, when the
    base changes by a few blocks (as in polish_schedule), re-solves only the changed periods: a
    sequence of drifting bases with reassign / unmine / mine variants -- including empty periods,
    blocks of non-positive density and large batches -- equals pp_npv_relaxed of every variant."""
    c = config(name)
    bm = c["bm"]
    vmax = c["vmax"].copy()
    vmax[:, ::13] = -np.abs(vmax[:, ::13])  # non-positive densities in every scenario
    eng = Engine.from_tables(bm, ScenarioTables(vmax, c["sigma"]))
    rng = np.random.default_rng(21)
    a = c["greedy"].copy().astype(np.int32)
    a[a == 3] = -1  # an empty period
    B, T = bm.n_blocks, bm.n_periods
    for step in range(8):
        m = int(rng.choice([3, 40, 700]))
        blocks = rng.integers(0, B, m).astype(np.int32)
        periods = rng.integers(-1, T, m).astype(np.int32)
        got = eng.npv_moves(a, blocks, periods)
        batch = np.repeat(a[None, :], m, axis=0)
        batch[np.arange(m), blocks] = periods
        ref = np.concatenate([eng.npv_relaxed(batch[i:i + 256]) for i in range(0, m, 256)])
        assert same(got, ref), (name, step)
        # drift the base like accepted polish moves: one to three blocks per step, sometimes many
        k = 1 + step % 3 if step != 5 else B // 3
        idx = rng.integers(0, B, k)
        a[idx] = rng.integers(-1, T, k)
    eng.close()


@pytest.mark.parametrize("name,modes", [("C1", 1), ("C1", 3), ("C2", 1)])
def test_device_ingestion_from_grades(name, modes):
    """pp_set_scenarios_grades builds the value table on the device from grades[S][B]
    (scenario_mode_values, evaluate.py:116-124, max over modes) bit-identical to the host table, and
    an engine fed grades evaluates exactly like one fed the host table."""
    import dataclasses

    from paper_2511_18296_b200.model import scenario_values

    c = config(name)
    bm = c["bm"]
    if modes > 1:
        bm = dataclasses.replace(bm, n_modes=modes, recovery_by_mode=(0.85, 0.9, 0.7),
                                 processing_cost_by_mode=(1.0, 1.6, 0.4))
    host = scenario_values(bm, c["grades"])
    e_dev = Engine.from_tables(bm, ScenarioTables(None, c["sigma"], grades=c["grades"]), c["assign"])
    assert same(e_dev.scenario_table(), host)
    e_host = Engine.from_tables(bm, ScenarioTables(host, c["sigma"]), c["assign"])
    for kw in (dict(net=True, stats=True), dict(net=False, trace=True)):
        a = e_dev.eval_candidates(c["cand"], None, **kw)
        b = e_host.eval_candidates(c["cand"], None, **kw)
        assert a["best"] == b["best"]
        for k in ("best_t", "best_val", "exp_delta", "cvar", "trace_val"):
            if k in a:
                assert same(a[k], b[k]), k
    e_dev.close()
    e_host.close()


@pytest.mark.parametrize("T,S", [(3, 1), (9, 7), (15, 20), (6, 64), (12, 129), (5, 256), (7, 300)])
def test_explicit_moves_shapes_against_oracle(oracle_lib, T, S):
    """k_moves_warp (a warp per move, 128-bit scenario-row loads; S <= 256) and its fallback
    k_eval_moves (S = 300) against the oracle: reassign / unmine and swaps, both flags, s = None and
    s = k, statistics and per-scenario deltas; the selected move (lowest index on ties)."""
    bm, vmax, sigma = _rand_instance(11 + T, n=(10, 8, 5), T=T, S=S, cf=0.5)
    from paper_2511_18296_b200 import synth

    rng = np.random.default_rng(T * 100 + S)
    assign = synth.full_greedy(bm)
    eng = Engine.from_tables(bm, ScenarioTables(vmax, sigma), assign)
    o = oracle_lib.Oracle(bm, vmax, sigma)
    M = 3000
    b = rng.integers(0, bm.n_blocks, M).astype(np.int32)
    t = rng.integers(-1, bm.n_periods, M).astype(np.int32)
    keys = ("feasible", "delta", "exp_delta", "cvar", "scen_delta")
    for net, s in ((False, None), (True, S - 1)):
        got = eng.eval_moves(b, t, "reassign", s, net=net, stats=True, scen=True)
        ref = o.eval_moves(assign, b, t, "reassign", s, net=net, stats=True, scen=True)
        _same_res(got, ref, keys)
        assert got["best"] == ref["best"]
    b2 = rng.integers(0, bm.n_blocks, M).astype(np.int32)
    got = eng.eval_moves(b, b2, "swap", None, net=True, stats=True, scen=True)
    ref = o.eval_moves(assign, b, b2, "swap", None, net=True, stats=True, scen=True)
    _same_res(got, ref, keys)
    assert got["best"] == ref["best"]
    eng.close()
