"""The drop-ins against the reference itself (its pip install under baseline/_ref, shipped to the
GPU box with the snapshot) as the checker, and proof that the product path executes no reference
code: every check reads the path counters (evaluate.path_counters).

The reference runs here only as the oracle of each test; the functions under test are this
package's drop-ins.  Skips when baseline/_ref is absent.
"""

import filecmp
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "pitplan")):
        pytest.skip("baseline/_ref (pip install of the reference) absent")
    if REF not in sys.path:
        sys.path.append(REF)
    import pitplan.blockmodel as BM
    import pitplan.colgen as CG
    import pitplan.evaluate as E
    import pitplan.hybrid as H
    import pitplan.scenarios as SC
    import pitplan.uncertainty as U

    return dict(BM=BM, CG=CG, E=E, H=H, SC=SC, U=U)


@pytest.fixture(autouse=True)
def _fresh():
    from paper_2511_18296_b200 import evaluate as ev

    ev.reset_path_counters()
    yield
    ev.clear_cache()


def _case(ref, n=180, dims=(6, 6, 5), T=5, S=4, seed=10, modes=1):
    inst = ref["BM"].generate_synthetic(n, dims, T, modes, seed=seed, n_rock_types=1)
    scen = ref["SC"].sample_lognormal(inst, S, 0.3, seed=seed + 1)
    sigma = ref["U"].uncertainty_factors(inst, scen.grades)
    return inst, scen, sigma


def _no_reference(min_device=1):
    from paper_2511_18296_b200 import evaluate as ev

    c = ev.path_counters()
    assert c["reference"] == {}, c
    assert sum(c["device"].values()) >= min_device, c
    return c


def test_trace_csv_bytes_equal_reference(ref, tmp_path):
    """The trace CSV (evaluate.py:423-428) is byte-identical to the reference's own file,
    including duplicated candidates, infeasible rows (-inf) and both s=None and s=k."""
    from paper_2511_18296_b200 import evaluate as ev

    inst, scen, sigma = _case(ref)
    sched = ref["H"].greedy_initialize(inst, scen, sigma)
    cand = [5, 17, 5, 120, 179, 0, 63, 64]
    for s in (None, 2):
        for net in (False, True):
            a, b = tmp_path / f"ref_{s}_{net}.csv", tmp_path / f"dev_{s}_{net}.csv"
            m_ref, best_ref = ref["E"].evaluate_candidates_parallel(inst, sched, cand, scen, s, sigma,
                                                                    net_mining_cost=net, trace_path=a)
            m_dev, best_dev = ev.evaluate_candidates_parallel(inst, sched, cand, scen, s, sigma,
                                                              net_mining_cost=net, trace_path=b)
            assert filecmp.cmp(a, b, shallow=False), (s, net)
            assert [m.__dict__ for m in m_dev] == [m.__dict__ for m in m_ref]
            assert (best_dev is None and best_ref is None) or best_dev.__dict__ == best_ref.__dict__
    _no_reference()


def test_literal_value_with_sigma_and_no_scenarios(ref):
    """literal_kernel_value=True, scenarios=None, sigma given: the sigma row still applies
    (evaluate.py:348-353)."""
    from paper_2511_18296_b200 import evaluate as ev

    inst, scen, sigma = _case(ref, seed=12)
    sched = ref["H"].greedy_initialize(inst, scen, sigma)
    cand = list(range(0, 180, 7))
    for s in (None, 1, -1):
        r = ref["E"].evaluate_candidates_parallel(inst, sched, cand, None, s, sigma, literal_kernel_value=True)
        d = ev.evaluate_candidates_parallel(inst, sched, cand, None, s, sigma, literal_kernel_value=True)
        assert [m.__dict__ for m in d[0]] == [m.__dict__ for m in r[0]], s
        assert d[1].__dict__ == r[1].__dict__
    _no_reference()


def test_negative_scenario_index_matches_reference(ref):
    from paper_2511_18296_b200 import evaluate as ev

    inst, scen, sigma = _case(ref, seed=14)
    sched = ref["H"].greedy_initialize(inst, scen, sigma)
    cand = list(range(0, 180, 5))
    for s in (-1, -4):
        r = ref["E"].evaluate_candidates_parallel(inst, sched, cand, scen, s, sigma)
        d = ev.evaluate_candidates_parallel(inst, sched, cand, scen, s, sigma)
        assert [m.__dict__ for m in d[0]] == [m.__dict__ for m in r[0]], s
    with pytest.raises(ev.InvalidArgs):
        ev.evaluate_candidates_parallel(inst, sched, [-1], scen, None, sigma)


@pytest.mark.parametrize("noise,slack", [(0.0, 1.0), (0.05, 1.0), (0.0, 1.4), (0.1, 1.25)])
def test_price_column_matches_reference(ref, noise, slack):
    """colgen.price_column (colgen.py:207-293): ENPV table, noise stream, greedy, slack trim, value
    and reduced cost -- all from the device path, equal to the reference's column."""
    from paper_2511_18296_b200 import evaluate as ev

    inst, scen, sigma = _case(ref, n=500, dims=(10, 10, 5), T=6, S=5, seed=21)
    rng = np.random.default_rng(4)
    B, T = inst.n_blocks, inst.n_periods
    duals = ref["CG"].DualPrices(block=rng.normal(0, 50, B), capacity=np.abs(rng.normal(0, 0.01, T)),
                                 convexity=np.abs(rng.normal(0, 10, 2)))
    for with_eval in (False, True):
        evr = ref["E"].ScheduleEvaluator(inst, scen, sigma) if with_eval else None
        evd = ev.ScheduleEvaluator(inst, scen, sigma) if with_eval else None
        cr, rcr = ref["CG"].price_column(inst, duals, scen, sigma, 1, (7, "price", 3), evr, 5000, slack, noise)
        cd, rcd = ev.price_column(inst, duals, scen, sigma, 1, (7, "price", 3), evd, 5000, slack, noise)
        assert np.array_equal(cd.assignment, cr.assignment)
        assert np.array_equal(cd.mass_per_period, cr.mass_per_period)
        assert cd.value == cr.value and rcd == rcr
    _no_reference(min_device=2)


def test_schedule_evaluator_attributes_and_values(ref):
    """The attributes callers read from an evaluator (hybrid.py:673-678, saa.py:60-65) equal the
    reference's; npv_relaxed / per_scenario_npv / objective are the reference's numbers."""
    from paper_2511_18296_b200 import evaluate as ev

    inst, scen, sigma = _case(ref, seed=30)
    r = ref["E"].ScheduleEvaluator(inst, scen, sigma)
    d = ev.ScheduleEvaluator(inst, scen, sigma)
    assert np.array_equal(d.values, r.values)
    assert np.array_equal(d.masses, r.masses) and np.array_equal(d.costs, r.costs)
    assert np.array_equal(d.discount, r.discount)
    sched = ref["H"].greedy_initialize(inst, scen, sigma)
    assert d.npv_relaxed(sched) == r.npv_relaxed(sched)
    assert np.array_equal(d.per_scenario_npv(sched), r.per_scenario_npv(sched))
    assert d.objective(sched) == r.objective(sched)
    assert len(d._stage2_cache) > 0
    _no_reference()


def test_lp_instance_goes_to_reference_explicitly_without_recursion(ref):
    """A multi-mode instance (stage-2 LP, out of scope): after install() the evaluator factory
    returns the reference's class and polish_schedule runs the reference's own function -- the one
    captured before install() rebound the name, so it cannot call itself --
    and both are counted."""
    from paper_2511_18296_b200 import evaluate as ev
    from paper_2511_18296_b200.install import install, uninstall

    inst, scen, sigma = _case(ref, n=27, dims=(3, 3, 3), T=3, S=2, seed=5, modes=2)
    H = ref["H"]
    sched = H.greedy_initialize(inst, scen, sigma)
    want = H.polish_schedule(inst, ref["E"].ScheduleEvaluator(inst, scen, sigma), sched, 2)
    install()
    try:
        e = H.ScheduleEvaluator(inst, scen, sigma)
        assert type(e).__module__ == "pitplan.evaluate"
        got = H.polish_schedule(inst, e, sched, 2)
    finally:
        uninstall()
    assert np.array_equal(got.assignment, want.assignment)
    c = ev.path_counters()["reference"]
    assert c == {"ScheduleEvaluator": 1, "polish_schedule": 1}, c


def test_hybrid_loop_runs_no_reference_code(ref):
    """The reference's hybrid GA+LNS+SA loop with the drop-ins installed: same result as without,
    and zero calls into reference code on the way (single-mode instance)."""
    from paper_2511_18296_b200.install import install, uninstall

    H = ref["H"]
    inst, scen, sigma = _case(ref, seed=40)
    cfg = H.HybridConfig(population=6, t_max=2, g_max=1, neighborhoods=2, init_multistarts=2,
                         repair_iters=5, seed=3)
    best_ref, trace_ref = H.hybrid_optimize(inst, scen, sigma, cfg)
    from paper_2511_18296_b200 import evaluate as ev

    ev.reset_path_counters()
    install()
    try:
        best_dev, trace_dev = H.hybrid_optimize(inst, scen, sigma, cfg)
    finally:
        uninstall()
    assert list(best_dev.assignment) == list(best_ref.assignment)
    assert [r.as_list() for r in trace_dev] == [r.as_list() for r in trace_ref]
    c = _no_reference(min_device=10)
    assert c["device"].get("pp_npv_relaxed", 0) + c["device"].get("pp_npv_moves", 0) > 0


def test_dw_loop_runs_no_reference_code(ref):
    """Column generation (colgen.run_dw) with the drop-ins installed: pricing, evaluation and the
    integerisation repair on the device, same result as the reference, zero reference calls."""
    from paper_2511_18296_b200 import evaluate as ev
    from paper_2511_18296_b200.install import install, uninstall

    CG = ref["CG"]
    inst, scen, sigma = _case(ref, n=180, dims=(6, 6, 5), T=5, S=3, seed=50)
    cfg = CG.DwConfig(max_iterations=3, initial_columns=4, max_columns=20, n_scenarios=3,
                      scenarios_per_iter=2, seed=1)
    want = CG.run_dw(inst, cfg, scenarios=scen, sigma=sigma)
    ev.reset_path_counters()
    install()
    try:
        got = CG.run_dw(inst, cfg, scenarios=scen, sigma=sigma)
    finally:
        uninstall()
    assert np.array_equal(got[0].assignment, want[0].assignment)
    assert [r.__dict__ for r in got[1]] == [r.__dict__ for r in want[1]]
    _no_reference(min_device=3)
