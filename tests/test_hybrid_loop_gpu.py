"""C5 end to end: the reference's own hybrid GA+LNS+SA loop (hybrid.py:1015-1026), unmodified,
with and without the device drop-ins installed (install.py) must produce the same best schedule
and the same per-iteration trace, bit for bit.

The reference is imported from its pip install under baseline/_ref (git-ignored, shipped to the
GPU box with the snapshot); the test skips when that install is absent.
"""

import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _import_ref():
    if not os.path.isdir(os.path.join(REF, "pitplan")):
        pytest.skip("baseline/_ref (pip install of the reference) absent")
    if REF not in sys.path:
        sys.path.append(REF)
    import pitplan.hybrid as H
    from pitplan.blockmodel import generate_synthetic
    from pitplan.scenarios import sample_lognormal
    from pitplan.uncertainty import uncertainty_factors

    return H, generate_synthetic, sample_lognormal, uncertainty_factors


@pytest.mark.parametrize("seed", [0, 1])
def test_hybrid_optimize_identical_with_device_dropins(seed):
    H, generate_synthetic, sample_lognormal, uncertainty_factors = _import_ref()
    from paper_2511_18296_b200 import evaluate as ev
    from paper_2511_18296_b200.install import install, uninstall

    inst = generate_synthetic(180, (6, 6, 5), 5, 1, seed=10 + seed, n_rock_types=1)
    scen = sample_lognormal(inst, 4, 0.3, seed=20 + seed)
    sigma = uncertainty_factors(inst, scen.grades)
    cfg = H.HybridConfig(population=6, t_max=2, g_max=1, neighborhoods=2, init_multistarts=2,
                         repair_iters=5, seed=seed)

    best_ref, trace_ref = H.hybrid_optimize(inst, scen, sigma, cfg)
    patched = install()
    try:
        assert "pitplan.hybrid.evaluate_candidates_parallel" in patched
        best_dev, trace_dev = H.hybrid_optimize(inst, scen, sigma, cfg)
    finally:
        uninstall()
        ev.clear_cache()
    assert list(best_dev.assignment) == list(best_ref.assignment)
    assert [r.as_list() for r in trace_dev] == [r.as_list() for r in trace_ref]
