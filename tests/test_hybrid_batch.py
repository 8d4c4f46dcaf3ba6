"""Host-side GA helpers (CPU): the native _mutate equals the reference's own loop -- the same
child and the same Generator state afterwards (so every later draw matches) -- on random
schedules, neighbourhoods and rates; the lazy members' batch bookkeeping."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "pitplan")):
        pytest.skip("baseline/_ref (pip install of the reference) absent")
    if REF not in sys.path:
        sys.path.append(REF)
    import pitplan.blockmodel as BM
    import pitplan.hybrid as H
    import pitplan.rng as R

    return BM, H, R


class _Search:  # what _mutate reads from a HybridSearch
    def __init__(self, inst):
        self.instance = inst


@pytest.mark.parametrize("seed", range(6))
def test_native_mutate_equals_reference(ref, seed):
    from paper_2511_18296_b200 import hybrid_batch as hb

    BM, H, R = ref
    inst = BM.generate_synthetic(512, (8, 8, 8), 6, 1, seed=60 + seed, n_rock_types=1)
    search = _Search(inst)
    rs = np.random.default_rng(seed)
    for trial in range(8):
        a0 = rs.integers(-1, 6, size=512).astype(np.int64)
        blocks = rs.permutation(512)[: int(rs.integers(1, 512))]
        rate = float(rs.choice([0.05, 0.2, 0.5, 1.0]))
        g_ref = R.substream(seed, "iter", trial)
        g_dev = R.substream(seed, "iter", trial)
        if trial % 2:  # leave a buffered uint32 half pending in both generators
            g_ref.integers(0, 7)
            g_dev.integers(0, 7)
        a_ref, a_dev = a0.copy(), a0.copy()
        H.HybridSearch._mutate(search, a_ref, g_ref, blocks, rate)
        hb.mutate(search, a_dev, g_dev, blocks, rate)
        assert np.array_equal(a_ref, a_dev), (seed, trial)
        assert g_ref.bit_generator.state == g_dev.bit_generator.state, (seed, trial)
        assert np.array_equal(g_ref.integers(0, 10, 5), g_dev.integers(0, 10, 5))
        assert g_ref.random() == g_dev.random()
