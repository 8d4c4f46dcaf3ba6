"""The VAE scenario decode (§8(f) row 4, ingestion; vae.py:284-321) against the reference's own
vae_generate on models the reference trained (tests/golden/vae.npz, make_golden.py vae).  The
reference decodes through numpy matmul (BLAS), whose summation order is not reproducible across
libraries, so the comparisons are to rounding: relative 1e-12 on every grade."""

import numpy as np
import pytest

from tests._fixtures import bm_from, load

RTOL = 1e-12


def _decoder(st, p):
    from paper_2511_18296_b200.model import VaeDecoder

    L = st[p + "widths"].size - 1
    return VaeDecoder([(st[p + f"W{k}"], st[p + f"b{k}"]) for k in range(L)], st[p + "norm_mean"], st[p + "norm_std"])


def _close(a, b):
    return np.all(np.abs(a - b) <= RTOL * np.maximum(np.abs(b), 1.0))


@pytest.mark.parametrize("p", ["v1_", "v2_"])
def test_host_restatement_matches_reference_decode(p):
    """model.VaeDecoder.decode_host (the numpy restatement) reproduces vae_generate's grades from
    the stored layers and the stored prior samples z (the substream of vae.py:288-290)."""
    st = load("vae")
    dec = _decoder(st, p)
    assert dec.widths == st[p + "widths"].tolist()
    assert _close(dec.decode_host(st[p + "z"]), st[p + "grades"])


@pytest.mark.gpu
@pytest.mark.parametrize("p", ["v1_", "v2_"])
def test_device_decode_matches_reference(p):
    from paper_2511_18296_b200.engine import Engine

    st = load("vae")
    bm = bm_from(st, p)
    eng = Engine.from_tables(bm, None)
    eng.set_vae_decoder(_decoder(st, p))
    g = eng.vae_decode(st[p + "z"])
    assert g.shape == st[p + "grades"].shape
    assert _close(g, st[p + "grades"]), float(np.max(np.abs(g - st[p + "grades"])))
    assert np.all(g >= 0.0)
    eng.close()


@pytest.mark.gpu
def test_vae_scenarios_bound_on_device_equal_the_grades_path():
    """pp_set_scenarios_vae (decode + value table on the device) gives exactly the value table of
    the same grades ingested through pp_set_scenarios_grades, and evaluations agree bit for bit."""
    from paper_2511_18296_b200.engine import Engine
    from paper_2511_18296_b200.model import ScenarioTables

    st = load("vae")
    p = "v2_"
    bm = bm_from(st, p)
    bm.base_grade = st[p + "norm_mean"].copy()
    rng = np.random.default_rng(2)
    a = np.where(rng.random(bm.n_blocks) < 0.7, rng.integers(0, bm.n_periods, bm.n_blocks), -1).astype(np.int32)
    e1 = Engine.from_tables(bm, None)
    e1.set_vae_decoder(_decoder(st, p))
    z = st[p + "z"]
    g = e1.vae_decode(z)
    e1.set_scenarios_vae(z)
    e1.set_schedule(a)
    e2 = Engine.from_tables(bm, ScenarioTables(None, None, grades=g), a)
    assert np.array_equal(e1.scenario_table(), e2.scenario_table())
    cand = rng.integers(0, bm.n_blocks, 300).astype(np.int32)
    r1 = e1.eval_candidates(cand, None, net=True, stats=True, use_sigma=False)
    r2 = e2.eval_candidates(cand, None, net=True, stats=True, use_sigma=False)
    for k in ("best_t", "best_val", "exp_delta", "cvar"):
        assert np.array_equal(r1[k], r2[k]), k
    assert r1["best"] == r2["best"]
    e1.close()
    e2.close()


@pytest.mark.gpu
def test_vae_decode_large_random_decoder_against_numpy():
    """A 50k-block decoder of the reference architecture (random weights): the device GEMMs against
    the numpy restatement over 64 scenarios (tiles at every edge: 64-wide outputs, 16-deep k)."""
    from paper_2511_18296_b200 import synth
    from paper_2511_18296_b200.engine import Engine
    from paper_2511_18296_b200.model import VaeDecoder

    c = synth.build_config("C2")
    bm = c["bm"]
    base = np.asarray(c["grades"]).mean(axis=0)
    dec = VaeDecoder.random_init(bm.n_blocks, base, 0.3 * base + 1e-3, seed=4)
    z = np.random.default_rng(5).standard_normal((67, dec.latent_dim))
    eng = Engine.from_tables(bm, None)
    eng.set_vae_decoder(dec)
    g = eng.vae_decode(z)
    ref = dec.decode_host(z)
    assert _close(g, ref), float(np.max(np.abs(g - ref) / np.maximum(np.abs(ref), 1.0)))
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_device_uncertainty_sigma_matches_reference(cfg):
    """uncertainty_factors' sigma[S][T] on the device (pp_uncertainty_sigma) against the
    reference's (C1: the golden fixture's, computed by pitplan) and the host restatement (C2), to
    rounding: the reference's Moran denominator is a BLAS dot product."""
    from paper_2511_18296_b200 import synth
    from paper_2511_18296_b200.engine import Engine
    from tests._fixtures import config

    if cfg == "C1":
        st = load("c1")
        c = config("C1")
        bm, grades, ref = c["bm"], st["C1_grades"], c["sigma"]
    else:
        c = synth.build_config("C2")
        bm, grades = c["bm"], c["grades"]
        ref = synth.uncertainty_sigma(bm, grades)
    eng = Engine.from_tables(bm, None)
    sig, moran, local = eng.uncertainty_sigma(grades)
    assert sig.shape == ref.shape
    assert _close(sig, ref), float(np.max(np.abs(sig - ref) / np.maximum(np.abs(ref), 1.0)))
    # a zero-variance field: Moran's I is undefined, f_spatial = 1 + local CV
    flat = np.full((1, bm.n_blocks), 1.5)
    s1, m1, l1 = eng.uncertainty_sigma(flat)
    assert np.isnan(m1[0]) and l1[0] == 0.0
    phi = np.exp(-0.1 * np.arange(bm.n_periods))
    assert np.array_equal(s1[0], np.clip((1.0 * phi) * s1[0, 0], 1e-6, 2.0))  # s1[0, 0] = psi (phi[0] = 1)
    eng.close()
