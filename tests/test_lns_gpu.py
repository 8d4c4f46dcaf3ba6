"""The device-resident lns_repair insertion loop (pp_lns_insert: one CUDA graph with a
conditional WHILE node per repair) against the host-driven loop of the same drop-in, round by
round equal -- the host loop is itself pinned to the reference's runs (test_gpu_parity.py
test_lns_repair_dropin_*) -- over destroy fractions, realism thresholds (never / default / almost
always the fallback), candidate widths 1..64, only_positive, max_iters limits, sigma on/off and
net mining cost, at C1 (4k blocks) and C2 (50k blocks, pools of thousands)."""

import numpy as np
import pytest

from tests._fixtures import config, load

pytestmark = pytest.mark.gpu


def _both(monkeypatch, bm, start, tables, sigma, **kw):
    from paper_2511_18296_b200 import evaluate as dropin
    from paper_2511_18296_b200.model import Schedule

    un = kw.pop("unassigned", [])
    before = dict(dropin.path_counters()["device"])
    g = dropin.lns_repair(bm, Schedule(start.copy()), un, tables, sigma, **kw)
    used = dropin.path_counters()["device"].get("pp_lns_insert", 0) - before.get("pp_lns_insert", 0)
    # the graph runs exactly when the destroy step leaves a pool
    _, added = dropin._entry(bm).engine.lns_destroy(np.asarray(start)[None, :], np.asarray(tables.grades).mean(axis=0),
                                                    kw.get("destroy_fraction", 0.0))
    assert used == int((bool(added.any()) or len(un) > 0) and kw.get("max_iters", 100) > 0)
    monkeypatch.setattr(dropin, "_LNS_GRAPH_WMAX", 0)  # the host-driven loop
    h = dropin.lns_repair(bm, Schedule(start.copy()), un, tables, sigma, **kw)
    monkeypatch.undo()
    return g.assignment, h.assignment, used


VARIANTS = [
    dict(max_iters=40, destroy_fraction=0.1),
    dict(max_iters=200, destroy_fraction=0.3, net_mining_cost=True),
    dict(max_iters=200, destroy_fraction=0.3, realism_threshold=0.0),
    dict(max_iters=200, destroy_fraction=0.3, realism_threshold=0.97, candidate_width=3),
    dict(max_iters=7, destroy_fraction=0.5, candidate_width=64),
    dict(max_iters=300, destroy_fraction=0.2, only_positive=True),
    dict(max_iters=300, destroy_fraction=0.2, candidate_width=1),
]


@pytest.mark.parametrize("v", range(len(VARIANTS)))
@pytest.mark.parametrize("use_sigma", [True, False])
def test_graph_loop_equals_host_loop_c1(monkeypatch, v, use_sigma):
    from paper_2511_18296_b200 import evaluate as dropin
    from paper_2511_18296_b200.model import ScenarioTables

    st = load("c1")
    c = config("C1")
    tables = ScenarioTables(c["vmax"], c["sigma"], grades=st["C1_grades"])
    ran = 0
    for k in range(st["C1_destroy_in"].shape[0]):
        g, h, used = _both(monkeypatch, c["bm"], st["C1_destroy_in"][k], tables, True if use_sigma else None,
                           **dict(VARIANTS[v]))
        ran += used
        assert np.array_equal(g, h), (v, k, int(np.sum(g != h)))
    assert ran >= 1  # the graph path ran on at least one of the schedules
    dropin.clear_cache()


def test_graph_loop_equals_host_loop_c2(monkeypatch):
    """50k blocks: a spatial chunk of ~8% of the mined blocks unmined (the _lns_diversify shape)
    plus the fixpoint, then a few hundred insertion rounds."""
    from paper_2511_18296_b200 import evaluate as dropin, synth
    from paper_2511_18296_b200.model import ScenarioTables, scenario_values

    c = synth.build_config("C2")
    bm = c["bm"]
    tables = ScenarioTables(scenario_values(bm, c["grades"]), c["sigma"], grades=c["grades"])
    a = np.asarray(c["assign"], dtype=np.int64).copy()
    mined = np.nonzero(a >= 0)[0]
    anchor = mined[len(mined) // 3]
    d = ((bm.coords[mined] - bm.coords[anchor]) ** 2).sum(axis=1)
    chunk = mined[np.argsort(d, kind="stable")[: len(mined) // 12]]
    a[chunk] = -1
    for kw in (dict(max_iters=300), dict(max_iters=300, realism_threshold=0.9, destroy_fraction=0.05)):
        g, h, used = _both(monkeypatch, bm, a, tables, True, unassigned=chunk.tolist(), **kw)
        assert used == 1
        assert np.array_equal(g, h), (kw, int(np.sum(g != h)))
    dropin.clear_cache()


def test_lns_insert_edges():
    """pp_lns_insert directly: empty pool and max_iters = 0 change nothing; a stall (no candidate
    with a feasible period) is reported; the width limit and a rook list of 8 are refused."""
    from paper_2511_18296_b200.engine import Engine
    from paper_2511_18296_b200.errors import ShapeMismatch
    from paper_2511_18296_b200.evaluate import _rook_csr
    from paper_2511_18296_b200.model import ScenarioTables, rook_neighbor_map, rook_padded

    st = load("c1")
    c = config("C1")
    bm = c["bm"]
    eng = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"], grades=st["C1_grades"]), c["greedy"])
    eng.set_rook(*_rook_csr(rook_padded(rook_neighbor_map(bm), bm.n_blocks)))
    mg = st["C1_grades"].mean(axis=0)
    a0 = np.asarray(c["greedy"], dtype=np.int32)
    none = np.zeros(bm.n_blocks, np.uint8)
    a, pl, it, stl = eng.lns_insert(a0, none, mg, max_iters=10)
    assert np.array_equal(a, a0) and it == 0 and not stl and not pl.any()
    pool = np.zeros(bm.n_blocks, np.uint8)
    pool[np.nonzero(a0 >= 0)[0][-5:]] = 1
    a, pl, it, stl = eng.lns_insert(a0, pool, mg, max_iters=0)
    assert np.array_equal(a, a0) and it == 0 and np.array_equal(pl, pool)
    # a stall: no period has capacity left for the pool block
    full = a0.copy()
    blk = int(np.nonzero(a0 >= 0)[0][-1])
    full[blk] = -1
    cap_pool = np.zeros(bm.n_blocks, np.uint8)
    cap_pool[blk] = 1
    saved = bm.capacity.copy()
    try:
        bm.capacity[:] = 1e-300  # (> 0: a valid instance) below every block mass
        eng2 = Engine.from_tables(bm, ScenarioTables(c["vmax"], c["sigma"], grades=st["C1_grades"]), full)
        eng2.set_rook(*_rook_csr(rook_padded(rook_neighbor_map(bm), bm.n_blocks)))
        a, pl, it, stl = eng2.lns_insert(full, cap_pool, mg, max_iters=5)
        assert it == 0 and stl and pl[blk] == 1 and np.array_equal(a, full)
        eng2.close()
    finally:
        bm.capacity[:] = saved
    with pytest.raises(ShapeMismatch):
        eng.lns_insert(a0, pool, mg, max_iters=5, candidate_width=65)
    rp = np.full(bm.n_blocks + 1, 8, np.int32)  # block 0 with 8 rook neighbours
    rp[0] = 0
    with pytest.raises(ShapeMismatch):
        eng.set_rook(rp, np.zeros(8, np.int32))
    eng.close()
