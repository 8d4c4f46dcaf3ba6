"""The drop-in functions (reference signatures) on the GPU, against the golden vectors."""

import csv

import numpy as np
import pytest

from paper_2511_18296_b200 import evaluate as ev
from paper_2511_18296_b200.errors import InvalidArgs
from paper_2511_18296_b200.model import Schedule
from tests._fixtures import bm_from, load, tables_from

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", range(0, 20, 3))
def test_evaluate_candidates_parallel_signature(case, tmp_path):
    st, p = load("small"), f"kd{case}_"
    bm, tables = bm_from(st, p), tables_from(st, p)
    sched = Schedule(st[p + "assign"].astype(int))
    cand = [int(b) for b in st[p + "cand"]]
    outs = []
    for wc in (1, 2, 4, 16):
        moves, best = ev.evaluate_candidates_parallel(bm, sched, cand, tables, 0, True, worker_count=wc)
        outs.append((tuple((m.block, m.period, m.improvement, m.feasible) for m in moves),
                     None if best is None else (best.block, best.period, best.improvement)))
    assert all(o == outs[0] for o in outs[1:])
    moves, best = outs[0]
    assert [m[1] for m in moves] == st[p + "s0_best_t"].tolist()
    assert [m[2] for m in moves] == st[p + "s0_best_val"].tolist()
    g = st[p + "s0_best"]
    assert (best is None) == (g[0] < 0)
    if best is not None:
        assert best == (int(g[0]), int(g[1]), float(g[2]))
    # trace CSV (evaluate.py:423-428)
    path = tmp_path / "kernel.csv"
    ev.evaluate_candidates_parallel(bm, sched, cand[:3], tables, 0, True, trace_path=path)
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["candidate", "period", "feasible", "value"]
    assert len(rows) == 1 + 3 * bm.n_periods
    keyed = {(int(r[0]), int(r[1])): (int(r[2]), float(r[3])) for r in rows[1:]}
    for i, b in enumerate(cand[:3]):
        for t in range(bm.n_periods):
            assert keyed[(b, t)] == (int(st[p + "s0_trace_feas"][i, t]), float(st[p + "s0_trace_val"][i, t]))
    # rows in the order of sorted((b, t, feasible, value)) (evaluate.py:427); byte identity with the
    # reference's own file is tests/test_reference_path_gpu.py::test_trace_csv_bytes_equal_reference
    keys = [(int(r[0]), int(r[1]), int(r[2]), float(r[3])) for r in rows[1:]]
    assert keys == sorted(keys)
    with pytest.raises(InvalidArgs):
        ev.evaluate_candidates_parallel(bm, sched, cand, tables, 0, True, worker_count=0)


def test_check_feasible_and_repair_signatures():
    st = load("small")
    p = "kd4_"
    bm = bm_from(st, p)
    for k, a in enumerate(st[p + "rand"]):
        r = ev.check_feasible(bm, Schedule(a.astype(int)))
        assert r.precedence_violations == st[p + "rand_pred"][k]
        assert r.capacity_excess == st[p + "rand_excess"][k]
        assert r.violation == st[p + "rand_viol"][k]
        x = a.astype(int).copy()
        ev.precedence_repair_pass(bm, x)
        assert np.array_equal(x, st[p + "rand_repair"][k])
    fe = ev.check_feasible(bm_from(st, "feas_capacity_"), Schedule(np.array([0, 0])))
    assert fe.capacity_excess == 200.0 and fe.violation == 0.2 and not fe.feasible
