"""Multi-rank evaluation with real engines: world size 2 over gloo, both ranks on cuda:0 (this
environment has one GPU; no kernel of one rank waits on the other's, only the host collectives
do).  The sharded all-gather argmax and realism key reduced by pp_reduce_best must equal a
single-engine evaluation of the whole candidate list, and the sharded lns_repair (broadcast delta,
pp_apply_moves on every replica) must return the reference's schedule (golden C1 run) on both
ranks."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_18296_b200 import evaluate as ev
        from paper_2511_18296_b200.distributed import DeviceShardedEvaluator, sharded_lns_repair
        from paper_2511_18296_b200.model import ScenarioTables, Schedule
        from tests._fixtures import config, load

        st = load("c1")
        c = config("C1")
        tables = ScenarioTables(c["vmax"], c["sigma"], grades=st["C1_grades"])
        e = ev._entry(c["bm"])
        ev._bind_scenarios(e, tables, True, None)
        e.engine.set_schedule(c["greedy"])
        sev = DeviceShardedEvaluator(e.engine)
        rng = np.random.default_rng(11)
        evals = []
        for k in range(4):
            cand = rng.integers(0, c["bm"].n_blocks, size=int(rng.integers(1, 4000))).astype(np.int32)
            best, real, _ = sev.evaluate(cand, None, net=bool(k % 2))
            evals.append((cand, bool(k % 2), best, real))
        out = sharded_lns_repair(c["bm"], Schedule(st["C1_destroy_in"][0]), [], tables, True, max_iters=40,
                                 destroy_fraction=0.1)
        q.put((rank, [(b, r) for _, _, b, r in evals], out.assignment.tolist(),
               [(cand.tolist(), net) for cand, net, _, _ in evals] if rank == 0 else None))
        ev.clear_cache()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_engines_match_single_engine(world):
    from paper_2511_18296_b200.engine import Engine
    from paper_2511_18296_b200.model import ScenarioTables
    from tests._fixtures import config, load

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, evals, assign, cands = q.get(timeout=600)
        res[r] = (evals, assign, cands)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(1, world):
        assert res[r][0] == res[0][0] and res[r][1] == res[0][1]
    st = load("c1")
    assert np.array_equal(np.array(res[0][1]), st["C1_lns"])
    c = config("C1")
    eng = Engine.from_tables(c["bm"], ScenarioTables(c["vmax"], c["sigma"]), c["greedy"])
    for (best, real), (cand, net) in zip(res[0][0], res[0][2]):
        single = eng.eval_candidates(np.array(cand, dtype=np.int32), None, net=net, realism=True)
        assert best == single["best"] and real == single["realism"]
    eng.close()
