"""Multi-rank host logic on CPU: world_size 2 (and 3) over gloo, oracle-backed shards.

The sharded all-gather argmax must select exactly the move a single evaluation of the
whole candidate list selects (evaluate.py:404-421), and the broadcast delta must leave
every replica's schedule identical."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2511_18296_b200.distributed import (
    better, pack_best, reduce_best, shard_bounds, unpack_best)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 16667, 250005):
        for w in (1, 2, 3, 8):
            parts = [shard_bounds(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1


def test_pack_roundtrip_and_order():
    recs = [(5, 2, 10.0), None, (3, 7, 10.0), (3, 1, 10.0), (9, 0, 9.5)]
    packed = np.stack([pack_best(r) for r in recs])
    assert unpack_best(packed) == recs
    assert reduce_best(recs) == (3, 1, 10.0)
    assert better((1, 0, -0.0), (0, 0, 0.0)) is False  # -0.0 == 0.0 -> lower block wins
    assert reduce_best([None, None]) is None


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2511_18296_b200.distributed import ShardedEvaluator
        from tests._fixtures import config

        c = config("C1")
        o = oracle.Oracle(c["bm"], c["vmax"], c["sigma"])
        assign = c["assign"].copy()

        def shard_fn(cand):
            if len(cand) == 0:
                return None
            return o.eval_candidates(assign, cand, None, net=True)["best"]

        ev = ShardedEvaluator(shard_fn)
        out = []
        for it in range(3):
            best, _ = ev.evaluate(c["cand"])
            move = ev.broadcast_move(None if best is None else (best[0], (best[1] + 1) % c["T"]), src=0)
            if move is not None:
                assign[move[0]] = move[1]
            out.append((best, int(np.sum(assign.astype(np.int64) * np.arange(assign.size)))))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_argmax_matches_single_process(world):
    from oracle import oracle
    from tests._fixtures import config

    oracle.build()
    c = config("C1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank saw the same global best and the same schedule after each broadcast delta
    for r in range(1, world):
        assert res[r] == res[0]
    # and the global best equals the single-process evaluation of the whole list
    o = oracle.Oracle(c["bm"], c["vmax"], c["sigma"])
    assign = c["assign"].copy()
    for best, _ in res[0]:
        single = o.eval_candidates(assign, c["cand"], None, net=True)["best"]
        assert best == single
        assign[best[0]] = (best[1] + 1) % c["T"]
