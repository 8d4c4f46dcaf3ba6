"""Multi-GPU evaluation: candidate sharding, all-gather argmax, accepted-delta broadcast.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch on the B200 box, gloo
in the CPU tests).  Candidates are independent given (assignment, period masses)
(evaluate.py:357-389), so each rank evaluates a contiguous shard with no data-path
collective; the only exchanges are

  1. the per-rank best move, 16 bytes (value f64, block i32, period i32), all-gathered
     and reduced in the total order of evaluate.py:404-409 -- a deterministic
     "allreduce-argmax" that needs no custom NCCL op and returns the same move as a
     single-GPU evaluation of the whole candidate list;
  2. the accepted schedule delta (block, new period), broadcast from the driver rank so
     every replica of the schedule and its period masses stays identical.
"""

from __future__ import annotations

import numpy as np

NONE = (-np.inf, -1, -1)


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced shard [lo, hi) of n candidates for `rank`."""
    return (n * rank) // world, (n * (rank + 1)) // world


def pack_best(best) -> np.ndarray:
    """(block, period, value) | None -> float64[2] with the ints bit-packed (pp_best layout)."""
    rec = np.zeros(2, dtype=np.float64)
    if best is None:
        rec[0] = -np.inf
        rec.view(np.int32)[2:4] = (-1, -1)
    else:
        b, t, v = best
        rec[0] = v
        rec.view(np.int32)[2:4] = (b, t)
    return rec


def unpack_best(rec: np.ndarray):
    rec = np.ascontiguousarray(rec, dtype=np.float64).reshape(-1, 2)
    out = []
    for r in rec:
        b, t = (int(x) for x in r.view(np.int32)[2:4])
        out.append(None if b < 0 else (b, t, float(r[0])))
    return out


def better(x, y) -> bool:
    """x beats y in the order of evaluate.py:404-409 (value, then lower block, lower period)."""
    if y is None:
        return x is not None
    if x is None:
        return False
    bx, tx, vx = x
    by, ty, vy = y
    return vx > vy or (vx == vy and (bx, tx) < (by, ty))


def reduce_best(records):
    best = None
    for r in records:
        if better(r, best):
            best = r
    return best


class ShardedEvaluator:
    """Evaluate a candidate list across the ranks of a process group.

    `evaluate_shard(cand_shard) -> (block, period, value) | None` runs the local
    evaluation (an `Engine` on this rank's GPU in production; any callable in tests).
    """

    def __init__(self, evaluate_shard, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.evaluate_shard = evaluate_shard
        self.device = device

    def local_shard(self, cand: np.ndarray) -> np.ndarray:
        lo, hi = shard_bounds(len(cand), self.world, self.rank)
        return np.asarray(cand)[lo:hi]

    def evaluate(self, cand):
        """Global best move over all ranks' shards; identical on every rank."""
        import torch

        local = self.evaluate_shard(self.local_shard(cand))
        rec = torch.from_numpy(pack_best(local))
        if self.device is not None:
            rec = rec.to(self.device)
        gathered = [torch.empty_like(rec) for _ in range(self.world)]
        self.dist.all_gather(gathered, rec, group=self.group)
        recs = unpack_best(np.stack([g.cpu().numpy() for g in gathered]))
        return reduce_best(recs), local

    def broadcast_move(self, move, src: int = 0):
        """Broadcast the accepted (block, period) delta from `src`; returns it on every rank."""
        import torch

        buf = torch.tensor(list(move) if move is not None else [-1, -1], dtype=torch.int64)
        if self.device is not None:
            buf = buf.to(self.device)
        self.dist.broadcast(buf, src=src, group=self.group)
        b, t = (int(x) for x in buf.cpu().tolist())
        return None if b < 0 else (b, t)


def engine_shard_fn(engine, scenario=None, **flags):
    """`evaluate_shard` backed by an Engine (host buffers)."""

    def fn(cand_shard):
        if len(cand_shard) == 0:
            return None
        return engine.eval_candidates(cand_shard, scenario, **flags)["best"]

    return fn
