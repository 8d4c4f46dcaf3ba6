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
        """Global best move over all ranks' shards; identical on every rank.  The gathered
        records are reduced by `reduce_fn` (default: the host order of evaluate.py:404-409;
        DeviceShardedEvaluator reduces them with pp_reduce_best on the device)."""
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


class DeviceShardedEvaluator:
    """Candidate sharding with one `Engine` per rank.

    Every rank holds the static tables and a replica of the schedule; `evaluate(cand)` takes the
    GLOBAL candidate list (identical on every rank), evaluates this rank's contiguous shard on its
    GPU and all-gathers two 16-byte records per rank -- the shard's best move (evaluate.py:404-409
    order) and its realism-fallback key (hybrid.py:256-263) -- which `pp_reduce_best` reduces on
    the device; every rank gets the same global records.  `apply(move, src)` broadcasts the
    accepted (block, period) delta from the deciding rank and applies it to every replica
    (`pp_apply_moves`; the period masses are recomputed with the pairwise tree, never patched).
    NCCL keeps the exchanged records in device memory; gloo (CPU tests) stages them on the host.
    """

    def __init__(self, engine, group=None):
        import torch
        import torch.distributed as dist

        self.eng = engine
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.dev = torch.device("cuda", engine.device)
        # a stream of our own: handle 0 (torch's legacy default stream) means "the engine's own
        # stream" to the C ABI, which would not be ordered after torch's copies
        self.stream = torch.cuda.Stream(self.dev)
        self._gath = torch.empty(self.world * 4, dtype=torch.float64, device=self.dev if self.nccl else "cpu")
        self._red = torch.empty(4, dtype=torch.float64, device=self.dev)

    def local_shard(self, cand) -> np.ndarray:
        lo, hi = shard_bounds(len(cand), self.world, self.rank)
        return np.ascontiguousarray(np.asarray(cand)[lo:hi], dtype=np.int32)

    def evaluate(self, cand, scenario=None, *, net=False, use_sigma=True):
        """(global best, global realism key, this rank's result dict or None); the moves are
        (block, period, value) tuples, value = improvement / geological consistency."""
        import torch

        shard = self.local_shard(cand)
        res = None
        if shard.size:
            res = self.eng.eval_candidates(shard, scenario, net=net, use_sigma=use_sigma, realism=True)
        mine = np.concatenate([pack_best(res["best"] if res else None), pack_best(res["realism"] if res else None)])
        t = torch.from_numpy(mine)
        with torch.cuda.stream(self.stream):
            if self.nccl:
                t = t.to(self.dev)
                self.dist.all_gather_into_tensor(self._gath, t, group=self.group)
                g = self._gath
            else:
                parts = [torch.empty(4, dtype=torch.float64) for _ in range(self.world)]
                self.dist.all_gather(parts, t, group=self.group)
                g = torch.cat(parts).to(self.dev)
            g = g.view(self.world, 2, 2)
            best_recs = g[:, 0, :].contiguous()
            real_recs = g[:, 1, :].contiguous()
            self.eng.reduce_best_device(best_recs, self._red[0:2], stream=self.stream.cuda_stream)
            self.eng.reduce_best_device(real_recs, self._red[2:4], stream=self.stream.cuda_stream)
            red = self._red.cpu().numpy()
        best, real = unpack_best(red.reshape(2, 2))
        return best, real, res

    def apply(self, move, src: int = 0):
        """Broadcast the accepted (block, period) from `src` and apply it on every replica."""
        import torch

        buf = torch.tensor(list(move) if move is not None else [-1, -1], dtype=torch.int64)
        if self.nccl:
            buf = buf.to(self.dev)
        self.dist.broadcast(buf, src=src, group=self.group)
        b, t = (int(x) for x in buf.cpu().tolist())
        if b < 0:
            return None
        self.eng.apply_moves([b], [t])
        return (b, t)


def sharded_lns_repair(instance, schedule, unassigned, scenarios, sigma, group=None, max_iters: int = 100,
                       realism_threshold: float = 0.5, destroy_fraction: float = 0.0, candidate_width: int = 16,
                       strict: bool = False, only_positive: bool = False, net_mining_cost: bool = False,
                       params=None, seed: int = 0):
    """lns_repair (hybrid.py:169-274) with its insertion evaluations sharded over the ranks of
    `group` (one GPU each).  The destroy step and the candidate ranking are replicated (identical
    host work on identical replicas); each round's candidate list is evaluated shard by shard,
    the global best and realism key come from the all-gathered records (pp_reduce_best), rank 0
    decides the move and broadcasts it, every rank applies it (pp_apply_moves).  Returns the same
    schedule as the single-GPU drop-in (and the reference) on every rank."""
    from . import evaluate as ev
    from .errors import RepairStalled
    from .model import neighbor_similarity_array, rook_neighbor_map, rook_padded, scheduled_neighbor_similarity

    e = ev._entry(instance)
    ev._bind_scenarios(e, scenarios, sigma, params)
    sched = schedule.copy()
    before = ev.check_feasible(instance, sched)
    pool = {int(b) for b in unassigned}
    grades = getattr(scenarios, "grades", None)
    if grades is None:
        raise ev.InvalidArgs("lns_repair needs scenarios with grades[S][B] (hybrid.py:214)")
    mean_grade = np.asarray(grades).mean(axis=0)
    a, added = e.engine.lns_destroy(np.asarray(sched.assignment)[None, :], mean_grade, destroy_fraction)
    sched.assignment[...] = a[0]
    pool.update(int(b) for b in np.nonzero(added[0])[0])
    spatial = e.engine.spatial()
    rook = e.rook if e.rook is not None else rook_neighbor_map(e.bm)
    e.rook = rook
    pad = e.rook_pad if e.rook_pad is not None else rook_padded(rook, e.bm.n_blocks)
    e.rook_pad = pad
    in_pool = np.zeros(e.bm.n_blocks, dtype=bool)
    in_pool[list(pool)] = True
    sev = DeviceShardedEvaluator(e.engine, group)
    e.engine.set_schedule(sched.assignment)
    iters, stalled = 0, False
    while pool and iters < max_iters:
        if pad is not None:
            ids = np.flatnonzero(in_pool)
            sims = neighbor_similarity_array(sched.assignment, ids, mean_grade, pad)
            cand = ids[np.lexsort((ids, -sims))[:candidate_width]]
        else:
            sims = scheduled_neighbor_similarity(sched.assignment, pool, mean_grade, rook)
            cand = np.array(sorted(pool, key=lambda b: (-sims[b], b))[:candidate_width])
        best, real, _ = sev.evaluate(cand, None, net=net_mining_cost, use_sigma=sigma is not None)
        if best is None or (only_positive and best[2] <= 0.0):
            stalled = best is None
            break
        chosen = best if spatial[best[0]] >= realism_threshold else real
        move = sev.apply((chosen[0], chosen[1]) if sev.rank == 0 else None, src=0)
        sched.assignment[move[0]] = move[1]
        pool.discard(move[0])
        in_pool[move[0]] = False
        iters += 1
    after = ev.check_feasible(instance, sched)
    if after.violation > before.violation:
        return schedule.copy()
    if stalled and strict:
        raise RepairStalled("no feasible insertion for remaining blocks", schedule=sched)
    return sched
