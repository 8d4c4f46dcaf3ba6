"""Seeded synthetic inputs, bit-identical to the reference's own builders.

The benchmark and the GPU parity tests run on a box without the reference
checkout, so the inputs the reference would build are rebuilt here, vectorised:

* `generate_block_model`  <- `generate_synthetic` (blockmodel.py:325-488)
* `sample_lognormal`      <- scenarios.py:130-146
* `uncertainty_sigma`     <- `uncertainty_factors` (uncertainty.py:50-111, 173-182, 276-321)
* `full_greedy`           <- `HybridSearch._full_greedy` (hybrid.py:643-667)
* `greedy_initialize`     <- hybrid.py:86-125
* `topological_order`     <- blockmodel.py:228-245
* `substream`             <- rng.py:15-32

Same numpy calls in the same order on the same machine give the same bits; the
golden fixtures carry sha256 digests of the reference-built tables so tests can
tell when a host's numpy/BLAS build changes the last ulp (then the oracle, run
on the same inputs, stays the parity checker).  Host-side input construction
only: nothing here is on the measured path.
"""

from __future__ import annotations

import heapq

import numpy as np

from .model import UNMINED, BlockModel


# -- rng.py:15-32 -------------------------------------------------------------
def substream(seed: int, *keys) -> np.random.Generator:
    words = [int(seed) & 0xFFFFFFFFFFFFFFFF]
    for key in keys:
        if isinstance(key, (int, np.integer)):
            k = int(key)
            words += [k & 0xFFFFFFFF, (k >> 32) & 0xFFFFFFFF]
        elif isinstance(key, str):
            words += list(key.encode("utf-8"))
        else:
            raise TypeError(f"unsupported substream key: {key!r}")
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(words)))


# -- blockmodel.py:325-355 ------------------------------------------------------
def _box_smooth(rng: np.random.Generator, dims, radius_cap: int = 2) -> np.ndarray:
    f = rng.standard_normal(tuple(dims))
    for axis, size in enumerate(dims):
        r = min(radius_cap, max(0, (size - 1) // 2))
        if size == 1 or r == 0:
            continue
        total = np.zeros_like(f)
        hits = np.zeros_like(f)
        idx = np.arange(size)
        shape = [1, 1, 1]
        shape[axis] = size
        for d in range(-r, r + 1):
            # a shifted copy that does not wrap around the grid edge
            valid = ((idx - d >= 0) & (idx - d < size)).astype(f.dtype).reshape(shape)
            moved = np.roll(f, d, axis=axis)
            if d != 0:
                moved = moved * np.broadcast_to(valid, f.shape)
                w = np.broadcast_to(valid, f.shape)
            else:
                w = np.ones_like(f)
            total += moved
            hits += w
        f = total / hits
    sd = f.std()
    if sd > 0:
        f = (f - f.mean()) / sd
    return f


def generate_block_model(
    n_blocks: int,
    grid_dims,
    n_periods: int,
    n_modes: int,
    seed: int,
    *,
    n_scenarios: int = 2,
    n_rock_types: int = 2,
    spacing: float = 1.0,
    grade_sigma: float = 0.5,
    capacity_factor: float = 1.3,
    mining_cost_rate: float = 0.8,
) -> BlockModel:
    """Vectorised restatement of `generate_synthetic` (blockmodel.py:358-488)."""
    nx, ny, nz = (int(d) for d in grid_dims)
    if n_blocks != nx * ny * nz:
        raise ValueError(f"n_blocks={n_blocks} != product of grid dims {grid_dims}")
    rng = substream(seed, "synthetic")
    grades3 = np.exp(grade_sigma * _box_smooth(rng, (nx, ny, nz)))

    # block b = (iz*ny + iy)*nx + ix, layer 0 is the surface
    iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ix, iy, iz = ix.ravel(), iy.ravel(), iz.ravel()
    coords = np.stack([ix * spacing, iy * spacing, iz * spacing], axis=1).astype(np.float64)

    # 45-degree cone: up to 9 predecessors in the layer above, (dy, dx) row-major
    slots_i, slots_ok = [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            px, py = ix + dx, iy + dy
            ok = (iz > 0) & (px >= 0) & (px < nx) & (py >= 0) & (py < ny)
            slots_i.append(((iz - 1) * ny + py) * nx + px)
            slots_ok.append(ok)
    pi = np.stack(slots_i, axis=1)
    ok = np.stack(slots_ok, axis=1)
    edges_i = pi[ok]
    edges_j = np.broadcast_to(np.arange(n_blocks)[:, None], pi.shape)[ok]

    masses = rng.uniform(800.0, 1200.0, size=n_blocks)
    gx = (coords[:, 0] / spacing).astype(np.int64)
    gy = (coords[:, 1] / spacing).astype(np.int64)
    gz = (coords[:, 2] / spacing).astype(np.int64)
    base_flat = grades3[gx, gy, gz]

    scen_fields = np.empty((n_scenarios, n_blocks))
    for s in range(n_scenarios):
        z = substream(seed, "synthetic-scen", s).standard_normal(n_blocks)
        scen_fields[s] = base_flat * np.exp(0.25 * z - 0.25**2 / 2)

    recovery = tuple(0.85 + 0.05 * o for o in range(n_modes))
    proc_cost = tuple(1.0 + 0.4 * o for o in range(n_modes))
    price = 6.0
    total_mass = masses.sum()
    cap = np.round(capacity_factor * total_mass / n_periods, 3)
    capacity = np.full(n_periods, cap, dtype=np.float64)

    stored = np.empty((n_scenarios, n_blocks, n_modes))
    for o in range(n_modes):
        stored[:, :, o] = scen_fields * masses[None, :] * price * recovery[o] - masses[None, :] * proc_cost[o]

    frng = substream(seed, "synthetic-feat")
    alteration = frng.uniform(0, 1, n_blocks)
    structural = frng.uniform(0, 1, n_blocks)
    intrusion = frng.uniform(0, spacing * max(nx, ny, nz), n_blocks)

    growth = np.array([1.0 + 0.02 * t for t in range(n_periods)])
    cost = np.round(masses[:, None] * mining_cost_rate * growth[None, :], 6)
    mean_rate = 500.0
    hours = np.full(n_periods, np.round(0.8 * cap / mean_rate, 3), dtype=np.float64)

    return BlockModel(
        n_blocks=n_blocks,
        n_periods=n_periods,
        edges_i=edges_i,
        edges_j=edges_j,
        mass=np.round(masses, 6),
        cost=cost,
        capacity=capacity,
        discount_rate=0.08,
        coords=coords,
        alteration=np.round(alteration, 9),
        structural=np.round(structural, 9),
        dist_intrusion=np.round(intrusion, 9),
        base_grade=np.round(base_flat, 9),
        price=price,
        recovery_by_mode=recovery,
        processing_cost_by_mode=proc_cost,
        n_modes=n_modes,
        stored_values=stored,
        plant_hours=hours,
        mode_rates=tuple(mean_rate * (1.0 + 0.2 * o) for o in range(n_modes)),
        n_rock_types=n_rock_types,
    )


# -- scenarios.py:130-146 --------------------------------------------------------
def sample_lognormal(bm: BlockModel, n_s: int, shock_sigma: float, seed: int) -> np.ndarray:
    """Mean-preserving lognormal grade shocks; returns grades[S][B]."""
    z = substream(seed, "lognormal").standard_normal((n_s, bm.n_blocks))
    return bm.base_grade[None, :] * np.exp(shock_sigma * z - shock_sigma**2 / 2.0)


# -- uncertainty.py:50-80 (rook adjacency in the reference's pair order) ------------
def rook_pairs(coords: np.ndarray):
    coords = np.asarray(coords, dtype=float)
    n = coords.shape[0]
    spacing = np.ones(3)
    for a in range(3):
        vals = np.unique(coords[:, a])
        if vals.size > 1:
            spacing[a] = np.min(np.diff(vals))
    key = np.rint(coords / spacing).astype(np.int64)
    lo = key.min(axis=0)
    span = key.max(axis=0) - lo + 1
    def enc(k):
        return ((k[:, 0] - lo[0]) * span[1] + (k[:, 1] - lo[1])) * span[2] + (k[:, 2] - lo[2])
    codes = enc(key)
    order = np.lexsort((np.arange(n), codes))
    sc = codes[order]
    # last block id wins for duplicate keys, as the reference's dict does
    last = np.r_[sc[1:] != sc[:-1], True]
    uc, ub = sc[last], order[last]
    nbr = np.full((n, 6), -1, dtype=np.int64)
    col = 0
    for axis in range(3):
        for step in (-1, 1):
            k2 = key.copy()
            k2[:, axis] += step
            inside = np.all((k2 >= lo) & (k2 < lo + span), axis=1)
            c2 = enc(np.where(inside[:, None], k2, lo))
            pos = np.clip(np.searchsorted(uc, c2), 0, max(uc.size - 1, 0))
            hit = inside & (uc[pos] == c2)
            nbr[:, col] = np.where(hit, ub[pos], -1)
            col += 1
    ok = nbr >= 0
    ii = np.broadcast_to(np.arange(n)[:, None], nbr.shape)[ok]
    return ii.astype(int), nbr[ok].astype(int)


def _morans_i(values: np.ndarray, ii: np.ndarray, jj: np.ndarray, w: np.ndarray) -> float:
    """uncertainty.py:95-111; nan for a zero-variance field."""
    n = values.size
    dev = values - values.mean()
    denom = float(dev @ dev)
    if denom <= 0:
        return float("nan")
    num = float(np.sum(w * dev[ii] * dev[jj]))
    return n * num / (float(w.sum()) * denom)


def uncertainty_sigma(bm: BlockModel, grades: np.ndarray, kappa: float = 0.1,
                      psi_weights=(0.4, 0.35, 0.25), psi_min: float = 0.5) -> np.ndarray:
    """sigma[S][T] of `uncertainty_factors` (uncertainty.py:276-321)."""
    grades = np.asarray(grades, dtype=float)
    n_s, n_t = grades.shape[0], bm.n_periods
    ii, jj = rook_pairs(bm.coords)
    w = np.ones(len(ii))
    diam = bm.diameter()
    w1, w2, w3 = psi_weights
    dist = bm.dist_intrusion
    dn = np.clip(dist / diam, 0.0, 1.0) if diam > 0 else np.zeros_like(dist)
    raw = float(np.mean(w1 * bm.alteration + w2 * bm.structural + w3 * dn))
    raw = min(max(raw, 0.0), 1.0)
    psi = psi_min + (1.0 - psi_min) * raw
    phi = np.exp(-kappa * np.arange(n_t))
    f_spatial = np.zeros(n_s)
    for s in range(n_s):
        mi = _morans_i(grades[s], ii, jj, w)
        mean = grades[s].mean()
        local = grades[s].std() / mean if mean > 0 else 0.0
        f_spatial[s] = (1.0 + local) if mi != mi else (1.0 - mi + local)
    return np.clip(f_spatial[:, None] * phi[None, :] * psi, 1e-6, 2.0)


# -- blockmodel.py:228-245 -----------------------------------------------------------
def topological_order(bm: BlockModel) -> np.ndarray:
    pred_ptr, _, succ_ptr, succ_idx = bm.csr()
    indeg = np.diff(pred_ptr).astype(np.int64)
    heap = [int(b) for b in np.nonzero(indeg == 0)[0]]
    heapq.heapify(heap)
    out = []
    sp, si = succ_ptr.tolist(), succ_idx.tolist()
    deg = indeg.tolist()
    while heap:
        b = heapq.heappop(heap)
        out.append(b)
        for k in range(sp[b], sp[b + 1]):
            c = si[k]
            deg[c] -= 1
            if deg[c] == 0:
                heapq.heappush(heap, c)
    if len(out) != bm.n_blocks:
        raise ValueError("cycle in precedence graph")
    return np.asarray(out, dtype=np.int64)


def _earliest_fit(bm: BlockModel, order) -> np.ndarray:
    pred_ptr, pred_idx, _, _ = bm.csr()
    pp, pi = pred_ptr.tolist(), pred_idx.tolist()
    m = bm.mass.tolist()
    cap = bm.capacity.tolist()
    T = bm.n_periods
    assign = [UNMINED] * bm.n_blocks
    load = [0.0] * T
    for b in order:
        b = int(b)
        t_min = 0
        blocked = False
        for k in range(pp[b], pp[b + 1]):
            tp = assign[pi[k]]
            if tp == UNMINED:
                blocked = True
                break
            if tp > t_min:
                t_min = tp
        if blocked:
            continue
        for t in range(t_min, T):
            if load[t] + m[b] <= cap[t]:
                assign[b] = t
                load[t] += m[b]
                break
    return np.asarray(assign, dtype=np.int64)


def full_greedy(bm: BlockModel) -> np.ndarray:
    """Every block that fits, earliest-feasible in topological order (hybrid.py:643-667)."""
    return _earliest_fit(bm, topological_order(bm))


def greedy_initialize(bm: BlockModel, grades: np.ndarray, sigma: np.ndarray | None,
                      noise_rng: np.random.Generator | None = None) -> np.ndarray:
    """Value-density greedy (hybrid.py:86-125)."""
    n_s = grades.shape[0]
    sig0 = np.ones(n_s) if sigma is None else sigma[:, 0]
    vd = (grades * sig0[:, None]).mean(axis=0) * bm.mass
    if noise_rng is not None:
        vd = vd * np.exp(0.35 * noise_rng.standard_normal(vd.size))
    order = np.lexsort((np.arange(bm.n_blocks), -vd))
    return _earliest_fit(bm, order)


def candidate_blocks(n_blocks: int, n_candidates: int, seed: int = 3) -> np.ndarray:
    """`substream(seed, "cand").integers(0, B)` candidate draw of SURVEY.md §8(d)."""
    return substream(seed, "cand").integers(0, n_blocks, size=n_candidates).astype(np.int32)


def build_config(name: str):
    """The BASELINE.json configurations; returns a dict of inputs."""
    cfgs = {
        # C1: 4k blocks, 10 periods, 10 scenarios, 1000 candidates x 10 periods
        "C1": dict(n=4000, dims=(20, 20, 10), T=10, S=10, C=1000, cf=1.3),
        # C2: headline, 50k blocks, 15 periods, 20 scenarios, 16,667 candidates x 15
        "C2": dict(n=50000, dims=(50, 50, 20), T=15, S=20, C=16667, cf=1.3),
        # C3: capacity binds, 200 scenarios
        "C3": dict(n=50000, dims=(50, 50, 20), T=15, S=200, C=16667, cf=0.3),
        # C4: 200k blocks, 20 periods, 50 scenarios, 66,667 candidates x 15 (1M moves)
        "C4": dict(n=200000, dims=(100, 100, 20), T=20, S=50, C=50000, cf=1.3),
    }
    c = cfgs[name]
    bm = generate_block_model(c["n"], c["dims"], c["T"], 1, seed=1, n_rock_types=1,
                              capacity_factor=c["cf"])
    grades = sample_lognormal(bm, c["S"], 0.3, seed=2)
    sigma = uncertainty_sigma(bm, grades)
    assign = full_greedy(bm)
    cand = candidate_blocks(bm.n_blocks, c["C"])
    return dict(name=name, bm=bm, grades=grades, sigma=sigma, assign=assign, cand=cand, **c)
