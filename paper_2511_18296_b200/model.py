"""Host-side data model: the reference's result records and the flat tables the
device holds.

`Schedule`, `CandidateMove` and `ViolationReport` mirror the reference dataclasses
(evaluate.py:28-79) field for field; when the engine is installed into `pitplan`
the drop-in functions return the reference's own classes instead (install.py).

`BlockModel` is the flattened, device-ready view of a `pitplan.blockmodel.Instance`
(blockmodel.py:91-185): precedence as an edge list plus CSR adjacency, per-block
masses / costs / geology features, per-period capacity.  `ScenarioTables` is the
per-scenario-set value table `vmax[s][b] = max_o v[s][b][o]` (evaluate.py:108-124)
plus the sigma[s][t] matrix (uncertainty.py:276-321).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidArgs, ShapeMismatch, ValidationError

UNMINED = -1  # blockmodel.py:18


@dataclass
class Schedule:
    """Stage-1 decision: period index per block, UNMINED (-1) for unmined (evaluate.py:28-60)."""

    assignment: np.ndarray

    def __post_init__(self):
        self.assignment = np.asarray(self.assignment, dtype=int)

    @classmethod
    def empty(cls, n_blocks: int) -> "Schedule":
        return cls(np.full(n_blocks, UNMINED, dtype=int))

    @property
    def n_blocks(self) -> int:
        return self.assignment.size

    def copy(self) -> "Schedule":
        return Schedule(self.assignment.copy())

    def digest(self) -> str:
        return hashlib.sha256(self.assignment.astype("<i8").tobytes()).hexdigest()


@dataclass
class ViolationReport:
    """evaluate.py:63-71."""

    precedence_violations: int
    capacity_excess: float
    violation: float

    @property
    def feasible(self) -> bool:
        return self.violation == 0.0


@dataclass
class CandidateMove:
    """evaluate.py:74-79."""

    block: int
    period: int
    improvement: float
    feasible: bool


@dataclass
class BlockModel:
    """Flat tables of one block-model instance (all numpy, host side)."""

    n_blocks: int
    n_periods: int
    edges_i: np.ndarray  # int32[E]  (i, j): i mined no later than j, reference list order
    edges_j: np.ndarray  # int32[E]
    mass: np.ndarray  # f64[B]
    cost: np.ndarray  # f64[B, T] undiscounted mining cost
    capacity: np.ndarray  # f64[T]
    discount_rate: float
    coords: np.ndarray  # f64[B, 3]
    alteration: np.ndarray  # f64[B]
    structural: np.ndarray  # f64[B]
    dist_intrusion: np.ndarray  # f64[B]
    base_grade: np.ndarray  # f64[B]
    price: float = 5.0
    recovery_by_mode: tuple = (0.85,)
    processing_cost_by_mode: tuple = (1.0,)
    n_modes: int = 1
    stored_values: np.ndarray | None = None  # f64[S_builtin, B, O] (blockmodel.py:141-147)
    plant_hours: np.ndarray | None = None  # f64[T] processing hours per period (blockmodel.py:97)
    mode_rates: tuple = ()  # throughput rate per operating mode (blockmodel.py:66)
    n_rock_types: int = 1
    _csr: tuple | None = field(default=None, repr=False)

    def __post_init__(self):
        B, T = self.n_blocks, self.n_periods
        self.edges_i = np.ascontiguousarray(self.edges_i, dtype=np.int32)
        self.edges_j = np.ascontiguousarray(self.edges_j, dtype=np.int32)
        self.mass = np.ascontiguousarray(self.mass, dtype=np.float64)
        self.cost = np.ascontiguousarray(self.cost, dtype=np.float64).reshape(B, T)
        self.capacity = np.ascontiguousarray(self.capacity, dtype=np.float64)
        self.coords = np.ascontiguousarray(self.coords, dtype=np.float64).reshape(B, 3)
        for name in ("alteration", "structural", "dist_intrusion", "base_grade"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.float64))
        if self.plant_hours is not None:
            self.plant_hours = np.ascontiguousarray(self.plant_hours, dtype=np.float64).reshape(T)
        self.mode_rates = tuple(float(r) for r in self.mode_rates)
        if T < 1:
            raise ValidationError("n_periods must be >= 1")
        if self.mass.shape != (B,) or self.capacity.shape != (T,):
            raise ShapeMismatch("mass / capacity arrays do not match n_blocks / n_periods")
        if self.edges_i.shape != self.edges_j.shape:
            raise ShapeMismatch("edge arrays differ in length")
        if self.edges_i.size and (
            self.edges_i.min() < 0 or self.edges_j.min() < 0
            or self.edges_i.max() >= B or self.edges_j.max() >= B
        ):
            raise ValidationError("precedence edge references unknown block")

    # -- derived -------------------------------------------------------------
    @property
    def n_edges(self) -> int:
        return int(self.edges_i.size)

    def csr(self):
        """(pred_ptr, pred_idx, succ_ptr, succ_idx): predecessors of j and successors
        of i in reference list order (blockmodel.py:180-184)."""
        if self._csr is None:
            B = self.n_blocks
            oj = np.argsort(self.edges_j, kind="stable")
            oi = np.argsort(self.edges_i, kind="stable")
            pred_ptr = np.zeros(B + 1, dtype=np.int32)
            succ_ptr = np.zeros(B + 1, dtype=np.int32)
            pred_ptr[1:] = np.cumsum(np.bincount(self.edges_j, minlength=B))
            succ_ptr[1:] = np.cumsum(np.bincount(self.edges_i, minlength=B))
            self._csr = (
                pred_ptr,
                np.ascontiguousarray(self.edges_i[oj], dtype=np.int32),
                succ_ptr,
                np.ascontiguousarray(self.edges_j[oi], dtype=np.int32),
            )
        return self._csr

    def discount(self) -> np.ndarray:
        """(1 + r) ** (-t) with Python float pow (evaluate.py:341)."""
        r = self.discount_rate
        return np.array([(1.0 + r) ** (-t) for t in range(self.n_periods)], dtype=np.float64)

    def diameter(self) -> float:
        """Instance diameter (evaluate.py:342-344)."""
        spans = self.coords.max(axis=0) - self.coords.min(axis=0)
        return float(np.sqrt((spans**2).sum()))

    def mean_capacity(self) -> float:
        """float(np.mean(mining_capacity)) (evaluate.py:103)."""
        return float(np.mean(self.capacity))

    def fingerprint(self) -> str:
        h = hashlib.sha256()
        for a in (self.edges_i, self.edges_j, self.mass, self.cost, self.capacity,
                  self.alteration, self.structural, self.dist_intrusion, self.coords):
            h.update(np.ascontiguousarray(a).tobytes())
        h.update(repr((self.n_blocks, self.n_periods, self.discount_rate)).encode())
        return h.hexdigest()

    # -- construction from the reference data model ----------------------------
    @classmethod
    def from_instance(cls, inst) -> "BlockModel":
        """Flatten a `pitplan.blockmodel.Instance` (duck-typed)."""
        blocks = inst.blocks
        B, T = len(blocks), int(inst.n_periods)
        prec = np.asarray(inst.precedence, dtype=np.int64).reshape(-1, 2)
        econ = inst.economics
        feats = np.array(
            [(b.features.alteration_intensity, b.features.structural_density,
              b.features.distance_to_intrusion) for b in blocks], dtype=np.float64,
        ).reshape(B, 3)
        stored = None
        if inst.modes and len(inst.modes[0].value) == B:
            stored = np.asarray(inst.builtin_values(), dtype=np.float64)
        return cls(
            n_blocks=B,
            n_periods=T,
            edges_i=prec[:, 0],
            edges_j=prec[:, 1],
            mass=inst.masses(),
            cost=inst.mining_costs().reshape(B, T),
            capacity=np.asarray(inst.mining_capacity, dtype=np.float64),
            discount_rate=float(inst.discount_rate),
            coords=inst.coords_array().reshape(B, 3),
            alteration=feats[:, 0],
            structural=feats[:, 1],
            dist_intrusion=feats[:, 2],
            base_grade=inst.base_grades(),
            price=float(econ.price),
            recovery_by_mode=tuple(econ.recovery_by_mode),
            processing_cost_by_mode=tuple(econ.processing_cost_by_mode),
            n_modes=len(inst.modes),
            stored_values=stored,
            plant_hours=np.asarray(inst.plant_hours, dtype=np.float64),
            mode_rates=tuple(float(m.rate) for m in inst.modes),
            n_rock_types=len(inst.rock_types),
        )

    @property
    def single_mode_fast(self) -> bool:
        """The stage-2 fast path of ScheduleEvaluator (evaluate.py:149-150): one mode, one rock
        type, positive rate."""
        return len(self.mode_rates) == 1 and self.n_rock_types == 1 and self.mode_rates[0] > 0


def scenario_values(bm: BlockModel, grades: np.ndarray | None, use_stored: bool = False) -> np.ndarray:
    """vmax[s][b] = max over modes of v[s][b][o] (evaluate.py:108-124, 300-303).

    v = ((grades * m) * price) * recovery_o - m * processing_cost_o, or the stored
    per-mode matrices when the scenario set is the instance's builtin one."""
    if use_stored:
        if bm.stored_values is None:
            raise InvalidArgs("scenario set uses stored values but the instance has none")
        return np.ascontiguousarray(bm.stored_values.max(axis=2))
    g = np.asarray(grades, dtype=np.float64)
    if g.ndim != 2 or g.shape[1] != bm.n_blocks:
        raise ShapeMismatch("scenario set does not match instance block count")
    m = bm.mass[None, :]
    best = None
    for o in range(bm.n_modes):
        rec = bm.recovery_by_mode[o % len(bm.recovery_by_mode)]
        cost = bm.processing_cost_by_mode[o % len(bm.processing_cost_by_mode)]
        v = g * m * bm.price * rec - m * cost
        best = v if best is None else np.maximum(best, v)
    return np.ascontiguousarray(best)


@dataclass
class ScenarioTables:
    """Per-scenario-set tables: vmax[S][B] (reference layout) and sigma[S][T] or None.

    vmax may be None when grades[S][B] is given: the engine then builds the value table on the
    device (pp_set_scenarios_grades, scenario_mode_values evaluate.py:116-124) and the host copy is
    fetched back only if someone asks for it (Engine.scenario_table)."""

    vmax: np.ndarray | None
    sigma: np.ndarray | None
    grades: np.ndarray | None = None  # [S][B], optional (lns_repair's mean grade, hybrid.py:214)

    def __post_init__(self):
        if self.vmax is None and self.grades is None:
            raise InvalidArgs("a scenario table needs vmax or grades")
        if self.vmax is not None:
            self.vmax = np.ascontiguousarray(self.vmax, dtype=np.float64)
        if self.sigma is not None:
            self.sigma = np.ascontiguousarray(self.sigma, dtype=np.float64)
            if self.sigma.shape[0] != self.n_scenarios:
                raise ShapeMismatch("sigma scenario count differs from the value table")

    @property
    def n_scenarios(self) -> int:
        return int((self.vmax if self.vmax is not None else np.asarray(self.grades)).shape[0])

    @classmethod
    def from_reference(cls, bm: BlockModel, scenarios, sigma) -> "ScenarioTables":
        """From a `pitplan.scenarios.ScenarioSet` and `UncertaintyFactors | None`: the stored
        per-mode values (use_stored_values) are reduced on the host; sampled grades go to the
        device as they are."""
        use_stored = bool(getattr(scenarios, "meta", {}).get("use_stored_values"))
        sig = None if sigma is None else np.asarray(sigma.sigma, dtype=np.float64)
        grades = getattr(scenarios, "grades", None)
        if use_stored:
            return cls(vmax=scenario_values(bm, None, True), sigma=sig, grades=grades)
        g = np.ascontiguousarray(grades, dtype=np.float64)
        if g.ndim != 2 or g.shape[1] != bm.n_blocks:
            raise ShapeMismatch("scenario set does not match instance block count")
        return cls(vmax=None, sigma=sig, grades=g)


@dataclass
class SequenceColumn:
    """A column of the Dantzig-Wolfe master (colgen.py:71-95), used when pitplan is absent."""

    id: int
    equipment: int
    assignment: np.ndarray
    mass_per_period: np.ndarray
    value: float
    reduced_cost: float = float("nan")
    birth: int = 0
    last_used: int = 0
    quality: float = 0.0

    def schedule(self) -> "Schedule":
        return Schedule(self.assignment.copy())


def cvar_k(n_scenarios: int) -> int:
    """ceil(0.1 n) lowest samples enter CVaR10 (saa.py:157)."""
    import math

    return max(1, math.ceil(0.1 * n_scenarios))


def rook_neighbor_map(bm: BlockModel) -> dict:
    """`_rook_neighbor_map` (hybrid.py:159-166): rook neighbours of every block, in the order
    of `rook_weights` (uncertainty.py)."""
    from .synth import rook_pairs

    ii, jj = rook_pairs(bm.coords)
    out: dict[int, list[int]] = {}
    for i, j in zip(ii.tolist(), jj.tolist()):
        out.setdefault(int(i), []).append(int(j))
    return out


def rook_padded(rook: dict, n_blocks: int):
    """rook_neighbor_map as a padded [B][L] id table (-1 padding, reference order), or None when a
    block has 8+ neighbours (numpy's mean switches from a sequential to a pairwise sum there)."""
    L = max((len(v) for v in rook.values()), default=0)
    if L >= 8:
        return None
    pad = np.full((n_blocks, max(L, 1)), -1, dtype=np.int64)
    for b, v in rook.items():
        pad[b, :len(v)] = v
    return pad


def neighbor_similarity_array(assign: np.ndarray, blocks: np.ndarray, mean_grade: np.ndarray,
                              pad: np.ndarray) -> np.ndarray:
    """scheduled_neighbor_similarity for an array of blocks at once, bit-identical to it: the
    mean of at most 7 values is numpy's sequential sum divided by the count."""
    ids = pad[blocks]
    valid = ids >= 0
    safe = np.where(valid, ids, 0)
    valid &= assign[safe] != UNMINED
    vals = np.abs(mean_grade[blocks][:, None] - mean_grade[safe])
    acc = np.zeros(len(blocks))
    started = np.zeros(len(blocks), dtype=bool)
    for k in range(ids.shape[1]):
        v = valid[:, k]
        acc = np.where(v, np.where(started, acc + vals[:, k], vals[:, k]), acc)
        started |= v
    cnt = valid.sum(axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        mean = acc / cnt
    return np.where(cnt > 0, -mean, -np.inf)


def scheduled_neighbor_similarity(assign: np.ndarray, blocks, mean_grade: np.ndarray, rook: dict) -> dict:
    """`_scheduled_neighbor_similarity` (hybrid.py:142-156): minus the mean absolute grade
    difference to the already-scheduled rook neighbours; -inf without one."""
    sims = {}
    for b in blocks:
        vals = [abs(mean_grade[b] - mean_grade[j]) for j in rook.get(b, ()) if assign[j] != UNMINED]
        sims[b] = -float(np.mean(vals)) if vals else -np.inf
    return sims


@dataclass
class VaeDecoder:
    """The decoder half of the reference's VAE (vae.py:61-93; nn.py:20-53): dense layers
    (W[out][in], b[out]) with relu between them and a linear last layer, then
    y * norm_std + norm_mean, clamped at zero by the prior decode (vae.py:284-292).  The engine
    runs it on the device (pp_set_vae_decoder / pp_vae_decode / pp_set_scenarios_vae)."""

    layers: list  # [(W, b)], W[out][in]
    norm_mean: np.ndarray  # [B]
    norm_std: np.ndarray  # [B]

    @property
    def widths(self) -> list:
        return [int(self.layers[0][0].shape[1])] + [int(W.shape[0]) for W, _ in self.layers]

    @property
    def latent_dim(self) -> int:
        return self.widths[0]

    def packed(self) -> np.ndarray:
        """W then b of every layer, concatenated (the C-ABI layout)."""
        return np.concatenate([np.concatenate([np.ascontiguousarray(W, dtype=np.float64).ravel(),
                                               np.ascontiguousarray(b, dtype=np.float64).ravel()])
                               for W, b in self.layers])

    def decode_host(self, z: np.ndarray) -> np.ndarray:
        """numpy restatement (row by row, as vae.py:288-291): test infrastructure for the device
        decode, which agrees with it to rounding."""
        rows = []
        for zi in np.atleast_2d(np.asarray(z, dtype=np.float64)):
            h = zi[None, :]
            for k, (W, b) in enumerate(self.layers):
                h = h @ W.T + b
                if k < len(self.layers) - 1:
                    h = np.maximum(h, 0.0)
            rows.append((h * self.norm_std + self.norm_mean)[0])
        return np.maximum(np.array(rows), 0.0)

    @classmethod
    def from_reference(cls, model) -> "VaeDecoder":
        """From a trained `pitplan.vae.VaeModel`."""
        return cls([(np.asarray(l.W, dtype=np.float64), np.asarray(l.b, dtype=np.float64)) for l in model.decoder.layers],
                   np.asarray(model.norm_mean, dtype=np.float64), np.asarray(model.norm_std, dtype=np.float64))

    @classmethod
    def random_init(cls, n_blocks: int, norm_mean: np.ndarray, norm_std: np.ndarray, latent_dim: int = 16,
                    widths: tuple = (64, 128, 256), seed: int = 0) -> "VaeDecoder":
        """The reference architecture (VaeConfig defaults, vae.py:32-44) with freshly initialised
        weights (Mlp.init's he / xavier scales, nn.py:24-27, 37-42): a synthetic scenario source of
        the right shape when no trained model is at hand."""
        rng = np.random.default_rng(seed)
        sizes = [latent_dim, *widths, n_blocks]
        layers = []
        for k in range(len(sizes) - 1):
            n_in, n_out = sizes[k], sizes[k + 1]
            std = np.sqrt(2.0 / n_in) if k < len(sizes) - 2 else np.sqrt(1.0 / n_in)
            layers.append((rng.standard_normal((n_out, n_in)) * std, np.zeros(n_out)))
        return cls(layers, np.asarray(norm_mean, dtype=np.float64), np.asarray(norm_std, dtype=np.float64))
