"""Per-size policy ranking over MEASURED schedule costs.

The reference ranks policies with an analytic makespan model
(``gemmsched.costmodel``, costmodel.py:91-128) — explicitly not a hardware
measurement.  On the B200 the cost of a (size, policy) is the measured
device time of its schedule (``sweep.py``); what is kept from the reference
is the record shape and the ranking rule:

* ``CostEstimate`` fields ``makespan``/``utilization``/``atomic_writes``/
  ``full_stores``/``per_wg_cost`` (costmodel.py:61-73) — ``makespan`` is the
  median kernel time in microseconds and ``utilization`` the achieved
  fraction of the dense tensor-core peak;
* ``TuneRecord`` (costmodel.py:76-88) and the ranking of
  :func:`rank_costs` — ascending ``(makespan, Policy.sort_key())``, so
  equal times (identical schedules) credit the lowest canonical ordinal and
  data-parallel wins ties (costmodel.py:141-164);
* ``dp_utilization`` — the wave-quantisation efficiency T / (ceil(T/g)*g)
  (costmodel.py:131-138) that defines "wave-quantisation-bound" shapes.

The reference's analytic model itself (``CostParams``, ``estimate``,
``pick_winner``; costmodel.py:26-164) is restated here too, item-wise over a
``Schedule`` (bit-for-bit the reference's arithmetic order) and in closed form per
workgroup (``wg_terms``: vectorised, no item lists), and CALIBRATED to B200
measurements (``calibrate``): the constants that best reproduce
the measured winners of a tuned grid, plus an affine map from model units to
microseconds so that predictions compare across tile shapes.  A calibrated model is
the selection prior for sizes the Bloom filters never saw (``tiles.TileBank``).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .types import GridInfo, Policy, PolicyKind, ProblemSize, TileShape


@dataclass(frozen=True)
class CostEstimate:
    makespan: float
    utilization: float
    atomic_writes: int
    full_stores: int
    per_wg_cost: tuple[float, ...] = ()


@dataclass(frozen=True)
class TuneRecord:
    size: ProblemSize
    costs: tuple[tuple[Policy, CostEstimate], ...]
    winner: Policy
    runner_up: Policy
    gain: float


def rank_costs(size: ProblemSize, costs) -> TuneRecord:
    """Winner, runner-up and relative gain from (policy, estimate) pairs."""
    costs = tuple(costs)
    if not costs:
        raise ValueError("policies must be nonempty")
    order = sorted(costs, key=lambda pc: (pc[1].makespan, pc[0].sort_key()))
    best_p, best = order[0]
    second_p, second = order[1] if len(order) > 1 else order[0]
    gain = (second.makespan - best.makespan) / second.makespan if second.makespan > 0 else 0.0
    return TuneRecord(size=size, costs=costs, winner=best_p, runner_up=second_p, gain=gain)


def dp_utilization(grid: GridInfo, g: int) -> float:
    if grid.total_tiles < 1:
        raise ValueError("total_tiles must be >= 1")
    if g < 1:
        raise ValueError("g must be >= 1")
    waves = -(-grid.total_tiles // g)
    return grid.total_tiles / (waves * g)


# -- the reference's analytic model (costmodel.py:26-164) ----------------------------


@dataclass(frozen=True, slots=True)
class CostParams:
    """Per-iteration, per-store and per-atomic costs and the fraction of atomic cost
    hidden when data-parallel work follows (costmodel.py:26-58; same validation)."""

    c_mac: float = 1.0
    c_store: float = 4.0
    c_atomic: float = 16.0
    overlap: float = 0.75

    def __post_init__(self) -> None:
        for name in ("c_mac", "c_store", "c_atomic"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        if not 0.0 <= self.overlap <= 1.0:
            raise ValueError("overlap must be in [0, 1]")

    @classmethod
    def from_dict(cls, data: dict) -> "CostParams":
        known = {"c_mac", "c_store", "c_atomic", "overlap"}
        unknown = set(data) - known
        if unknown:
            raise ValueError(f"unknown cost parameter(s): {sorted(unknown)}")
        return cls(**{k: float(v) for k, v in data.items()})

    @classmethod
    def from_json(cls, path) -> "CostParams":
        with open(path, "r", encoding="utf-8") as fh:
            data = json.load(fh)
        if not isinstance(data, dict):
            raise ValueError("cost parameter file must hold a JSON object")
        return cls.from_dict(data)

    def to_dict(self) -> dict:
        return {"c_mac": self.c_mac, "c_store": self.c_store, "c_atomic": self.c_atomic, "overlap": self.overlap}


def estimate(sched, params: CostParams) -> CostEstimate:
    """Cost a ``Schedule`` workgroup by workgroup (costmodel.py:91-128): iterations x
    c_mac, c_store per full store, c_atomic per partial -- discounted by ``overlap``
    when a data-parallel item follows it in the same workgroup."""
    from .scheduler import Phase, WriteMode

    per_wg = []
    atomic_writes = 0
    full_stores = 0
    for items in sched.assignments:
        last_dp = -1
        for i, item in enumerate(items):
            if item.phase is Phase.DATA_PARALLEL:
                last_dp = i
        cost = 0.0
        for i, item in enumerate(items):
            cost += item.iterations * params.c_mac
            if item.write_mode is WriteMode.FULL_STORE:
                cost += params.c_store
                full_stores += 1
            else:
                atomic_writes += 1
                cost += params.c_atomic * (1.0 - params.overlap) if i < last_dp else params.c_atomic
        per_wg.append(cost)
    makespan = max(per_wg) if per_wg else 0.0
    util = (sched.grid.total_iters * params.c_mac) / (sched.g * makespan) if makespan > 0 else 1.0
    return CostEstimate(makespan, util, atomic_writes, full_stores, tuple(per_wg))


def pick_winner(size: ProblemSize, tile: TileShape, hw, policies: list, params: CostParams) -> TuneRecord:
    """Estimate every policy's schedule and rank by makespan (costmodel.py:141-164)."""
    from .scheduler import build_schedule

    if not policies:
        raise ValueError("policies must be nonempty")
    return rank_costs(size, ((p, estimate(build_schedule(size, tile, hw, p), params)) for p in policies))


def wg_terms(size: ProblemSize, tile: TileShape, g: int, policy: Policy) -> np.ndarray:
    """Closed-form per-workgroup cost terms, float64 ``[g, 4]``: (iterations, full stores,
    partials paying full c_atomic, partials followed by data-parallel work).

    cost_x = c_mac*t0 + c_store*t1 + c_atomic*(t2 + (1-overlap)*t3) is ``estimate``'s
    per-workgroup cost without materialising the items (SK range
    [lo, hi) of ceil(I/g) iterations, DP tiles x, x+g, ... < dp; Stream-K-first hybrids
    run their partials before their data-parallel tiles, DP-first ones after).
    """
    mt = -(-size.m // tile.blk_m)
    nt = -(-size.n // tile.blk_n)
    ipt = -(-size.k // tile.blk_k)
    T = mt * nt
    if policy.kind is PolicyKind.DATA_PARALLEL:
        sk = 0
    elif policy.kind is PolicyKind.ALL_STREAM_K:
        sk = T
    else:
        rem = T % g
        sk = min(T, (policy.sk_batches - 1) * g + (rem or g))
    dp = T - sk
    I = sk * ipt
    if I >= 2 ** 53 or T * ipt >= 2 ** 53:
        raise ValueError("problem too large for the closed-form cost terms")
    x = np.arange(g, dtype=np.int64)
    ipw = -(-I // g) if I else 0
    lo = np.minimum(x * ipw, I)
    hi = np.minimum((x + 1) * ipw, I)
    busy = hi > lo
    n_items = np.where(busy, (hi - 1) // ipt - lo // ipt + 1, 0) if ipt else np.zeros(g, np.int64)
    n_full = np.where(busy, np.maximum(0, hi // ipt - (-(-lo // ipt))), 0) if ipt else np.zeros(g, np.int64)
    atomic = n_items - n_full
    n_dp = np.where(x < dp, -(-(dp - x) // g), 0)
    disc = policy.kind is PolicyKind.HYBRID and policy.sk_first
    out = np.empty((g, 4), dtype=np.float64)
    out[:, 0] = (hi - lo) + n_dp * ipt
    out[:, 1] = n_full + n_dp
    out[:, 2] = np.where(disc & (n_dp > 0), 0, atomic)
    out[:, 3] = np.where(disc & (n_dp > 0), atomic, 0)
    return out


def _weights(params: CostParams) -> np.ndarray:
    return np.array([params.c_mac, params.c_store, params.c_atomic, params.c_atomic * (1.0 - params.overlap)])


def estimate_closed(size: ProblemSize, tile: TileShape, g: int, policy: Policy, params: CostParams) -> float:
    """Model makespan from ``wg_terms`` (equal to ``estimate(...).makespan`` up to float
    summation order)."""
    return float((wg_terms(size, tile, g, policy) @ _weights(params)).max())


# -- calibration to B200 measurements ------------------------


@dataclass(frozen=True)
class Calibration:
    """Constants fitted to measured winners, and model units -> microseconds."""

    tile: TileShape
    g: int
    params: CostParams
    us_offset: float
    us_per_unit: float
    fraction_within: float  # in-sample: model pick within tolerance of the measured best
    tolerance: float
    sizes: int

    def predict_us(self, size: ProblemSize, policy: Policy) -> float:
        return self.us_offset + self.us_per_unit * estimate_closed(size, self.tile, self.g, policy, self.params)

    def to_dict(self) -> dict:
        return {"tile": [self.tile.blk_m, self.tile.blk_n, self.tile.blk_k], "g": self.g,
                "params": self.params.to_dict(), "us_offset": self.us_offset, "us_per_unit": self.us_per_unit,
                "fraction_within": self.fraction_within, "tolerance": self.tolerance, "sizes": self.sizes}

    @classmethod
    def from_dict(cls, d: dict) -> "Calibration":
        return cls(TileShape(*d["tile"]), int(d["g"]), CostParams.from_dict(d["params"]), float(d["us_offset"]),
                   float(d["us_per_unit"]), float(d["fraction_within"]), float(d["tolerance"]), int(d["sizes"]))


CALIBRATION_GRID = {
    "c_store": (0.0, 0.5, 1.0, 2.0, 4.0, 8.0, 16.0, 32.0),
    "c_atomic": (0.0, 1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0, 128.0),
    "overlap": (0.0, 0.25, 0.5, 0.75, 1.0),
}


def calibrate(measured, tile: TileShape, g: int, tolerance: float = 0.2, grid: dict | None = None) -> Calibration:
    """Fit ``CostParams`` (c_mac = 1: only ratios rank) to measured policy times.

    ``measured``: iterable of ``(ProblemSize, [(Policy, microseconds), ...])`` over the
    same policy list for every size.  Every grid point is scored by the fraction of sizes
    whose model-picked policy (reference tie-break) measures within ``tolerance`` of that
    size's fastest, ties broken by the geometric-mean slowdown; the winner's makespans are
    then mapped to microseconds by a relative-error least-squares fit ``us = a + b*m``.
    """
    measured = list(measured)
    if not measured:
        raise ValueError("need at least one measured size")
    policies = sorted({p for _, row in measured for p, _ in row}, key=lambda p: p.sort_key())
    col = {p: i for i, p in enumerate(policies)}
    S, P = len(measured), len(policies)
    us = np.full((S, P), np.inf)
    terms = np.zeros((S, P, g, 4))
    for si, (size, row) in enumerate(measured):
        for pol, t in row:
            us[si, col[pol]] = t
        for pol in policies:
            terms[si, col[pol]] = wg_terms(size, tile, g, pol)
    best_us = us.min(axis=1)
    grid = grid or CALIBRATION_GRID
    best = None
    for cs in grid["c_store"]:
        for ca in grid["c_atomic"]:
            for ov in grid["overlap"]:
                w = np.array([1.0, cs, ca, ca * (1.0 - ov)])
                span = (terms @ w).max(axis=2)              # [S, P]
                pick = span.argmin(axis=1)                  # first minimum = reference tie-break
                ratio = us[np.arange(S), pick] / best_us
                score = (float((ratio <= 1.0 + tolerance).mean()), -float(np.log(ratio).mean()))
                if best is None or score > best[0]:
                    best = (score, CostParams(1.0, cs, ca, ov), span)
    (frac, _), params, span = best
    m, t = span.ravel(), us.ravel()
    ok = np.isfinite(t) & (t > 0)
    m, t = m[ok], t[ok]
    # minimise sum(((a + b m) - t) / t)^2: weighted least squares with weights 1/t^2
    wgt = 1.0 / t
    A = np.stack([wgt, m * wgt], axis=1)
    (a, b), *_ = np.linalg.lstsq(A, np.ones_like(t), rcond=None)
    return Calibration(tile, g, params, float(a), float(b), frac, tolerance, S)

