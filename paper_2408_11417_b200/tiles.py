"""Joint (tile shape, policy) selection: one Bloom bank per tile shape.

The reference tunes the seven policies for a single tile shape and notes
additional tuning parameters as future work (SURVEY §8(f) rank
4).  On the B200 the tile shape matters as much as the policy (e.g. the
256x256 CTA-pair tile is ~1.5x faster on large Llama projections, the
128x128 tile wins on skinny split-K shapes), so the sweep measures every
(tile, policy) and the winner of a size is inserted into the bank of its
tile.  Each per-tile bank is an ordinary reference-format ``SKPS`` bank; a
JSON manifest lists the tiles in priority order.

Query: candidates = union over tiles of (tile, p) for p in bank[tile].query(size),
plus the baseline (first tile, data-parallel), which is always evaluated.
There are no false negatives: the measured winner is always a candidate.
Sizes absent from every bank fall back to the baseline, or — with
``nearest=True`` — to the candidates of the nearest tuned power-of-two size,
``"corners"`` — the union over the enclosing power-of-two sizes, ``"model"`` — the
pick of the calibrated cost model (``costmodel.calibrate``, stored per tile in the
manifest as ``prior``), or ``"corners+model"`` — both.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

from .costmodel import Calibration, CostEstimate, TuneRecord, rank_costs
from .sieve import SieveBank
from .types import Policy, ProblemSize, TileShape, kernel_tile, tile_grid, tile_order

Config = tuple  # (TileShape, Policy)

BANK_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "banks", "b200")


def default_bank_dir() -> str:
    """The tile bank shipped with the package: per-tile SKPS banks + manifest built from the
    B200 sweep (``python -m paper_2408_11417_b200.sweep``), used by the bench and the CLI."""
    return BANK_DIR


def tile_label(t: TileShape) -> str:
    """``MxNxK`` for the reference's tile order on one workgroup per SM; ``bG`` appends G-row
    bands, ``gN`` a persistent grid of N workgroups (KernelTile)."""
    band, grid = tile_order(t), tile_grid(t)
    return f"{t.blk_m}x{t.blk_n}x{t.blk_k}" + (f"b{band}" if band else "") + (f"g{grid}" if grid else "")


def parse_tile(s: str) -> TileShape:
    """Inverse of :func:`tile_label`."""
    rest, _, grid = s.partition("g")
    dims, _, band = rest.partition("b")
    return kernel_tile(*(int(v) for v in dims.split("x")), int(band) if band else 0, int(grid) if grid else 0)


@dataclass(frozen=True)
class JointRecord:
    """Per-size measurements of every (tile, policy) and the joint winner."""

    size: ProblemSize
    per_tile: tuple  # ((TileShape, TuneRecord), ...) in tile priority order
    winner: Config
    winner_us: float

    def time_of(self, cfg: Config) -> float:
        tile, pol = cfg
        for t, rec in self.per_tile:
            if t == tile:
                for p, e in rec.costs:
                    if p == pol:
                        return e.makespan
        raise KeyError(cfg)


def joint_winner(size: ProblemSize, per_tile) -> JointRecord:
    """Argmin over (tile, policy); ties go to the earlier tile, then the reference tie-break."""
    best = None
    for ti, (tile, rec) in enumerate(per_tile):
        for pol, est in rec.costs:
            key = (est.makespan, ti, pol.sort_key())
            if best is None or key < best[0]:
                best = (key, (tile, pol))
    return JointRecord(size, tuple(per_tile), best[1], best[0][0])


class TileBank:
    """Per-tile SieveBanks behind one (tile, policy) query."""

    def __init__(self, tiles: list[TileShape], banks: list[SieveBank] | None = None, **bank_kwargs):
        if not tiles:
            raise ValueError("need at least one tile shape")
        self.tiles = list(tiles)
        self.banks = banks if banks is not None else [SieveBank(**bank_kwargs) for _ in tiles]
        if len(self.banks) != len(self.tiles):
            raise ValueError("one bank per tile")
        self._tuned_keys: set | None = None
        self.priors: list[Calibration | None] = [None] * len(self.tiles)  # per tile, optional

    @property
    def baseline(self) -> Config:
        return (self.tiles[0], Policy.data_parallel())

    def insert(self, size: ProblemSize, cfg: Config) -> None:
        tile, pol = cfg
        self.banks[self.tiles.index(tile)].insert(size, pol)

    def query(self, size: ProblemSize, nearest=False) -> list[Config]:
        """(tile, policy) candidates reported by the filters, tile-major.

        For a size absent from every filter: ``nearest=True`` (or ``"pow2"``) asks the
        filters about the nearest power-of-two size; ``nearest="corners"`` takes the union
        of their answers over the (up to 8) power-of-two sizes enclosing it.
        """
        out = [(t, p) for t, b in zip(self.tiles, self.banks) for p in b.query(size)]
        if out or not nearest:
            return out
        if nearest != "model":
            probes = snap_corners(size) if nearest in ("corners", "corners+model") else [snap_pow2(size)]
            for z in probes:
                if z == size:
                    continue
                for c in ((t, p) for t, b in zip(self.tiles, self.banks) for p in b.query(z)):
                    if c not in out:
                        out.append(c)
        if nearest in ("model", "corners+model") and any(c is not None for c in self.priors):
            pick = self.prior_pick(size)
            if pick not in out:
                out.append(pick)
        return out

    def prior_pick(self, size: ProblemSize) -> Config:
        """The (tile, policy) with the lowest calibrated-model time (ties: earlier tile,
        then the reference tie-break), over the tiles that carry a prior."""
        from .types import canonical_policies

        ckey = (size.m, size.n, size.k, tuple(id(c) for c in self.priors))
        cache = self.__dict__.setdefault("_prior_cache", {})
        if ckey in cache:
            return cache[ckey]
        best = None
        for ti, (tile, cal) in enumerate(zip(self.tiles, self.priors)):
            if cal is None:
                continue
            for pol in canonical_policies():
                key = (cal.predict_us(size, pol), ti, pol.sort_key())
                if best is None or key < best[0]:
                    best = (key, (tile, pol))
        if best is None:
            raise ValueError("no tile of this bank carries a calibrated cost-model prior")
        if len(cache) > 65536:
            cache.clear()
        cache[ckey] = best[1]
        return best[1]

    def candidates(self, size: ProblemSize, nearest=False) -> list[Config]:
        cand = self.query(size, nearest)
        if self.baseline not in cand:
            cand.append(self.baseline)
        return cand

    def save(self, out_dir: str) -> None:
        os.makedirs(out_dir, exist_ok=True)
        manifest = []
        for t, b, prior in zip(self.tiles, self.banks, self.priors):
            name = f"bank_{tile_label(t)}.sieve"
            b.save(os.path.join(out_dir, name))
            entry = {"tile": tile_label(t), "bank": name}
            if prior is not None:
                entry["prior"] = prior.to_dict()
            manifest.append(entry)
        with open(os.path.join(out_dir, "tilebank.json"), "w") as fh:
            json.dump({"format": "skpp-tilebank-1", "tiles": manifest}, fh, indent=1)

    @classmethod
    def load(cls, out_dir: str) -> "TileBank":
        with open(os.path.join(out_dir, "tilebank.json")) as fh:
            man = json.load(fh)
        tiles = [parse_tile(e["tile"]) for e in man["tiles"]]
        banks = [SieveBank.load(os.path.join(out_dir, e["bank"])) for e in man["tiles"]]
        tb = cls(tiles, banks)
        tb.priors = [Calibration.from_dict(e["prior"]) if "prior" in e else None for e in man["tiles"]]
        return tb


def snap_pow2(size: ProblemSize) -> ProblemSize:
    """Nearest power of two per dimension (in log space)."""
    def snap(v: int) -> int:
        return 1 << max(0, round(math.log2(v)))

    return ProblemSize(snap(size.m), snap(size.n), snap(size.k))


def snap_corners(size: ProblemSize) -> list[ProblemSize]:
    """The power-of-two sizes enclosing ``size`` (floor / ceil per dimension, deduplicated)."""
    def both(v: int) -> list[int]:
        lo = 1 << max(0, int(math.floor(math.log2(v))))
        return [lo] if lo == v else [lo, lo * 2]

    return [ProblemSize(m, n, k) for m in both(size.m) for n in both(size.n) for k in both(size.k)]


def build_tile_bank(records: list[JointRecord], tiles: list[TileShape], **bank_kwargs) -> TileBank:
    """Insert every size's joint winner, in (m, n, k) order (bytes independent of sweep order)."""
    tb = TileBank(tiles, **bank_kwargs)
    for rec in sorted(records, key=lambda r: (r.size.m, r.size.n, r.size.k)):
        tb.insert(rec.size, rec.winner)
    return tb


def evaluate_selection(bank: TileBank, records: list[JointRecord], tolerance: float = 0.2,
                       nearest=False) -> dict:
    """Selected = fastest measured candidate of bank.candidates(size); compare to the measured oracle.

    ``records`` may come from a different measurement run than the one the bank
    was built from (held-out validation) or hold sizes the bank never saw.
    """
    n_all = sum(len(rec.costs) for _, rec in records[0].per_tile) if records else 0
    within = 0
    ratios = []
    evaluated = 0
    vs_dp = []
    for rec in records:
        cand = bank.candidates(rec.size, nearest)
        evaluated += len(cand) - 1
        times = [(rec.time_of(c), i) for i, c in enumerate(cand)]
        chosen_us = min(times)[0]
        ratio = chosen_us / rec.winner_us if rec.winner_us > 0 else 1.0
        ratios.append(ratio)
        within += ratio <= 1.0 + tolerance
        vs_dp.append(rec.time_of(bank.baseline) / chosen_us)
    possible = len(records) * max(n_all - 1, 1)
    ratios.sort()
    return {
        "sizes": len(records),
        "candidates_per_size_all": n_all,
        "tolerance": tolerance,
        "fraction_within": within / len(records) if records else 1.0,
        "median_slowdown_vs_oracle": ratios[len(ratios) // 2] if ratios else 1.0,
        "p95_slowdown_vs_oracle": ratios[int(0.95 * (len(ratios) - 1))] if ratios else 1.0,
        "max_slowdown_vs_oracle": ratios[-1] if ratios else 1.0,
        "eliminated_fraction": 1.0 - evaluated / possible if possible else 1.0,
        "geomean_speedup_vs_baseline_dp": math.exp(sum(math.log(v) for v in vs_dp) / len(vs_dp)) if vs_dp else 1.0,
    }


class Selector:
    """Stream-K++ selection at run time: Bloom-pruned candidates, measured once per size.

    ``config(size)`` returns the (tile, policy) to run: the candidates of
    ``bank.candidates(size, nearest)`` (the filters' answer plus the baseline; a size the
    filters never saw takes the union over its enclosing power-of-two sizes and the
    calibrated cost model's pick, when the bank carries priors); a single
    candidate is used directly, several are timed once on the device with ``timer`` and the
    fastest is cached for the size — the paper's "evaluate only the policies the filters
    did not eliminate", lifted to (tile, policy).  ``gemm`` runs C = A @ B
    with the selected configuration.
    """

    def __init__(self, bank: TileBank, nearest="corners+model", timer=None):
        self.bank = bank
        self.nearest = nearest
        self.timer = timer  # timer(size, [(tile, policy), ...], a, b, out) -> [us, ...]
        self.cache: dict = {}
        self.measured = 0   # sizes that needed a measurement (more than one candidate)

    def config(self, size: ProblemSize, a=None, b=None, out=None) -> Config:
        key = (size.m, size.n, size.k, getattr(a, "dtype", None), getattr(out, "dtype", None))
        cfg = self.cache.get(key)
        if cfg is not None:
            return cfg
        cand = self.bank.candidates(size, self.nearest)
        if len(cand) == 1:
            cfg = cand[0]
        else:
            times = (self.timer or _device_timer)(size, cand, a, b, out)
            self.measured += 1
            cfg = min(zip(times, range(len(cand)), cand))[2]
        self.cache[key] = cfg
        return cfg

    def gemm(self, a, b, out=None, out_dtype=None):
        import torch

        from .executor import GemmPlan

        if out is None:
            out = torch.empty((a.shape[0], b.shape[1]), dtype=out_dtype or torch.float32, device=a.device)
        size = ProblemSize(a.shape[0], b.shape[1], a.shape[1])
        tile, policy = self.config(size, a, b, out)
        return GemmPlan(a, b, out, policy, tile).launch()


def _device_timer(size, cand, a, b, out):
    """Median device time (us) of each candidate on the caller's operands (graph replays)."""
    import torch

    from .executor import GemmPlan
    from .sweep import MeasureParams, time_plan

    if a is None or b is None:
        raise ValueError("measuring candidates needs the operands")
    if out is None:
        out = torch.empty((size.m, size.n), dtype=torch.float32, device=a.device)
    params = MeasureParams(warmup=2, reps=5, max_inner=16, target_us=100.0)
    return [time_plan(GemmPlan(a, b, out, pol, tile), params) for tile, pol in cand]


def joint_records_from_csvs(paths_by_tile: list[tuple[TileShape, str]]) -> list[JointRecord]:
    """Rebuild joint records from per-tile records CSVs (reference schema)."""
    from .pipeline import read_records_csv, records_from_rows

    per_size: dict[ProblemSize, list] = {}
    for tile, path in paths_by_tile:
        for rec in records_from_rows(read_records_csv(path)):
            per_size.setdefault(rec.size, []).append((tile, rec))
    tiles = [t for t, _ in paths_by_tile]
    out = []
    for size, lst in per_size.items():
        lst.sort(key=lambda tr: tiles.index(tr[0]))
        out.append(joint_winner(size, lst))
    out.sort(key=lambda r: (r.size.m, r.size.n, r.size.k))
    return out


__all__ = [
    "BANK_DIR", "JointRecord", "Selector", "TileBank", "build_tile_bank", "default_bank_dir", "evaluate_selection", "joint_records_from_csvs",
    "joint_winner", "parse_tile", "snap_corners", "snap_pow2", "tile_label", "CostEstimate", "TuneRecord", "rank_costs",
]
