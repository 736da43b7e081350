"""Stream-K++ schedules: geometry, the closed form, materialised items, audit.

Drop-in for ``gemmsched.scheduler`` (reference ``scheduler.py``).  The B200
build represents a schedule by six scalars (``skpp_sched_make`` in the C ABI)
that both the host and every CTA of the GEMM kernel expand with the same
cursor (``csrc/skpp_sched.h``); :func:`build_schedule` materialises that
expansion as the reference's ``WorkItem`` tuples so the two can be compared
field for field, and :func:`validate_schedule` runs the reference's interval
sweep natively.

Reference map: ``WriteMode``/``Phase``/``WorkItem``/``Schedule`` 40-92,
``grid_info`` 119-128, ``grid_size`` 131-133, ``streamk_ranges`` 136-152,
``locate_iter`` 155-165, ``hybrid_sk_tiles`` 168-178, ``build_schedule``
226-254, ``validate_schedule`` 257-291.
"""

from __future__ import annotations

import ctypes

from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple

import numpy as np

from . import _lib
from .types import GridInfo, HardwareModel, Policy, PolicyKind, ProblemSize, TileShape

_U64_MAX = (1 << 64) - 1


class WriteMode(Enum):
    FULL_STORE = "full-store"
    ATOMIC_PARTIAL = "atomic-partial"


class Phase(Enum):
    STREAM_K = "streamk"
    DATA_PARALLEL = "data-parallel"


_MODES = (WriteMode.FULL_STORE, WriteMode.ATOMIC_PARTIAL)
_PHASES = (Phase.STREAM_K, Phase.DATA_PARALLEL)


@dataclass(frozen=True, slots=True)
class WorkItem:
    """k-iterations [local_iter_begin, local_iter_end) of tile ``tile_idx``."""

    tile_idx: int
    local_iter_begin: int
    local_iter_end: int
    write_mode: WriteMode
    phase: Phase

    def __post_init__(self) -> None:
        if self.tile_idx < 0:
            raise ValueError(f"tile_idx must be >= 0, got {self.tile_idx}")
        if not 0 <= self.local_iter_begin < self.local_iter_end:
            raise ValueError(
                f"empty or inverted iteration range "
                f"[{self.local_iter_begin}, {self.local_iter_end})"
            )

    @property
    def iterations(self) -> int:
        return self.local_iter_end - self.local_iter_begin


@dataclass(frozen=True)
class Schedule:
    """Ordered work items of every workgroup for one (problem, tile, g, policy)."""

    grid: GridInfo
    g: int
    policy: Policy
    assignments: tuple[tuple[WorkItem, ...], ...]

    def items(self):
        for wg in self.assignments:
            yield from wg


class IterLocation(NamedTuple):
    tile_idx: int
    tile_m: int
    tile_n: int
    local_iter: int


@dataclass(frozen=True, slots=True)
class CoverageReport:
    covered_once: bool
    duplicates: int
    gaps: int


def _cdiv(a: int, b: int) -> int:
    return (a + b - 1) // b


def grid_info(size: ProblemSize, tile: TileShape) -> GridInfo:
    mt = _cdiv(size.m, tile.blk_m)
    nt = _cdiv(size.n, tile.blk_n)
    ipt = _cdiv(size.k, tile.blk_k)
    tiles = mt * nt
    iters = tiles * ipt
    if iters > _U64_MAX:
        raise ValueError("problem too large: total iteration count exceeds 2^64-1")
    return GridInfo(mt, nt, ipt, tiles, iters)


def grid_size(hw: HardwareModel) -> int:
    return hw.cu_count * hw.occupancy


def streamk_ranges(total_iters: int, g: int) -> list[tuple[int, int]]:
    """g ordered half-open ranges of ceil(total/g) iterations; the tail may be empty."""
    if total_iters < 0:
        raise ValueError("total_iters must be >= 0")
    if g < 1:
        raise ValueError("g must be >= 1")
    ipw = _cdiv(total_iters, g)
    return [(min(x * ipw, total_iters), min(x * ipw + ipw, total_iters)) for x in range(g)]


def locate_iter(iteration: int, grid: GridInfo) -> IterLocation:
    if not 0 <= iteration < grid.total_iters:
        raise ValueError(f"iteration {iteration} out of range [0, {grid.total_iters})")
    tile, local = divmod(iteration, grid.iters_per_tile)
    tm, tn = divmod(tile, grid.n_tiles)
    return IterLocation(tile, tm, tn, local)


def hybrid_sk_tiles(total_tiles: int, g: int, sk_batches: int) -> int:
    """Tiles in a hybrid's Stream-K region: the last (partial) wave plus s-1 waves."""
    rem = total_tiles % g
    return min(total_tiles, (sk_batches - 1) * g + (rem or g))


# -- closed form through the C ABI ------------------------------------------


def policy_to_c(policy: Policy) -> _lib.PolicyC:
    kind = {
        PolicyKind.DATA_PARALLEL: _lib.DATA_PARALLEL,
        PolicyKind.HYBRID: _lib.HYBRID,
        PolicyKind.ALL_STREAM_K: _lib.ALL_STREAM_K,
    }[policy.kind]
    batches = min(policy.sk_batches, 0x7FFFFFFF)
    return _lib.PolicyC(kind, batches, 1 if policy.sk_first else 0)


def closed_form(size: ProblemSize, tile: TileShape, g: int, policy: Policy) -> _lib.SchedC:
    """The six-scalar schedule the kernel decodes (dp/sk split, ipt, ipw, order)."""
    if size.m > _U64_MAX or tile.blk_m > 0xFFFFFFFF or tile.blk_n > 0xFFFFFFFF or tile.blk_k > 0xFFFFFFFF:
        raise ValueError("tile dimensions must fit in 32 bits")
    if not 1 <= g <= 0xFFFFFFFF:
        raise ValueError("g must be in [1, 2^32)")
    out = _lib.SchedC()
    rc = _lib.lib.skpp_sched_make(
        _lib.Problem(size.m, size.n, size.k),
        _lib.tile_c(tile),
        g,
        policy_to_c(policy),
        out,
    )
    if rc != _lib.OK:
        raise ValueError(_lib.last_error())
    return out


def tile_coords(sched_c: _lib.SchedC, tile_order: int, tile: int) -> tuple[int, int]:
    """C tile (tile_m, tile_n) the GEMM kernel writes for tile index ``tile`` under
    ``tile_order`` (0 = the reference's ``locate_iter``, G > 0 = bands of G tile rows)."""
    tm, tn = ctypes.c_uint64(), ctypes.c_uint64()
    _lib.check(_lib.lib.skpp_tile_coords(sched_c, tile_order, tile, ctypes.byref(tm), ctypes.byref(tn)))
    return int(tm.value), int(tn.value)


def schedule_arrays(sched_c: _lib.SchedC) -> tuple[np.ndarray, np.ndarray]:
    """(items[n, 8] int64, offsets[g+1]) of the closed form, workgroup-major.

    Item columns: tile, kb, ke, write_mode (0 full / 1 partial), phase
    (0 Stream-K / 1 data-parallel), role (0 full / 1 owner / 2 peer), and the
    C tile (tile_m, tile_n) of the reference's row-major ``locate_iter``.
    """
    total = np.zeros(1, dtype=np.uint64)
    _lib.check(_lib.lib.skpp_sched_count(sched_c, total.ctypes.data_as(_lib._u64p), None))
    n = int(total[0])
    items = np.zeros((max(n, 1), _lib.TRACE_FIELDS), dtype=np.int64)
    offsets = np.zeros(sched_c.g + 1, dtype=np.uint64)
    _lib.check(
        _lib.lib.skpp_sched_items(
            sched_c, items.ctypes.data_as(_lib._i64p), n, offsets.ctypes.data_as(_lib._u64p)
        )
    )
    return items[:n], offsets


def build_schedule(
    size: ProblemSize, tile: TileShape, hw: HardwareModel, policy: Policy
) -> Schedule:
    """Materialise the closed-form schedule as per-workgroup ``WorkItem`` tuples."""
    grid = grid_info(size, tile)
    g = grid_size(hw)
    sched_c = closed_form(size, tile, g, policy)
    items, offsets = schedule_arrays(sched_c)
    rows = items[:, :5].tolist()
    made = [
        WorkItem(t, kb, ke, _MODES[wm], _PHASES[ph]) for t, kb, ke, wm, ph in rows
    ]
    bounds = offsets.tolist()
    assignments = tuple(tuple(made[bounds[x] : bounds[x + 1]]) for x in range(g))
    sched = Schedule(grid, g, policy, assignments)
    # Marks this object as the unmodified closed form, so the executor can skip
    # re-deriving it (Schedule is not slotted, mirroring the reference class).
    object.__setattr__(sched, "_skpp_closed_form", (size, tile, assignments))
    return sched


def validate_schedule(sched: Schedule) -> CoverageReport:
    """Exactly-once audit of any schedule by interval sweep (scheduler.py:257-291)."""
    ipt = sched.grid.iters_per_tile
    total = sched.grid.total_iters
    starts, ends = [], []
    for it in sched.items():
        base = it.tile_idx * ipt
        starts.append(base + it.local_iter_begin)
        ends.append(base + it.local_iter_end)
    if any(v > _U64_MAX for v in ends) or total > _U64_MAX:
        return _validate_python(starts, ends, total)
    s = np.array(starts, dtype=np.uint64)
    e = np.array(ends, dtype=np.uint64)
    dup = np.zeros(1, dtype=np.uint64)
    gaps = np.zeros(1, dtype=np.uint64)
    _lib.check(
        _lib.lib.skpp_validate_intervals(
            s.ctypes.data_as(_lib._u64p),
            e.ctypes.data_as(_lib._u64p),
            len(starts),
            total,
            dup.ctypes.data_as(_lib._u64p),
            gaps.ctypes.data_as(_lib._u64p),
        )
    )
    d, gp = int(dup[0]), int(gaps[0])
    return CoverageReport(d == 0 and gp == 0, d, gp)


def _validate_python(starts, ends, total) -> CoverageReport:
    # Only reachable with iteration indices beyond 2^64 (hand-built schedules).
    events = sorted([(s, 1) for s in starts] + [(e, -1) for e in ends])
    covered = dup = depth = prev = 0
    for pos, delta in events:
        span = pos - prev
        if span > 0 and depth > 0:
            inside = min(pos, total) - min(prev, total)
            covered += inside
            dup += (depth - 1) * inside + depth * (span - inside)
        prev = pos
        depth += delta
    gaps = total - covered
    return CoverageReport(dup == 0 and gaps == 0, dup, gaps)


def schedule_signature(sched_c: _lib.SchedC) -> tuple:
    """Identity of the executed schedule: policies with equal signatures run identical items."""
    order = sched_c.sk_first if (sched_c.dp_tiles and sched_c.sk_tiles) else 1
    return (sched_c.dp_tiles, sched_c.sk_tiles, order)


def count_partials(sched_c: _lib.SchedC) -> tuple[int, int, int]:
    """(atomic-partial items, full stores, non-owner partials) of a closed-form schedule."""
    items, _ = schedule_arrays(sched_c)
    partial = int((items[:, 3] == 1).sum())
    full = int(items.shape[0] - partial)
    peers = int((items[:, 5] == 2).sum())
    return partial, full, peers
