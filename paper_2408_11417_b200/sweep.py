"""GPU autotuning sweep: measure every (size, policy) schedule on the B200.

Replaces the analytic ``tune_grid`` loop of the reference
(pipeline.py:102-114 -> costmodel.py:141-164 ``pick_winner``): each
(size, policy) is timed on the device instead of costed by a formula.

* Policies whose closed forms coincide (same data-parallel/Stream-K split and
  order — e.g. every hybrid equals all-Stream-K when the grid has fewer tiles
  than SMs) execute identical work; each distinct schedule is measured once
  and its time is credited to all policies that share it, so the ranking's
  ordinal tie-break picks the lowest one (costmodel.py:158).
* One measurement = ``warmup`` launches, then ``reps`` CUDA-graph replays of
  ``inner`` back-to-back launches timed with CUDA events on the launching
  stream; the cost is the median per-launch time (paper protocol: warm-up +
  mean of repeated launches).
* Operands live in preallocated device buffers sized for the largest problem
  of the sweep; problem views are carved from them, so the sweep allocates
  nothing per size.
* Multi-GPU: :func:`lpt_partition` splits the sizes over ranks by estimated
  cost (longest processing time first); ranks share nothing on the data path
  and their records are merged on the host — bank bytes do not depend on the
  partition because ``build_bank`` inserts in lexicographic order.
"""

from __future__ import annotations

import dataclasses
import heapq
import math
import time
from dataclasses import dataclass

import torch

from .costmodel import CostEstimate, TuneRecord, rank_costs
from .executor import GemmPlan, default_g
from .scheduler import count_partials, schedule_signature
from .types import Policy, ProblemSize, TileShape, canonical_policies

DENSE_BF16_PEAK_TFLOPS = 2250.0  # nominal dense bf16/fp16 (148 SM x 8192 FLOP/clk x ~1.86 GHz)


@dataclass(frozen=True)
class MeasureParams:
    warmup: int = 3
    reps: int = 10
    target_us: float = 200.0   # aim for graph replays of roughly this length
    max_inner: int = 64
    in_dtype: torch.dtype = torch.bfloat16
    out_dtype: torch.dtype = torch.float32
    peak_tflops: float = DENSE_BF16_PEAK_TFLOPS
    use_graphs: bool = True
    timed_us: float = 20000.0  # timed work per schedule for big problems (>= 3 samples)
    # Cold L2: sizes whose operand set (A, B, C) is at least cold_min_bytes and fits in the
    # L2 are timed rotating over enough distinct operand sets (> 4 x L2 in total, at most
    # cold_max_sets) that every launch reads its operands from HBM, as in production and in
    # bench.py's timed region; sets up to 2.5 x L2 rotate over two (cold_sets).  Warm timing picked a different winner for 16 of 628 such
    # sizes, 4 of them > 20% slower cold (profiles/round2/cold_l2_check.json).
    cold: bool = False
    cold_min_bytes: int = 4 << 20
    cold_max_sets: int = 64


class OperandPool:
    """Device buffers large enough for every problem of a sweep."""

    def __init__(self, sizes: list[ProblemSize], in_dtype=torch.bfloat16, out_dtype=torch.float32,
                 device: int | None = None, seed: int = 0):
        dev = torch.cuda.current_device() if device is None else device
        max_a = max(s.m * _pad8(s.k) for s in sizes)
        max_b = max(_pad8(s.k) * _pad8(s.n) for s in sizes)
        max_c = max(s.m * _pad8(s.n) for s in sizes)
        gen = torch.Generator(device=f"cuda:{dev}")
        gen.manual_seed(seed)
        self.a = torch.randn(max_a, generator=gen, device=f"cuda:{dev}", dtype=torch.float32).to(in_dtype)
        self.b = torch.randn(max_b, generator=gen, device=f"cuda:{dev}", dtype=torch.float32).to(in_dtype)
        self.c = torch.empty(max_c, device=f"cuda:{dev}", dtype=out_dtype)

    def views(self, size: ProblemSize):
        kp, np_ = _pad8(size.k), _pad8(size.n)
        a = self.a[: size.m * kp].view(size.m, kp)[:, : size.k]
        b = self.b[: kp * np_].view(kp, np_)[: size.k, : size.n]
        c = self.c[: size.m * np_].view(size.m, np_)[:, : size.n]
        return a, b, c


def _pad8(v: int) -> int:
    return (v + 7) // 8 * 8


_SIDE_STREAMS: dict = {}


def _side_stream(device: int) -> torch.cuda.Stream:
    """One capture stream per device, reused by every measurement (creating a stream per
    measurement was a visible share of a sweep's host time)."""
    st = _SIDE_STREAMS.get(device)
    if st is None:
        st = _SIDE_STREAMS[device] = torch.cuda.Stream(device=device)
    return st


L2_BYTES = 126 * 1024 * 1024


def cold_sets(size: ProblemSize, params: MeasureParams) -> int:
    """Operand sets a cold measurement of ``size`` rotates over (0 = time it warm).

    Sets that fit in the L2 rotate over enough copies to exceed 4x the L2.  Sets up to 2.5x
    the L2 rotate over two: a single repeated set that size still keeps much of B resident
    across launches (B of an N = 14336, K = 4096 projection alone is 117 MB), which hid the
    banded tile order's benefit and picked row-major tiles 20-30% slower cold for
    1024-2048 x 14336 x 4096 (`tools/llama_bench_table.py --oracle`).  Larger sets stream
    from HBM on their own."""
    b = 2 * (size.m * _pad8(size.k) + _pad8(size.k) * _pad8(size.n)) + 4 * size.m * _pad8(size.n)
    if not params.cold or b < params.cold_min_bytes:
        return 0
    if b > L2_BYTES:
        return 2 if 2 * b <= 5 * L2_BYTES else 0
    return int(min(params.cold_max_sets, max(2, math.ceil(4 * L2_BYTES / b))))


class ColdPool:
    """Raw device memory carved into rotating operand sets for cold-L2 timing."""

    def __init__(self, params: MeasureParams, device: int | None = None, seed: int = 0):
        dev = torch.cuda.current_device() if device is None else device
        # n sets of b bytes with n = ceil(4 L2 / b) <= 5 for b <= L2 (and n * b <= 64 x b for small b)
        self.nbytes = 5 * L2_BYTES + (64 << 20)
        gen = torch.Generator(device=f"cuda:{dev}")
        gen.manual_seed(seed)
        self.raw = torch.randn(self.nbytes // 2, generator=gen, device=f"cuda:{dev}").to(params.in_dtype)
        self.out_dtype = params.out_dtype

    def sets(self, size: ProblemSize, n: int):
        kp, np_ = _pad8(size.k), _pad8(size.n)
        ea, eb = size.m * kp, kp * np_
        ec = size.m * np_ * (4 if self.out_dtype == torch.float32 else 2) // 2  # in 16-bit elements
        step = (ea + eb + ec + 63) // 64 * 64
        if n * step > self.raw.numel():
            raise ValueError("cold pool too small")
        out = []
        for r in range(n):
            base = self.raw[r * step:(r + 1) * step]
            a = base[:ea].view(size.m, kp)[:, : size.k]
            b = base[ea:ea + eb].view(kp, np_)[: size.k, : size.n]
            c = base[ea + eb:ea + eb + ec].view(torch.uint8).view(self.out_dtype).view(size.m, np_)[:, : size.n]
            out.append((a, b, c))
        return out


def time_plan(plan, params: MeasureParams, est_us: float | None = None) -> float:
    """Median per-launch device time (microseconds) of a prepared GEMM, or of a rotation of
    prepared GEMMs over distinct operand sets (a list of plans: cold L2)."""
    if isinstance(plan, (list, tuple)):
        return _time_rotation(list(plan), params)
    stream = torch.cuda.current_stream()
    if params.warmup:
        plan.launch()
    if est_us is None:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        plan.launch()
        t1.record(stream)
        t1.synchronize()
        est_us = max(t0.elapsed_time(t1) * 1e3, 1.0)
    # the remaining warm-up launches only matter for short kernels: a launch of
    # >= 0.5 ms is its own warm-up (caches and clocks settle within it)
    if est_us < 500.0:
        for _ in range(params.warmup - 1):
            plan.launch()
    inner = int(max(1, min(params.max_inner, params.target_us // est_us)))
    # big problems: fewer replays (keep ~timed_us of timed work per schedule, >= 3 samples)
    reps = int(min(params.reps, max(3, math.ceil(params.timed_us / (inner * est_us)))))
    if params.use_graphs:
        # Raw capture: torch.cuda.graph() would synchronise, gc.collect() and empty_cache()
        # before every capture — ~5 ms per measurement, the largest host cost of a
        # multi-tile sweep.  The plan's own fixup workspace (captured launches never use
        # the shared per-stream one) is created here, outside the capture, so the graph
        # holds no allocation or memset.
        dev = stream.device_index
        graph = torch.cuda.CUDAGraph()
        side = _side_stream(dev)
        plan.prepare_for_capture(side)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            graph.capture_begin()
            try:
                for _ in range(inner):
                    plan.launch()
            finally:
                graph.capture_end()
        stream.wait_stream(side)
        run = graph.replay
        if inner > 1 or est_us < 500.0:
            graph.replay()  # first replay of a fresh graph carries upload cost
    else:
        def run():
            for _ in range(inner):
                plan.launch()
    # all replays queued back to back, one event pair each, a single sync at the end
    events = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        events.append((e0, e1))
    events[-1][1].synchronize()
    times = [e0.elapsed_time(e1) * 1e3 / inner for e0, e1 in events]
    times.sort()
    return times[len(times) // 2]


def _time_rotation(plans: list, params: MeasureParams) -> float:
    """Cold timing: one graph launches every plan of the rotation once (each on its own
    operand set, all on one shared workspace); median per-launch time over replays."""
    stream = torch.cuda.current_stream()
    side = _side_stream(stream.device_index)
    plans[0].prepare_for_capture(side)
    for p in plans[1:]:
        p.share_workspace_of(plans[0])
    side.wait_stream(stream)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        for p in plans[: params.warmup]:
            p.launch()
        graph.capture_begin()
        try:
            for p in plans:
                p.launch()
        finally:
            graph.capture_end()
    stream.wait_stream(side)
    graph.replay()
    events = []
    for _ in range(max(3, min(params.reps, 5))):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        graph.replay()
        e1.record(stream)
        events.append((e0, e1))
    events[-1][1].synchronize()
    times = sorted(e0.elapsed_time(e1) * 1e3 / len(plans) for e0, e1 in events)
    return times[len(times) // 2]


def measure_size(
    size: ProblemSize,
    tile: TileShape,
    g: int,
    policies: list[Policy],
    params: MeasureParams,
    pool: OperandPool,
    cold_pool: "ColdPool | None" = None,
) -> TuneRecord:
    """Time every policy's schedule for one size (identical schedules measured once).

    With ``params.cold`` (and a ``cold_pool``), sizes whose operands fit in the L2 are timed
    cold: each schedule rotates over :func:`cold_sets` distinct operand sets.

    Heavy sizes (a first launch >= ``HEAVY_US``) run at the power cap, where the clock
    needs tens of milliseconds to settle after the load changes: measured in one pass,
    the first few schedules of such a size came out up to 1.6x slower than the same
    schedules measured later (8192x14336x4096: DP 1231 us vs 763 us for hybrid5, which
    interleaved re-measurement puts within a few %).  They are therefore preceded by a
    ~20 ms soak of the first schedule (skipped when another heavy size was measured just
    before) and measured in two passes of half the timed work (forward, then reverse
    order), keeping each schedule's faster pass.
    """
    a, b, c = pool.views(size)
    plans: dict[tuple, GemmPlan] = {}
    sig_of = []
    for pol in policies:
        plan = GemmPlan(a, b, c, pol, tile, g)
        sig = schedule_signature(plan.sched_c)
        plans.setdefault(sig, plan)
        sig_of.append((pol, sig))
    order = list(plans)
    n_cold = cold_sets(size, params) if cold_pool is not None else 0
    first = plans[order[0]]
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    first.launch()
    t0.record(stream)
    first.launch()
    t1.record(stream)
    t1.synchronize()
    first_us = t0.elapsed_time(t1) * 1e3
    times: dict[tuple, float] = {}
    global _last_heavy_end
    if n_cold:
        sets = cold_pool.sets(size, n_cold)
        rot = {sig: [GemmPlan(sa, sb, sc, plans[sig].policy, tile, g) for sa, sb, sc in sets] for sig in order}
        if first_us >= HEAVY_US:  # power-capped: soak, then two passes in opposite orders (below)
            if time.perf_counter() - _last_heavy_end > SOAK_GAP_S:
                for i in range(int(math.ceil(SOAK_US / first_us))):
                    rot[order[0]][i % n_cold].launch()
            for rnd in range(2):
                for sig in (order if rnd == 0 else order[::-1]):
                    us = _time_rotation(rot[sig], params)
                    times[sig] = min(us, times.get(sig, us))
            _last_heavy_end = time.perf_counter()
        else:
            times = {sig: _time_rotation(rot[sig], params) for sig in order}
        return _record(size, params, plans, sig_of, times)
    if first_us >= HEAVY_US:
        # the soak only matters on a light -> heavy transition: right after another heavy
        # size the clock already sits at its power-capped steady state
        if time.perf_counter() - _last_heavy_end > SOAK_GAP_S:
            for _ in range(int(math.ceil(SOAK_US / first_us))):
                first.launch()
        half = dataclasses.replace(params, timed_us=params.timed_us / 2)  # same total timed work
        for rnd in range(2):
            for sig in (order if rnd == 0 else order[::-1]):
                us = time_plan(plans[sig], half)
                times[sig] = min(us, times.get(sig, us))
        _last_heavy_end = time.perf_counter()
    else:
        for sig in order:
            times[sig] = time_plan(plans[sig], params, first_us if sig == order[0] else None)
    return _record(size, params, plans, sig_of, times)


def _record(size, params, plans, sig_of, times) -> TuneRecord:
    by_sig: dict[tuple, CostEstimate] = {}
    costs = []
    for pol, sig in sig_of:
        est = by_sig.get(sig)
        if est is None:
            us = times[sig]
            tflops = size.flops / (us * 1e-6) / 1e12
            partial, full, _ = count_partials(plans[sig].sched_c)
            est = CostEstimate(makespan=us, utilization=tflops / params.peak_tflops,
                               atomic_writes=partial, full_stores=full)
            by_sig[sig] = est
        costs.append((pol, est))
    return rank_costs(size, costs)


HEAVY_US = 200.0   # sizes whose schedules run at the power cap (see measure_size)
SOAK_US = 20000.0
SOAK_GAP_S = 0.05  # a heavy size measured less than this ago leaves the clock settled
_last_heavy_end = 0.0


def measure_size_tiles(
    size: ProblemSize,
    tiles: list[TileShape],
    policies: list[Policy],
    params: MeasureParams,
    pool: OperandPool,
    rounds: int = 5,
) -> list[tuple[TileShape, TuneRecord]]:
    """Time every (tile, policy) of one size with the distinct schedules measured
    round-robin (``rounds`` passes, rotated start, median per schedule), so clock
    drift under the power cap during the measurement does not favour whichever
    tile happened to run first."""
    a, b, c = pool.views(size)
    keys: dict[tuple, GemmPlan] = {}
    cfg_key = []
    for ti, tile in enumerate(tiles):
        g = default_g(tile)
        for pol in policies:
            plan = GemmPlan(a, b, c, pol, tile, g)
            key = (ti, schedule_signature(plan.sched_c))
            keys.setdefault(key, plan)
            cfg_key.append((ti, pol, key))
    order = list(keys)
    samples: dict[tuple, list[float]] = {k: [] for k in order}
    for r in range(rounds):
        for i in range(len(order)):
            key = order[(i + r) % len(order)]
            samples[key].append(time_plan(keys[key], params))
    out = []
    for ti, tile in enumerate(tiles):
        costs = []
        for tj, pol, key in cfg_key:
            if tj != ti:
                continue
            us = sorted(samples[key])[len(samples[key]) // 2]
            tflops = size.flops / (us * 1e-6) / 1e12
            partial, full, _ = count_partials(keys[key].sched_c)
            costs.append((pol, CostEstimate(makespan=us, utilization=tflops / params.peak_tflops,
                                            atomic_writes=partial, full_stores=full)))
        out.append((tile, rank_costs(size, costs)))
    return out


def tune_sizes(
    sizes: list[ProblemSize],
    tile: TileShape,
    g: int | None = None,
    policies: list[Policy] | None = None,
    params: MeasureParams | None = None,
    pool: OperandPool | None = None,
    progress=None,
    seconds: dict | None = None,
) -> list[TuneRecord]:
    """Measured records for ``sizes`` on the current device, in input order.  With
    ``seconds``, each size's measurement wall time is added to ``seconds[size]``
    (the cost table a later sweep can partition by)."""
    if policies is None:
        policies = canonical_policies()
    if params is None:
        params = MeasureParams()
    if g is None:
        g = default_g(tile)
    if pool is None:
        pool = OperandPool(sizes, params.in_dtype, params.out_dtype)
    cold_pool = None
    if params.cold and any(cold_sets(z, params) for z in sizes):
        cold_pool = _cold_pool(params)
    out = []
    for i, size in enumerate(sizes):
        t0 = time.perf_counter() if seconds is not None else 0.0
        out.append(measure_size(size, tile, g, policies, params, pool, cold_pool))
        if seconds is not None:
            seconds[size] = seconds.get(size, 0.0) + time.perf_counter() - t0
        if progress is not None:
            progress(i + 1, len(sizes))
    return out


_COLD_POOLS: dict = {}


def _cold_pool(params: MeasureParams) -> ColdPool:
    """One cold pool per (device, dtypes), reused by every tile of a sweep."""
    key = (torch.cuda.current_device(), params.in_dtype, params.out_dtype, params.cold_max_sets)
    if key not in _COLD_POOLS:
        _COLD_POOLS[key] = ColdPool(params)
    return _COLD_POOLS[key]


def estimated_cost_s(size: ProblemSize, n_policies: int = 7, peak_tflops: float = 1000.0,
                     launch_us: float = 8.0, fixed_s: float = 2.5e-3, sms: int = 148,
                     tile_mn: int = 128) -> float:
    """Wall time of measuring one size with :func:`measure_size` (for LPT partitioning).

    Models what a measurement does: per distinct schedule a fixed host cost
    (plan, graph capture/instantiate) plus warm-up, one estimate launch and
    ``reps`` graph replays of ``inner`` launches, with the same adaptive
    inner/reps rules as :func:`time_plan`.  Small grids (fewer tiles than SMs)
    have only two distinct schedules (every Stream-K policy is all-Stream-K).
    """
    t_us = size.flops / (peak_tflops * 1e6) + launch_us
    inner = max(1, min(64, int(200.0 // t_us)))
    reps = min(10, max(3, math.ceil(20000.0 / (inner * t_us))))
    tiles = -(-size.m // tile_mn) * -(-size.n // tile_mn)
    distinct = 2 if tiles <= sms else n_policies
    return distinct * (fixed_s + (4 + inner * (1 + reps)) * t_us * 1e-6)


def save_cost_table(path: str, seconds: dict) -> None:
    """Per-size measurement wall times of a sweep ({"m,n,k": s}), for :func:`measured_cost`."""
    import json

    with open(path, "w") as fh:
        json.dump({f"{z.m},{z.n},{z.k}": round(v, 6) for z, v in sorted(
            seconds.items(), key=lambda kv: (kv[0].m, kv[0].n, kv[0].k))}, fh)


def load_cost_table(paths) -> dict:
    import json

    table = {}
    for path in paths:
        with open(path) as fh:
            for key, v in json.load(fh).items():
                m, n, k = (int(x) for x in key.split(","))
                table[ProblemSize(m, n, k)] = float(v)
    return table


def measured_cost(table: dict, fallback=estimated_cost_s):
    """LPT cost = a previous sweep's measured wall time for the size (the best predictor of
    the next one), scaled to the analytic model's units for sizes it did not see."""
    known = [z for z in table if table[z] > 0]
    scale = (sum(table[z] for z in known) / sum(fallback(z) for z in known)) if known else 1.0

    def cost(size: ProblemSize) -> float:
        v = table.get(size)
        return v if v is not None and v > 0 else scale * fallback(size)

    return cost


def lpt_partition(sizes: list[ProblemSize], world: int, cost=estimated_cost_s) -> list[list[ProblemSize]]:
    """Longest-processing-time-first assignment of sizes to `world` ranks."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0.0, r) for r in range(world)]
    parts: list[list[ProblemSize]] = [[] for _ in range(world)]
    for size in sorted(sizes, key=lambda s: (-cost(s), s.m, s.n, s.k)):
        load, r = heapq.heappop(heap)
        parts[r].append(size)
        heapq.heappush(heap, (load + cost(size), r))
    return parts


def sweep_throughput(n_sizes: int, n_policies: int, seconds: float) -> float:
    """(size, policy) evaluations per second."""
    return n_sizes * n_policies / seconds if seconds > 0 else math.inf


class Stopwatch:
    def __enter__(self):
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        self.seconds = time.perf_counter() - self.t0


# -- sharded sweep driver ---------------------------------------------------------


def shard_path(out_dir, rank: int) -> str:
    import os

    return os.path.join(out_dir, f"records.rank{rank}.csv")


def run_shard(sizes: list[ProblemSize], rank: int, world: int, measure, out_dir=None,
              cost=estimated_cost_s) -> list[TuneRecord]:
    """Measure this rank's LPT share of ``sizes`` with ``measure(sizes) -> records``.

    Ranks exchange nothing on the data path: each writes its records CSV
    shard (reference schema) and the host merges the shards afterwards.
    """
    from .pipeline import write_records_csv

    mine = lpt_partition(sizes, world, cost)[rank]
    mine.sort(key=lambda s: (s.m, s.n, s.k))
    records = measure(mine) if mine else []
    if out_dir is not None:
        if records:
            write_records_csv(shard_path(out_dir, rank), records)
        else:
            open(shard_path(out_dir, rank), "w").close()
    return records


def merge_shards(out_dir, world: int) -> list[TuneRecord]:
    """Concatenate every rank's shard back into records in (m, n, k) order."""
    import os

    from .pipeline import read_records_csv, records_from_rows

    rows = []
    for r in range(world):
        path = shard_path(out_dir, r)
        if os.path.getsize(path) == 0:
            continue
        rows.extend(read_records_csv(path))
    recs = records_from_rows(rows)
    recs.sort(key=lambda rec: (rec.size.m, rec.size.n, rec.size.k))
    return recs


def gpu_measure(tile: TileShape, policies: list[Policy] | None = None, params: MeasureParams | None = None):
    """measure(sizes) on the current GPU (one OperandPool for the whole shard)."""

    def measure(sizes):
        return tune_sizes(sizes, tile, None, policies, params)

    return measure


def run_shard_tiles(sizes: list[ProblemSize], rank: int, world: int, tiles: list[TileShape],
                    params: MeasureParams, out_dir: str, tag: str = "records", cost=estimated_cost_s) -> None:
    """Measure this rank's LPT share of ``sizes`` under every tile; one CSV shard per tile,
    plus ``costs.<tag>.rank<r>.json`` (per-size measurement seconds, summed over tiles)."""
    import os

    from .pipeline import write_records_csv
    from .tiles import tile_label

    mine = lpt_partition(sizes, world, cost)[rank]
    mine.sort(key=lambda s: (s.m, s.n, s.k))
    pool = OperandPool(mine, params.in_dtype, params.out_dtype) if mine else None
    seconds: dict = {}
    for tile in tiles:
        path = os.path.join(out_dir, f"{tag}.{tile_label(tile)}.rank{rank}.csv")
        if mine:
            write_records_csv(path, tune_sizes(mine, tile, None, None, params, pool, seconds=seconds))
        else:
            open(path, "w").close()
    save_cost_table(os.path.join(out_dir, f"costs.{tag}.rank{rank}.json"), seconds)


def merge_tiles(out_dir: str, world: int, tiles: list[TileShape], tag: str = "records"):
    """Per-tile merged CSVs (reference schema) and the joint (tile, policy) records."""
    import os

    from .pipeline import read_records_csv, write_records_csv, records_from_rows
    from .tiles import joint_records_from_csvs, tile_label

    paths = []
    for tile in tiles:
        rows = []
        for r in range(world):
            p = os.path.join(out_dir, f"{tag}.{tile_label(tile)}.rank{r}.csv")
            if os.path.getsize(p):
                rows.extend(read_records_csv(p))
        recs = records_from_rows(rows)
        recs.sort(key=lambda rec: (rec.size.m, rec.size.n, rec.size.k))
        merged = os.path.join(out_dir, f"{tag}.{tile_label(tile)}.csv")
        write_records_csv(merged, recs)
        paths.append((tile, merged))
    return joint_records_from_csvs(paths), paths


def heldout_sizes(n: int, seed: int = 7) -> list[ProblemSize]:
    """Off-grid sizes (not powers of two) for held-out selection checks."""
    import random

    rnd = random.Random(seed)
    out = set()
    while len(out) < n:
        m = int(2 ** rnd.uniform(0, 13))
        nn = int(2 ** rnd.uniform(6, 13))
        k = int(2 ** rnd.uniform(4, 15))
        if m & (m - 1) or nn & (nn - 1) or k & (k - 1):
            out.add(ProblemSize(m, nn, k))
    return sorted(out, key=lambda s: (s.m, s.n, s.k))


def main(argv=None) -> int:
    """Sweep CLI.  Single GPU:  python -m paper_2408_11417_b200.sweep --out DIR
    Multi GPU (one process per GPU):  torchrun --nproc-per-node N -m paper_2408_11417_b200.sweep --out DIR
    """
    import argparse
    import json
    import os

    from . import pipeline as pl
    from .sieve import elimination_stats
    from .tiles import build_tile_bank, evaluate_selection, parse_tile, tile_label

    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("--out", required=True)
    ap.add_argument("--grid", default="paper", help="paper | small | llama | paper+llama")
    ap.add_argument("--tiles", default="128x128x64", help="comma list; the first is the baseline tile")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--max-gflop", type=float, default=0.0, help="skip sizes above this (0 = no limit)")
    ap.add_argument("--cold", action="store_true",
                    help="time sizes whose operands fit in the L2 cold (rotating operand sets), as production "
                         "and bench.py see them")
    ap.add_argument("--validate", action="store_true", help="re-measure everything (held-out run)")
    ap.add_argument("--heldout", type=int, default=0, help="also measure N off-grid sizes")
    ap.add_argument("--cost-table", default="",
                    help="comma list of costs.*.json from an earlier sweep: LPT partitions by the measured "
                         "per-size times instead of the analytic estimate")
    ap.add_argument("--emulate-world", default="",
                    help="comma list of world sizes: run every rank's LPT share back to back on this GPU "
                         "and report max-over-ranks time per world size (single-GPU scaling estimate)")
    args = ap.parse_args(argv)
    if args.emulate_world:
        return emulate_worlds(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.makedirs(args.out, exist_ok=True)
    sizes = grid_sizes(args.grid)
    if args.max_gflop > 0:
        sizes = [s for s in sizes if s.flops <= args.max_gflop * 1e9]
    tiles = [parse_tile(t) for t in args.tiles.split(",")]
    params = MeasureParams(warmup=args.warmup, reps=args.reps, cold=args.cold)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")  # host rendezvous only: records travel as files

    def barrier():
        if dist is not None:
            dist.barrier()

    cost = measured_cost(load_cost_table(args.cost_table.split(","))) if args.cost_table else estimated_cost_s
    sw = Stopwatch()
    with sw:
        run_shard_tiles(sizes, rank, world, tiles, params, args.out, "records", cost)
    with open(os.path.join(args.out, f"timing.rank{rank}.json"), "w") as fh:
        json.dump({"rank": rank, "world": world, "seconds": sw.seconds, "tiles": len(tiles)}, fh)
    if args.validate:
        run_shard_tiles(sizes, rank, world, tiles, params, args.out, "validate")
    if args.heldout:
        run_shard_tiles(heldout_sizes(args.heldout), rank, world, tiles, params, args.out, "heldout")
    barrier()
    if rank == 0:
        joint, paths = merge_tiles(args.out, world, tiles, "records")
        tb = build_tile_bank(joint, tiles)
        # calibrated cost model per tile: the prior for sizes the filters never saw
        from .costmodel import calibrate

        for tile, path in paths:
            recs = pl.records_from_rows(pl.read_records_csv(path))
            tb.priors[tiles.index(tile)] = calibrate(
                ((r.size, [(p, e.makespan) for p, e in r.costs]) for r in recs), tile,
                default_g(tile))
        tb.save(os.path.join(args.out, "tilebank"))
        times = [json.load(open(os.path.join(args.out, f"timing.rank{r}.json")))["seconds"] for r in range(world)]
        n_pairs = len(sizes) * 7 * len(tiles)
        per_tile = {}
        for tile, path in paths:
            recs = pl.records_from_rows(pl.read_records_csv(path))
            bank = pl.build_bank(recs)
            el = elimination_stats(bank, recs)
            per_tile[tile_label(tile)] = {
                "winner_counts": pl.winner_counts(recs),
                "eliminated_fraction": el.eliminated_fraction,
                "false_negatives": el.false_negatives,
            }
        summary = {
            "sizes": len(sizes), "policies": 7, "tiles": [tile_label(t) for t in tiles], "world": world,
            "sweep_seconds_max_over_ranks": max(times),
            "shape_policy_per_s": n_pairs / max(times),
            "per_tile": per_tile,
            "joint_winner_tiles": {tile_label(t): sum(1 for r in joint if r.winner[0] == t) for t in tiles},
            "selection_in_sample": evaluate_selection(tb, joint),
        }
        if args.validate:
            joint2, _ = merge_tiles(args.out, world, tiles, "validate")
            summary["selection_heldout_run"] = evaluate_selection(tb, joint2)
        if args.heldout:
            jh, _ = merge_tiles(args.out, world, tiles, "heldout")
            summary["selection_offgrid_baseline_fallback"] = evaluate_selection(tb, jh, nearest=False)
            summary["selection_offgrid_nearest_pow2"] = evaluate_selection(tb, jh, nearest=True)
            summary["selection_offgrid_pow2_corners"] = evaluate_selection(tb, jh, nearest="corners")
            summary["selection_offgrid_corners_and_model"] = evaluate_selection(tb, jh, nearest="corners+model")
        summary["costmodel_priors"] = {tile_label(t): c.to_dict() for t, c in zip(tiles, tb.priors)}
        with open(os.path.join(args.out, "summary.json"), "w") as fh:
            json.dump(summary, fh, indent=1)
        print(json.dumps(summary))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def emulate_worlds(args) -> int:
    """Per-world-size sweep time when ranks run their LPT shares independently (no comms).

    Each rank's share is measured separately on this GPU (one process, back to
    back); a world of N GPUs would take max-over-ranks of those times, since
    the shares share nothing.  Results are labelled as emulated.
    """
    import json
    import os

    from .tiles import parse_tile, tile_label

    os.makedirs(args.out, exist_ok=True)
    sizes = grid_sizes(args.grid)
    if args.max_gflop > 0:
        sizes = [s for s in sizes if s.flops <= args.max_gflop * 1e9]
    tiles = [parse_tile(t) for t in args.tiles.split(",")]
    params = MeasureParams(warmup=args.warmup, reps=args.reps)
    pool = OperandPool(sizes, params.in_dtype, params.out_dtype)
    # warm the process (kernel setup, allocator) so rank 0 is not charged for it
    tune_sizes(sizes[:3], tiles[0], None, None, params, pool)
    out = {"mode": "emulated: each rank's share measured back to back on one GPU; "
                   "wall time of a world = max over its ranks", "sizes": len(sizes),
           "tiles": [tile_label(t) for t in tiles], "policies": 7}
    # World 1 measures every size once and records its wall time; larger worlds are then
    # partitioned both by the analytic estimate and by those measured times (what a re-tune
    # with a previous sweep's cost table does, --cost-table).
    table: dict = {}
    worlds = [int(w) for w in args.emulate_world.split(",")]
    if 1 not in worlds:
        worlds = [1] + worlds
    for label, key in (("analytic", "worlds_analytic_cost"), ("measured", "worlds")):
        out[key] = {}
        for world in worlds:
            if label == "measured" and world == 1:
                out[key]["1"] = out["worlds_analytic_cost"]["1"]
                continue
            cost = estimated_cost_s if label == "analytic" else measured_cost(table)
            parts = lpt_partition(sizes, world, cost)
            secs = []
            for part in parts:
                part = sorted(part, key=lambda s: (s.m, s.n, s.k))
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for tile in tiles:
                    tune_sizes(part, tile, None, None, params, pool,
                               seconds=table if (label == "analytic" and world == 1) else None)
                torch.cuda.synchronize()
                secs.append(time.perf_counter() - t0)
            pairs = len(sizes) * 7 * len(tiles)
            out[key][str(world)] = {
                "rank_seconds": [round(v, 3) for v in secs],
                "max_rank_seconds": round(max(secs), 3),
                "shape_policy_per_s": round(pairs / max(secs), 1),
                "load_imbalance": round(max(secs) / (sum(secs) / len(secs)), 3),
            }
            print(json.dumps({label: {world: out[key][str(world)]}}), flush=True)
    out["lpt_cost"] = {"worlds": "measured per-size times of the world-1 pass",
                       "worlds_analytic_cost": "estimated_cost_s (analytic)"}
    save_cost_table(os.path.join(args.out, "costs.emulate.json"), table)
    with open(os.path.join(args.out, "scaling_emulated.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    return 0


def grid_sizes(name: str) -> list[ProblemSize]:
    from . import pipeline as pl

    out: list[ProblemSize] = []
    for part in name.split("+"):
        if part == "paper":
            out += pl.gen_problem_grid(pl.DEFAULT_GRID)
        elif part == "small":
            out += pl.gen_problem_grid(pl.GridSpec(pl.AxisRange(1, 1024), pl.AxisRange(64, 1024),
                                                   pl.AxisRange(16, 4096)))
        elif part == "llama":
            out += pl.llama3_8b_sizes()
        else:
            raise ValueError(f"unknown grid {part!r}")
    return list(dict.fromkeys(out))


if __name__ == "__main__":  # pragma: no cover
    raise SystemExit(main())
