#!/usr/bin/env python
"""Stream-K++ on B200 — headline benchmark (one JSON line on rank 0).

Metric (BASELINE.json): "GEMM TFLOP/s vs dense TC peak; % shapes within 20%
of oracle policy".  Both halves are measured in this run:

  * GEMM TFLOP/s — default workload = BASELINE config 3 at its largest
    single-GPU shape: the Llama-3-8B MLP projection at 8192 tokens,
    bf16 8192 x 14336 x 4096 with fp32 output, under the (tile, policy) the
    Stream-K++ selection layer picks: the shipped tile bank's Bloom candidates
    (``paper_2408_11417_b200/banks/b200``, corners + calibrated prior for sizes it
    never saw) plus the data-parallel baseline, each timed once, fastest wins.
    Every (tile, canonical policy) of the candidate tiles is also measured so the
    line reports the selected configuration against the measured oracle.
    Timed region: K steps, one persistent-kernel launch per step, back to back on
    one stream between ONE pair of CUDA events (max over ranks); the steps rotate
    over R distinct operand sets whose total is > 4x the 126 MB L2 (cold L2).
  * % shapes within 20% — a bounded selection check of the paper grid
    (``--sweep-grid``, default the reference's 1,456-size DEFAULT_GRID, one tile,
    seven policies): pass 1 measures every (size, policy) on the GPU and builds
    the Bloom bank from the winners, pass 2 re-measures independently and the
    fraction of sizes whose Bloom-selected policy is within 20% of that pass's
    oracle is reported.  With N GPUs the sizes are LPT-partitioned across the
    ranks (no data-path collective; records are gathered on the host), so the
    ``sweep`` block carries shape x policy/s and distinct schedules/s at N.

Also reported: ``e2e`` (the same GEMM through the public
``execute_schedule`` with pinned host bf16 inputs, H2D + kernel + D2H every
step, wall clock), ``roofline`` for the GEMM kernel, ``cpu_baseline`` (the
oracle's float64 numpy port of the reference executor on this box's cores).

``--impl reference`` times the reference's CPU implementation of the path
(the oracle port of gemmsched's execute_schedule, float64 numpy/OpenBLAS,
all host cores) on the same workload under the configuration the shipped bank
selects host-side (no GPU involved); under torchrun only rank 0 runs it.
With N GPUs each rank runs the same GEMM (the GEMM runs on one GPU;
replicas only), so ``value`` is N x the per-replica throughput ("weak").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GEMM TFLOP/s vs dense TC peak; % shapes within 20% of oracle policy"
ROTATE_BYTES = 4 * 128 * 1024 * 1024  # operand sets rotated through per step: 4x the 126 MB L2
ISOLATED_STEPS = 50

WORKLOADS = {
    "cfg3": dict(m=8192, n=14336, k=4096, dtype="bf16",
                 desc="BASELINE cfg3 (largest single-GPU shape): Llama-3-8B MLP gate/up projection at 8192 "
                      "tokens, bf16 8192x14336x4096, fp32 out, Bloom-selected (tile, policy)"),
    "cfg2": dict(m=512, n=512, k=16384, dtype="bf16",
                 desc="BASELINE cfg2: skinny split-K-bound bf16 GEMM M=N=512 K=16384, fp32 out, "
                      "Bloom-selected (tile, policy) among the 7 canonical policies x candidate tiles"),
    "cfg1": dict(m=1024, n=1024, k=1024, dtype="fp16",
                 desc="BASELINE cfg1: fp16 GEMM 1024^3, fp32 out, Bloom-selected (tile, policy)"),
    "square8192": dict(m=8192, n=8192, k=8192, dtype="bf16",
                       desc="large square bf16 GEMM 8192^3, fp32 out (70%-of-peak target), Bloom-selected (tile, policy)"),
}
# Candidate tiles of the joint (tile, policy) selection, baseline (DP) tile first.
BENCH_TILES = ["128x128x64", "128x64x128", "128x128x128", "256x128x128", "256x256x64", "256x256x128",
               "128x128x128b16", "256x256x128b16"]
SWEEP_TILE = "128x128x128"

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                  "source": "fallback (B200_PROFILING.md)"}
REASON_FIELDS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


def load_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        return dict(FALLBACK_PEAKS)


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled while the timed region runs.

    NVML (pynvml) is polled every ``period_ms`` from a thread that stamps each sample when
    it is taken, so even a ~10 ms timed region gets several samples (an ``nvidia-smi -lms``
    pipe delivers its lines block-buffered, late and in bursts, and left short regions with
    none).  ``summary`` keeps the samples taken between ``mark_start()`` and ``mark_end()``.
    Falls back to ``nvidia-smi -lms`` when NVML is unavailable.
    """

    _NVML_REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                     "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int, period_ms: int = 2):
        self.gpu = gpu_index
        self.period = period_ms / 1e3
        self.samples: list[tuple[float, float, float, int]] = []  # (time, sm MHz, max MHz, reasons)
        self.t0 = self.t1 = None
        self.stop = False
        self.thread = None
        self.nvml = None

    def _poll(self):
        nv, h = self.nvml, self.handle
        try:  # ~3 ms per call on this driver (the clock and reason queries are ~0.2 ms): once
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001
            mx = float("nan")
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((time.time(), float(sm), mx, int(rs)))
            except Exception:  # noqa: BLE001 — a failed poll only loses a sample
                pass
            time.sleep(self.period)

    def _poll_smi(self):
        cmd = ["nvidia-smi", f"--id={self.gpu}", "--query-gpu=clocks.sm,clocks.max.sm," + ",".join(
            f"clocks_event_reasons.{r}" for r in REASON_FIELDS), "--format=csv,noheader,nounits"]
        while not self.stop:
            try:
                ln = subprocess.run(cmd, capture_output=True, text=True, timeout=5).stdout.strip()
                parts = [p.strip() for p in ln.split(",")]
                bits = sum(self._NVML_REASONS[r] for r, v in zip(REASON_FIELDS, parts[2:])
                           if v.lower().startswith("active"))
                self.samples.append((time.time(), float(parts[0]), float(parts[1]), bits))
            except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
                pass

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            target = self._poll
        except Exception:  # noqa: BLE001 — no NVML: poll nvidia-smi instead
            self.nvml = None
            target = self._poll_smi
        self.thread = threading.Thread(target=target, daemon=True)
        self.thread.start()
        time.sleep(0.05)
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        # a region shorter than the poller's period (or one during which the poller did not get
        # the GIL) may end before any sample was taken after it started: wait for one (<= 0.5 s)
        deadline = time.time() + 0.5
        while (self.t0 is not None and self.thread is not None and self.thread.is_alive()
               and not any(smp[0] >= self.t0 for smp in self.samples) and time.time() < deadline):
            time.sleep(0.002)
        self.stop = True
        if self.thread is not None:
            self.thread.join(timeout=10)
        if self.nvml is not None:
            try:
                self.nvml.nvmlShutdown()
            except Exception:  # noqa: BLE001
                pass

    def summary(self) -> dict:
        t0 = self.t0 if self.t0 is not None else 0.0
        t1 = self.t1 if self.t1 is not None else time.time()
        window = [smp for smp in self.samples if t0 <= smp[0] <= t1]
        if not window:  # region shorter than one poll: the first sample after it started
            window = [smp for smp in self.samples if smp[0] >= t0][:1]
        if not window:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = sorted(r for r, bit in self._NVML_REASONS.items() if any(smp[3] & bit for smp in window))
        return {"sm_mhz": statistics.median(smp[1] for smp in window), "sm_max_mhz": max(smp[2] for smp in window),
                "reasons": reasons, "samples": len(window),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def physical_gpu(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local_rank < len(ids) and ids[local_rank].strip().isdigit():
            return int(ids[local_rank])
    return local_rank


def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and n_gpus != world:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    return world, rank, local


def ncu_traffic(workload: str, tile_label: str, policy_label: str):
    """DRAM bytes per launch of the GEMM kernel from the committed ncu capture of this workload
    (profiles/ncu_bench_<workload>.json, made by tools/gpurun_profile.sh), or None when the
    capture is of a different kernel configuration than the one this run selected."""
    path = os.path.join(ROOT, "profiles", f"ncu_bench_{workload}.json")
    from paper_2408_11417_b200.tiles import parse_tile

    t = parse_tile(tile_label)
    # template args <BN, BK, CG, RASTER>
    want = f"<{t.blk_n}, {t.blk_k}, {t.blk_m // 128}, {1 if getattr(t, 'band_rows', 0) else 0}>"
    try:
        with open(path) as fh:
            rows = json.load(fh)
        row = next(r for r in rows if "streamk_gemm" in r.get("kernel", "") and want in r["kernel"]
                   and r.get("policy", policy_label) == policy_label)
        return int(row["dram_traffic_bytes"]), os.path.relpath(path, ROOT)
    except (OSError, ValueError, KeyError, StopIteration):
        return None, None


def sweep_check(world: int, rank: int, grid: str, tile_label_: str) -> dict | None:
    """Bounded in-run selection check over the paper grid (the metric's second half).

    Pass 1 measures every (size, canonical policy) of this rank's LPT share on the GPU
    (identical schedules once), the records of all ranks are gathered on the host and the
    Bloom bank is built from the winners (``build_bank``: lexicographic insertion, so its
    bytes do not depend on the partition).  Pass 2 re-measures independently and reports
    the fraction of sizes whose Bloom-selected policy (fastest of ``query | {DP}`` by pass-2
    time) is within 20% of pass 2's oracle, plus eliminated fraction and false negatives.
    Sweep time per pass = CUDA events around the rank's whole share, max over ranks.
    """
    import hashlib

    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import pipeline as pl, sweep
    from paper_2408_11417_b200.scheduler import closed_form, schedule_signature
    from paper_2408_11417_b200.tiles import parse_tile

    if grid == "none":
        return None
    sizes = sweep.grid_sizes(grid)
    tile = parse_tile(tile_label_)
    g = sk.executor.default_g(tile)
    pols = sk.canonical_policies()
    params = sweep.MeasureParams(warmup=3, reps=10)
    mine = sorted(sweep.lpt_partition(sizes, world)[rank], key=lambda z: (z.m, z.n, z.k))
    pool = sweep.OperandPool(mine or sizes[:1], params.in_dtype, params.out_dtype, seed=rank)
    stream = torch.cuda.current_stream()

    def one_pass():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        recs = sweep.tune_sizes(mine, tile, g, pols, params, pool) if mine else []
        e1.record(stream)
        torch.cuda.synchronize()
        secs = e0.elapsed_time(e1) / 1e3
        if world > 1:
            gathered = [None] * world
            torch.distributed.all_gather_object(gathered, (secs, recs))
        else:
            gathered = [(secs, recs)]
        merged = [r for _, part in gathered for r in part]
        merged.sort(key=lambda r: (r.size.m, r.size.n, r.size.k))
        return merged, [sec for sec, _ in gathered]

    rec1, secs1 = one_pass()
    rec2, secs2 = one_pass()
    if rank != 0:
        return None
    bank = pl.build_bank(rec1)
    q = pl.selection_quality(rec2, bank, 0.20)
    el = sk.elimination_stats(bank, rec2)
    distinct = sum(len({schedule_signature(closed_form(z, tile, g, p)) for p in pols}) for z in sizes)
    t1 = max(secs1)
    return {
        "grid": grid, "sizes": len(sizes), "policies": len(pols), "tile": tile_label_, "g": g,
        "n_gpus": world, "partition": "LPT by estimated cost, sizes sharded, no data-path collective",
        "pct_within_20pct_of_oracle": round(100 * q["fraction_within"], 2),
        "median_slowdown_vs_oracle": round(q["median_slowdown"], 4),
        "max_slowdown_vs_oracle": round(q["max_slowdown"], 4),
        "eliminated_fraction": round(el.eliminated_fraction, 4),
        "false_negatives_vs_pass2_winners": el.false_negatives,
        "pass1_seconds_max_over_ranks": round(t1, 3),
        "pass2_seconds_max_over_ranks": round(max(secs2), 3),
        "rank_seconds_pass1": [round(v, 3) for v in secs1],
        "shape_policy_per_s": round(len(sizes) * len(pols) / t1, 1),
        "distinct_schedules": distinct,
        "distinct_schedules_per_s": round(distinct / t1, 1),
        "bank_sha256": hashlib.sha256(bank.to_bytes()).hexdigest(),
        "winners_sha256": hashlib.sha256(";".join(
            f"{r.size.m},{r.size.n},{r.size.k}:{r.winner.label}" for r in rec1).encode()).hexdigest(),
        "method": "pass 1 (build bank) and pass 2 (independent re-measurement) each time every (size, "
                  "policy) with CUDA-graph replays (warm-up 3, median of <=10); selected = fastest "
                  "pass-2 time among query(size) | {DP}; times are device events around each rank's share",
        "note": "bank bytes depend only on the winners (lexicographic insertion); winners of near-tied "
                "sizes can differ between runs, so compare winners_sha256 before bank_sha256",
    }


def host_selection(size, dtype: str):
    """The configuration the shipped tile bank selects WITHOUT timing anything: its Bloom
    candidates (corners + calibrated prior) plus the baseline; with several candidates the
    calibrated cost model's pick if it is one of them, else the first.  Used by the
    reference arm (which must not touch the GPU) and reported by ours for comparison."""
    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import tiles as tl

    bank = tl.TileBank.load(sk.default_bank_dir())
    cand = bank.candidates(size, "corners+model")
    if len(cand) == 1:
        return cand[0], cand
    try:
        pick = bank.prior_pick(size)
    except ValueError:
        pick = None
    return (pick if pick in cand else cand[0]), cand


def roofline(flops: float, nbytes: float, seconds: float, peaks: dict, sustained: bool = False) -> dict:
    """Roofline of the GEMM kernel.  Tensor-bound kernels are compared with the burst cuBLAS
    figure, or with the sustained one when the timed region ran long enough (> 100 ms back to
    back) to sit under the power cap (B200_PROFILING.md)."""
    t_tc = flops / (peaks["bf16_tflops"] * 1e12)
    t_hbm = nbytes / (peaks["hbm_gbs"] * 1e9)
    if t_tc >= t_hbm:
        ach = flops / seconds / 1e12
        peak = peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"]
        return {"bound": "tensor", "achieved": round(ach, 2), "peak": peak, "unit": "TFLOP/s",
                "frac": round(ach / peak, 4), "frac_of_burst": round(ach / peaks["bf16_tflops"], 4),
                "traffic": None,
                "peak_source": peaks["source"] + (", sustained bf16 (timed region > 100 ms back to back)"
                                                  if sustained else ", burst bf16")}
    ach = nbytes / seconds / 1e9
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None,
            "peak_source": peaks["source"] + ", copy bandwidth"}


def fixup_summary(plan, tile, policy, workload: str, flops: float, nbytes: float, seconds: float) -> dict:
    """Stream-K partial-tile (fixup workspace) traffic of one launch.

    Analytic: every partial item writes its valid rows x columns of fp32 once and the reducers
    read them back once.  Measured: the committed ncu difference between this shape's Stream-K
    launch and its data-parallel launch (same operands, same C): L2 write sectors and DRAM bytes
    (profiles/round2/ncu_fixup.json, tools/fixup_traffic.py), when that capture is of this
    (tile, policy)."""
    from paper_2408_11417_b200.scheduler import count_partials
    from paper_2408_11417_b200.tiles import tile_label

    partial, full, peers = count_partials(plan.sched_c)
    per_item = min(tile.blk_m, plan.size.m) * min(tile.blk_n, plan.size.n) * 4
    written = partial * per_item
    out = {
        "partial_items": partial, "non_owner_partials": peers, "full_tile_stores": full,
        "analytic_bytes_written": written, "analytic_bytes_read": written,
        "vs_algorithmic_bytes": round(2 * written / nbytes, 3),
        "analytic_rate_over_step_gbs": round(2 * written / seconds / 1e9, 1),
        "measured": None,
    }
    try:
        with open(os.path.join(ROOT, "profiles", "round2", "ncu_fixup.json")) as fh:
            rows = json.load(fh)["rows"]
        row = next(r for r in rows if r["workload"] == workload and r["tile"] == tile_label(tile)
                   and policy.label == "hybrid1")
        out["measured"] = {k: row[k] for k in ("workspace_dram_bytes", "workspace_hbm_gbs", "workspace_hbm_frac_of_peak",
                                               "l2_write_bytes_delta", "l2_write_delta_vs_analytic",
                                               "dp_l2_write_bytes_vs_c_bytes", "workspace_l2_write_gbs",
                                               "sk_duration_us", "source")}
        out["measured"]["file"] = "profiles/round2/ncu_fixup.json"
        out["measured"]["note"] = ("ncu (Stream-K launch) - (data-parallel launch): the partials stay in L2 "
                                   "(workspace HBM traffic ~0); L2 write sectors count 1.5x the stored bytes on "
                                   "this part for C as well (dp_l2_write_bytes_vs_c_bytes)")
    except (OSError, ValueError, KeyError, StopIteration):
        pass
    return out


def cpu_oracle_gemm(wl: dict, policy_kind: str, sk_batches: int, sk_first: bool, max_seconds: float,
                    max_reps: int, seed: int = 0, wg_stride: int = 1):
    """Time the oracle port of the reference executor (float64) on this host.

    ``wg_stride`` > 1 bounds the sample: each run executes the items of every
    ``wg_stride``-th workgroup of the schedule only.  Returns [(seconds, flops executed)]."""
    import numpy as np

    from oracle import gemm as ogemm
    from oracle import schedule as osched

    m, n, k = wl["m"], wl["n"], wl["k"]
    bm, bn, bk = wl["tile"]
    rng = np.random.default_rng(seed)
    a = ogemm.random_int_matrix(m, k, rng)
    b = ogemm.random_int_matrix(k, n, rng)
    # the tile's declared grid, else one workgroup per SM (per SM pair for 256-row tiles)
    g = wl.get("g") or 148 // (bm // 128)
    sched = osched.build_schedule(m, n, k, bm, bn, bk, g, policy_kind, sk_batches, sk_first)
    sched = sched[::wg_stride]
    n_tiles = -(-n // bn)
    flops = 0
    for wg in sched:
        for t, kb, ke, _wm, _ph in wg:
            tm, tn = divmod(t, n_tiles)
            flops += 2 * (min(bm, m - tm * bm)) * (min(bn, n - tn * bn)) * (min(ke * bk, k) - kb * bk)
    out = []
    # every host core for OpenBLAS, whatever OMP_NUM_THREADS the launcher set (torchrun sets 1)
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=len(os.sched_getaffinity(0))):
        t_start = time.perf_counter()
        while len(out) < max_reps and (not out or time.perf_counter() - t_start < max_seconds):
            t0 = time.perf_counter()
            ogemm.execute_schedule(a, b, sched, m, n, k, bm, bn, bk, n_tiles)
            out.append((time.perf_counter() - t0, flops))
    return out


def _policy_tuple(policy) -> tuple:
    return (policy.kind.value, policy.sk_batches, policy.sk_first)


def _config_keys(wl: dict, tile, g: int, policy_label: str, world: int) -> dict:
    """The ``config`` object both arms print (identical keys and values for the same selection)."""
    return {"workload": wl["desc"], "m": wl["m"], "n": wl["n"], "k": wl["k"],
            "tile": [tile.blk_m, tile.blk_n, tile.blk_k], "tile_order": getattr(tile, "band_rows", 0),
            "g": g, "policy": policy_label, "parallelism": f"replicas x{world} (GEMM is single-GPU)"}


CPU_STEP_BUDGET_S = 4.0  # reference arm: target CPU seconds per step (bounded sample)


def run_reference(args, wl: dict) -> None:
    world, rank, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    import paper_2408_11417_b200 as sk

    cores = len(os.sched_getaffinity(0))
    m, n, k = wl["m"], wl["n"], wl["k"]
    size = sk.ProblemSize(m, n, k)
    (tile, policy), cand = host_selection(size, wl["dtype"])
    g = sk.tile_grid(tile) or 148 // (tile.blk_m // 128)
    wlt = dict(wl, tile=(tile.blk_m, tile.blk_n, tile.blk_k), g=g)
    pol = _policy_tuple(policy)
    # One probe run of a 1/16 sample sizes the per-step sample so the whole --steps/--warmup
    # run stays within a few minutes: full schedule when a step fits CPU_STEP_BUDGET_S.
    probe = cpu_oracle_gemm(wlt, *pol, max_seconds=0, max_reps=1, wg_stride=16)[0]
    est_full = probe[0] * (2.0 * m * n * k) / probe[1]
    stride = max(1, int(-(-est_full // CPU_STEP_BUDGET_S)))
    cpu_oracle_gemm(wlt, *pol, max_seconds=1e9, max_reps=args.warmup, wg_stride=stride)  # warm-up
    runs = cpu_oracle_gemm(wlt, *pol, max_seconds=1e9, max_reps=args.steps, wg_stride=stride)
    total = sum(t for t, _ in runs)
    value = sum(f for _, f in runs) / total / 1e12
    sample = (f"{len(runs)} steps, each a {'full' if stride == 1 else f'1/{stride} workgroup sample of the'} "
              f"{m}x{n}x{k} schedule ({runs[0][1] / 1e9:.1f} GFLOP executed per step) run by the oracle port of "
              f"gemmsched executor.py:51-112 (float64 numpy/OpenBLAS)")
    line = {
        "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": len(runs), "warmup": args.warmup, "ms_per_step": round(total / len(runs) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (integer-valued float64, seed 0)",
        "config": _config_keys(wl, tile, g, policy.label, args.gpus),
        "selection": {"how": "host-side: shipped tile bank candidates (corners + calibrated prior), "
                             "calibrated-model pick among them (no GPU)",
                      "candidates": [f"{sk.tiles.tile_label(t)}/{p.label}" for t, p in cand]},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def select_config(size, tiles, pool):
    """The Stream-K++ selection for the workload: the shipped tile bank's Bloom candidates
    (corners + calibrated prior for sizes it never saw) plus the baseline, each timed, fastest
    wins.  Every (tile, canonical policy) of ``tiles`` is measured too (round-robin over 5
    rounds, median) — the measured oracle the selection is compared against."""
    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import sweep, tiles as tl

    bank = tl.TileBank.load(sk.default_bank_dir())
    cand = bank.candidates(size, "corners+model")
    all_tiles = list(tiles) + [t for t, _ in cand if t not in tiles]
    params = sweep.MeasureParams(warmup=3, reps=5, in_dtype=pool.a.dtype)
    per_tile = sweep.measure_size_tiles(size, all_tiles, sk.canonical_policies(), params, pool, rounds=5)
    rec = tl.joint_winner(size, per_tile)
    tile, policy = min(cand, key=lambda c: (rec.time_of(c), all_tiles.index(c[0]), c[1].sort_key()))
    return tile, policy, rec, cand


def run_ours(args, wl: dict) -> None:
    import numpy as np
    import torch

    world, rank, local = dist_setup(args.gpus)
    # Test hook: SKPP_BENCH_SHARED_GPU=1 runs every rank on cuda:0 over gloo, so the N > 1 control
    # flow (barriers, max-over-ranks, the sharded sweep's gather) can be exercised on a one-GPU box
    # (NCCL refuses two ranks on one device).  Numbers from such a run are not bench values.
    shared = os.environ.get("SKPP_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import sweep

    peaks = load_peaks()
    m, n, k = wl["m"], wl["n"], wl["k"]
    in_dtype = torch.bfloat16 if wl["dtype"] == "bf16" else torch.float16
    size = sk.ProblemSize(m, n, k)
    from paper_2408_11417_b200 import tiles as tl

    cand_tiles = [tl.parse_tile(t) for t in BENCH_TILES]
    pool = sweep.OperandPool([size], in_dtype, torch.float32, seed=rank)
    tile, policy, rec, cand = select_config(size, cand_tiles, pool)
    g = sk.executor.default_g(tile)
    wl = dict(wl, tile=(tile.blk_m, tile.blk_n, tile.blk_k), g=g)
    a, b, c = pool.views(size)
    plan = sk.GemmPlan(a, b, c, policy, tile, g)
    flops = 2.0 * m * n * k
    nbytes = 2.0 * (m * k + k * n) + 4.0 * m * n
    # Cold-L2 methodology: the timed steps rotate over R distinct operand sets (A, B, C)
    # whose total exceeds 4x the 126 MB L2, so every step reads its operands from HBM
    # (the set a step uses was last touched R-1 steps earlier, with >= 3 L2 capacities
    # of other traffic since).  Steps run back to back on one stream (PDL lets each
    # launch's prologue overlap the previous kernel's tail), bracketed by ONE pair of
    # CUDA events, so per-step time is the steady-state launch-to-launch time.
    set_bytes = 2 * (m * k + k * n) + 4 * m * n
    n_sets = max(2, -(-ROTATE_BYTES // set_bytes))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1000 + rank)
    plans = [plan]
    for _ in range(n_sets - 1):
        ar = torch.randn(m, k, generator=gen, device="cuda").to(in_dtype)
        br = torch.randn(k, n, generator=gen, device="cuda").to(in_dtype)
        cr = torch.empty(m, n, device="cuda", dtype=torch.float32)
        plans.append(sk.GemmPlan(ar, br, cr, policy, tile, g))
    stream = torch.cuda.current_stream()

    for i in range(max(args.warmup, 3) + n_sets):
        plans[i % n_sets].launch()
    torch.cuda.synchronize()

    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(physical_gpu(local)) as clocks:
        clocks.mark_start()
        t_start.record(stream)
        for i in range(args.steps):
            plans[i % n_sets].launch()
        t_end.record(stream)
        torch.cuda.synchronize()
        clocks.mark_end()
    if world > 1:
        torch.distributed.barrier()
    total_ms = t_start.elapsed_time(t_end)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cpu" if shared else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    per_step_s = total_ms / args.steps / 1e3
    value = world * flops * args.steps / (total_ms / 1e3) / 1e12

    # Isolated launches (informational): L2 flushed (256 MiB write + 256 MiB read, clean
    # lines) before every launch, one event pair per launch.  Includes the ~6 us an
    # event-timed EMPTY kernel costs after a flush on this GPU (tools/launchbench.cu).
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    scrub = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")
    iso = []
    for _ in range(ISOLATED_STEPS):
        flush.zero_()
        torch.sum(scrub, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.launch()
        e1.record(stream)
        iso.append((e0, e1))
    torch.cuda.synchronize()
    iso_us = statistics.median(e0.elapsed_time(e1) * 1e3 for e0, e1 in iso)
    del flush, scrub

    # end to end through the public API with pinned host inputs
    e2e_steps = min(args.steps, args.e2e_steps)
    a_h = a.cpu().pin_memory()
    b_h = b.cpu().pin_memory()
    sched = sk.build_schedule(size, tile, sk.HardwareModel(g, 1), policy)
    for _ in range(3):
        sk.execute_schedule(a_h, b_h, sched, tile, size)
    torch.cuda.synchronize()
    # at least e2e_steps calls and at least 0.5 s; the per-call median is robust to the
    # occasional slow host-side call (page-cache / pinned-pool hiccups)
    e2e_t = []
    t_loop = time.perf_counter()
    while len(e2e_t) < e2e_steps or (time.perf_counter() - t_loop < 0.5 and len(e2e_t) < 20 * e2e_steps):
        t0 = time.perf_counter()
        out = sk.execute_schedule(a_h, b_h, sched, tile, size)
        e2e_t.append(time.perf_counter() - t0)
    e2e_steps = len(e2e_t)
    e2e_med = statistics.median(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_med], dtype=torch.float64, device="cpu" if shared else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_med = float(t.item())
    e2e_value = world * flops / e2e_med / 1e12
    e2e_mean_value = world * flops * e2e_steps / sum(e2e_t) / 1e12
    assert out.shape == (m, n)

    sweep_block = sweep_check(world, rank, args.sweep_grid, args.sweep_tile)
    ref_cfg, _ = host_selection(size, wl["dtype"])
    if rank == 0:
        cores = len(os.sched_getaffinity(0))
        cpu_runs = cpu_oracle_gemm(wl, policy.kind.value, policy.sk_batches, policy.sk_first,
                                   max_seconds=args.cpu_seconds, max_reps=20) if world == 1 else []
        cpu_value = statistics.median(f / t for t, f in cpu_runs) / 1e12 if cpu_runs else None
        per_config = {f"{tl.tile_label(t)}/{p.label}": round(size.flops / (e.makespan * 1e-6) / 1e12, 2)
                      for t, r in rec.per_tile for p, e in r.costs}
        roof = roofline(flops, nbytes, per_step_s, peaks, sustained=total_ms > 100.0)
        roof["algorithmic_bytes"] = int(nbytes)
        roof["algorithmic_flops"] = int(flops)
        traffic, tsrc = ncu_traffic(args.workload, tl.tile_label(tile), policy.label)
        roof["traffic"] = traffic
        roof["traffic_source"] = tsrc
        best_us = rec.winner_us
        chosen_us = rec.time_of((tile, policy))
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "TFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(per_step_s * 1e3, 5),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": wl["dtype"],
            "data": "synthetic (randn operands, seeded)",
            "config": _config_keys(wl, tile, g, policy.label, world),
            "method": {
                "out_dtype": "fp32", "candidate_tiles": BENCH_TILES,
                "l2": f"cold: steps rotate over {n_sets} distinct operand sets "
                      f"({n_sets * set_bytes / 2**20:.0f} MiB > 4x the 126 MB L2); no flush",
                "timing": "one CUDA-event pair around K back-to-back launches on one stream",
            },
            "pct_of_dense_peak": {
                "measured_bf16": round(value / world / peaks["bf16_tflops"], 4),
                "spec_2250": round(value / world / 2250.0, 4),
            },
            "selection": {
                "selected": f"{tl.tile_label(tile)}/{policy.label}",
                "oracle_best": f"{tl.tile_label(rec.winner[0])}/{rec.winner[1].label}",
                "selected_vs_oracle": round(chosen_us / best_us, 4),
                "within_20pct": chosen_us <= 1.2 * best_us,
                "candidates": [f"{tl.tile_label(t)}/{p.label}" for t, p in cand],
                "bank": os.path.relpath(sk.default_bank_dir(), ROOT),
                "reference_arm_config": f"{tl.tile_label(ref_cfg[0])}/{ref_cfg[1].label}",
                "reference_arm_config_is_selected": ref_cfg == (tile, policy),
                "per_config_tflops": per_config,
                "note": "per-(tile, policy) times from CUDA-graph replays with warm L2 (selection sweep)",
            },
            "roofline": roof,
            "fixup": fixup_summary(plan, tile, policy, args.workload, flops, nbytes, per_step_s),
            "sweep": sweep_block,
            # the CPU leg runs on rank 0 at N = 1 only (the reference arm times it at every N)
            "cpu_baseline": {
                "value": round(cpu_value, 6), "unit": "TFLOP/s", "cores": cores, "kind": "port",
                "sample": f"{len(cpu_runs)} full {m}x{n}x{k} runs of the oracle port of gemmsched "
                          f"execute_schedule (float64 numpy/OpenBLAS, policy {policy.label})",
            } if cpu_value is not None else None,
            "e2e": {
                "value": round(e2e_value, 3), "unit": "TFLOP/s",
                "h2d_bytes_per_step": int(2 * (m * k + k * n)), "d2h_bytes_per_step": int(4 * m * n),
                "api": f"paper_2408_11417_b200.execute_schedule(pinned host {wl['dtype']} tensors)",
                "steps": e2e_steps, "statistic": "median per-call wall time (max over ranks)",
                "mean_value": round(e2e_mean_value, 3),
            },
            "isolated_launch": {
                "us_median": round(iso_us, 2), "tflops": round(flops / (iso_us * 1e-6) / 1e12, 2),
                "steps": ISOLATED_STEPS,
                "method": "L2 flushed before each launch, one event pair per launch (includes ~6 us "
                          "event+launch floor of an empty kernel, tools/launchbench.cu)",
            },
            "gpu_launches": args.steps,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3")
    ap.add_argument("--sweep-grid", default="paper",
                    help="grid of the in-run selection check (sweep.grid_sizes name, or 'none')")
    ap.add_argument("--sweep-tile", default=SWEEP_TILE)
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
