"""bench.py host-side pieces that need no GPU: the committed ncu captures resolve to the
kernel configurations the bench selects (roofline.traffic, template arguments including the
tile order), the reference arm's host-side selection, and the shared config keys."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_committed_ncu_traffic_matches_selected_configs():
    for wl in ("cfg2", "cfg1"):
        line = json.load(open(os.path.join(ROOT, "profiles", "round1", f"bench_{wl}.json")))
        tile = "x".join(str(v) for v in line["config"]["tile"])
        traffic, src = bench.ncu_traffic(wl, tile, line["config"]["policy"])
        assert traffic is not None and traffic > 0, (wl, tile)
        assert src == f"profiles/ncu_bench_{wl}.json"


def test_ncu_traffic_distinguishes_the_tile_order():
    """The round-1 square8192 capture is of the banded instantiation <256, 128, 2, 1>; the
    reference-order tile 256x256x128 must not pick it up, the banded tile must."""
    assert bench.ncu_traffic("square8192", "256x256x128", "data-parallel") == (None, None)
    traffic, _ = bench.ncu_traffic("square8192", "256x256x128b16", "data-parallel")
    assert traffic and traffic > 0


def test_reference_arm_selection_is_host_only_and_in_the_candidates():
    import paper_2408_11417_b200 as sk

    for wl in bench.WORKLOADS.values():
        size = sk.ProblemSize(wl["m"], wl["n"], wl["k"])
        cfg, cand = bench.host_selection(size, wl["dtype"])
        assert cfg in cand
        assert (sk.TileShape(128, 128, 64), sk.Policy.data_parallel()) in cand  # the baseline


def test_both_arms_print_the_same_config_keys():
    import paper_2408_11417_b200 as sk

    wl = bench.WORKLOADS["cfg3"]
    t = sk.kernel_tile(256, 256, 128, 16)
    cfg = bench._config_keys(wl, t, 74, "hybrid1", 1)
    assert cfg["tile"] == [256, 256, 128] and cfg["tile_order"] == 16 and cfg["m"] == 8192
    assert set(cfg) == {"workload", "m", "n", "k", "tile", "tile_order", "g", "policy", "parallelism"}


def test_default_workload_is_cfg3_and_sweep_check_can_be_disabled():
    import argparse  # noqa: F401

    assert bench.WORKLOADS["cfg3"]["n"] == 14336
    assert bench.sweep_check(1, 0, "none", bench.SWEEP_TILE) is None


def test_clock_sampler_summary_window_and_reasons():
    """Samples are stamped when taken; only those inside [mark_start, mark_end] count, and the
    reason bits map to the names the driver checks (NVML clock-event reason masks)."""
    import bench

    cs = bench.ClockSampler(0)
    cs.t0, cs.t1 = 10.0, 10.02
    cs.samples = [(9.99, 1000.0, 1965.0, 0), (10.005, 1965.0, 1965.0, 0x4), (10.012, 1950.0, 1965.0, 0),
                  (10.019, 1965.0, 1965.0, 0x40), (10.05, 800.0, 1965.0, 0x8)]
    out = cs.summary()
    assert out["samples"] == 3 and out["sm_mhz"] == 1965.0 and out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["hw_thermal_slowdown", "sw_power_cap"]
    cs.t0, cs.t1 = 10.03, 10.031  # region shorter than one poll: the first sample after its start
    assert cs.summary()["samples"] == 1 and cs.summary()["reasons"] == ["hw_slowdown"]


def test_clock_sampler_exit_waits_for_a_sample_after_the_region_started():
    """A timed region shorter than one poll (or one during which the poller did not run) still
    gets a sample: __exit__ waits (bounded) for the first sample taken after mark_start."""
    import threading
    import time

    import bench

    cs = bench.ClockSampler(0)

    def late_poll():
        time.sleep(0.05)
        cs.samples.append((time.time(), 1950.0, 1965.0, 0))
        while not cs.stop:
            time.sleep(0.002)

    cs.thread = threading.Thread(target=late_poll, daemon=True)
    cs.thread.start()
    cs.mark_start()
    cs.mark_end()
    cs.__exit__(None, None, None)
    out = cs.summary()
    assert out["samples"] == 1 and out["sm_mhz"] == 1950.0
