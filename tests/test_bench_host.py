"""bench.py host-side pieces that need no GPU: the committed ncu captures resolve to the
kernel configurations the bench selects (roofline.traffic), and the sweep summary loads."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_committed_ncu_traffic_matches_selected_configs():
    for wl in ("cfg2", "cfg1", "square8192"):
        line = json.load(open(os.path.join(ROOT, "profiles", "round1", f"bench_{wl}.json")))
        tile = "x".join(str(v) for v in line["config"]["tile"])
        traffic, src = bench.ncu_traffic(wl, tile, line["config"]["policy"])
        assert traffic is not None and traffic > 0, (wl, tile)
        assert src == f"profiles/ncu_bench_{wl}.json"


def test_sweep_summary_reports_selection_quality():
    s = bench.sweep_summary()
    assert s is not None and s["sizes"] > 1000
    assert s["pct_within_20pct_of_oracle_heldout_run"] >= 97.6  # the paper's figure
