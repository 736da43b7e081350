#!/usr/bin/env python
"""Summarise gpurun_out/prof/ (tools/gpurun_profile.sh) into profiles/: ncu_bench_<workload>.json
(one row per captured (tile, policy), read by bench.py for roofline.traffic), the launch list and
the bench lines under profiles/<round>/."""
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.ncu_summary import launches, raw  # noqa: E402


def main(src="gpurun_out/prof", round_dir="profiles/round1"):
    src = os.path.join(ROOT, src)
    out = os.path.join(ROOT, round_dir)
    os.makedirs(out, exist_ok=True)
    per_wl = {}
    for rep in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
        name = os.path.basename(rep)[:-8]
        wl, tile, policy = name.split("_", 2)
        pol = {"dp": "data-parallel", "ask": "all-streamk"}.get(policy, policy)
        for row in raw(rep):
            row.update({"tile": tile, "policy": pol, "capture": f"{name}.ncu-rep (ncu --set full, 1 launch)"})
            per_wl.setdefault(wl, []).append(row)
    for wl, rows in per_wl.items():
        with open(os.path.join(ROOT, "profiles", f"ncu_bench_{wl}.json"), "w") as fh:
            json.dump(rows, fh, indent=1)
        with open(os.path.join(out, f"ncu_{wl}.json"), "w") as fh:
            json.dump(rows, fh, indent=1)
    for lp in glob.glob(os.path.join(src, "launches_*.csv")):
        name = os.path.basename(lp)[:-4]
        with open(os.path.join(out, f"{name}.json"), "w") as fh:
            json.dump(launches(lp), fh, indent=1)
    for f in glob.glob(os.path.join(src, "bench_*.json")):
        shutil.copy(f, out)
    print("wrote", sorted(per_wl), "to profiles/")


if __name__ == "__main__":
    main(*sys.argv[1:])
