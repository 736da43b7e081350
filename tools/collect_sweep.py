#!/usr/bin/env python
"""Copy a joint sweep (tools/gpurun_sweep_paper.sh -> gpurun_out/sweep_joint5/) into
profiles/round1/sweep_joint5_*: per-tile records / validate / heldout CSVs, the summary,
the per-size cost table and the tile bank (with its calibrated cost-model priors)."""
import glob
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(src="gpurun_out/sweep_joint5", prefix="sweep_joint5", bank="tilebank5"):
    src = os.path.join(ROOT, src)
    dst = os.path.join(ROOT, "profiles", "round1")
    n = 0
    for tag in ("records", "validate", "heldout"):
        for p in glob.glob(os.path.join(src, f"{tag}.*.csv")):
            name = os.path.basename(p)
            if ".rank" in name:
                continue
            tile = name[len(tag) + 1:-4]
            shutil.copy(p, os.path.join(dst, f"{prefix}_{tag}.{tile}.csv"))
            n += 1
    shutil.copy(os.path.join(src, "summary.json"), os.path.join(dst, f"{prefix}_summary.json"))
    costs = os.path.join(src, "costs.records.rank0.json")
    if os.path.exists(costs):
        shutil.copy(costs, os.path.join(dst, f"{prefix}_costs.json"))
    out_bank = os.path.join(dst, bank)
    shutil.rmtree(out_bank, ignore_errors=True)
    shutil.copytree(os.path.join(src, "tilebank"), out_bank)
    print(f"copied {n} CSVs, summary, costs and {bank}/ into profiles/round1/")


if __name__ == "__main__":
    main(*sys.argv[1:])
