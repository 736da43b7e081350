#!/usr/bin/env python
"""Copy a joint sweep (e.g. tools/gpurun_sweep_r2.sh -> gpurun_out/sweep_r2/) into
profiles/<round>/<prefix>_*: per-tile records and held-out CSVs (the validate pass is kept
only as the summary's selection_heldout_run), the summary, the per-size cost table and the
tile bank (with its calibrated cost-model priors); optionally install the bank as the
package's shipped bank (paper_2408_11417_b200/banks/b200)."""
import glob
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(src="gpurun_out/sweep_r2", prefix="sweep_r2", bank="tilebank7", rnd="round2", install="1"):
    src = os.path.join(ROOT, src)
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    n = 0
    for tag in ("records", "heldout"):
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
    if install == "1":
        ship = os.path.join(ROOT, "paper_2408_11417_b200", "banks", "b200")
        shutil.rmtree(ship, ignore_errors=True)
        shutil.copytree(os.path.join(src, "tilebank"), ship)
    print(f"copied {n} CSVs, summary, costs and {bank}/ into profiles/{rnd}/" + (" and installed the bank" if install == "1" else ""))


if __name__ == "__main__":
    main(*sys.argv[1:])
