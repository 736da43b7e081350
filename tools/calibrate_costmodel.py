#!/usr/bin/env python
"""Calibrate the reference's analytic cost model (CostParams) to the B200 sweep and
score it as a selection prior.  CPU only: reads the committed
records CSVs (reference schema, makespan = measured microseconds).

  on-grid  : profiles/round1/sweep_joint5_records.<tile>.csv   (fit)
  held-out : profiles/round1/sweep_joint5_heldout.<tile>.csv   (300 off-grid sizes, score)
  validate : profiles/round1/sweep_joint5_validate.<tile>.csv  (on-grid re-measurement, score)

Writes profiles/round1/costmodel_calibration.json and the priors into the tile bank
manifest (profiles/round1/tilebank5/tilebank.json) so TileBank.load picks them up.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2408_11417_b200 import costmodel as cm, tiles as tl  # noqa: E402
from paper_2408_11417_b200.pipeline import read_records_csv, records_from_rows  # noqa: E402

PROF = os.path.join(ROOT, "profiles", "round1")
TILES = ["128x128x64", "128x64x128", "128x128x128", "256x256x64", "256x256x128"]


def load(kind, tile):
    return records_from_rows(read_records_csv(os.path.join(PROF, f"sweep_joint5_{kind}.{tile}.csv")))


def g_of(tile):
    return 148 // (tile.blk_m // 128)


def per_tile_score(cal_params, tile, recs, tol=0.2):
    g = g_of(tile)
    within, ratios = 0, []
    for r in recs:
        pols = sorted((p for p, _ in r.costs), key=lambda p: p.sort_key())
        us = {p: e.makespan for p, e in r.costs}
        spans = [cm.estimate_closed(r.size, tile, g, p, cal_params) for p in pols]
        pick = pols[int(np.argmin(spans))]
        ratio = us[pick] / min(us.values())
        ratios.append(ratio)
        within += ratio <= 1 + tol
    return within / len(recs), float(np.exp(np.mean(np.log(ratios))))


def main():
    tiles = [tl.parse_tile(t) for t in TILES]
    cals, out = {}, {"tiles": {}, "method": cm.calibrate.__doc__.split("\n\n")[0].strip()}
    for label, tile in zip(TILES, tiles):
        fit = load("records", label)
        cal = cm.calibrate(((r.size, [(p, e.makespan) for p, e in r.costs]) for r in fit), tile, g_of(tile))
        cals[label] = cal
        row = {"calibration": cal.to_dict()}
        for kind in ("records", "validate", "heldout"):
            recs = load(kind, label)
            fc, gc = per_tile_score(cal.params, tile, recs)
            fd, gd = per_tile_score(cm.CostParams(), tile, recs)
            dp = [min(1e9, dict((p, e.makespan) for p, e in r.costs)[cm.Policy.data_parallel()] /
                      min(e.makespan for _, e in r.costs)) for r in recs]
            row[kind] = {"sizes": len(recs), "calibrated_within_20pct": fc, "calibrated_geomean_slowdown": gc,
                         "reference_default_params_within_20pct": fd, "reference_default_geomean_slowdown": gd,
                         "dp_only_within_20pct": float(np.mean(np.array(dp) <= 1.2))}
        # affine us fit quality on held-out
        ho = load("heldout", label)
        err = [abs(cal.predict_us(r.size, p) - e.makespan) / e.makespan for r in ho for p, e in r.costs]
        row["heldout_us_prediction_median_rel_err"] = float(np.median(err))
        out["tiles"][label] = row
        print(label, json.dumps({k: row[k] for k in ("records", "heldout")}), flush=True)

    # joint (tile, policy) prior vs Bloom selection on the held-out and validation sets
    bank = tl.TileBank.load(os.path.join(PROF, "tilebank5"))
    bank.priors = [cals[tl.tile_label(t)] for t in bank.tiles]
    for kind in ("heldout", "validate"):
        recs = tl.joint_records_from_csvs([(t, os.path.join(PROF, f"sweep_joint5_{kind}.{tl.tile_label(t)}.csv"))
                                           for t in bank.tiles])
        res = {}
        for mode in (False, "corners", "model", "corners+model"):
            res[str(mode)] = tl.evaluate_selection(bank, recs, nearest=mode)
        # the model alone (no Bloom filters, no measurement): one pick per size
        within, ratios = 0, []
        for r in recs:
            pick = bank.prior_pick(r.size)
            ratio = r.time_of(pick) / r.winner_us
            ratios.append(ratio)
            within += ratio <= 1.2
        res["model_only_single_pick"] = {"fraction_within": within / len(recs),
                                         "geomean_slowdown": float(np.exp(np.mean(np.log(ratios))))}
        out[f"joint_{kind}"] = res
        print(kind, json.dumps({k: (v.get("fraction_within"), v.get("eliminated_fraction")) for k, v in res.items()}))
    with open(os.path.join(PROF, "costmodel_calibration.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    bank_dir = os.path.join(PROF, "tilebank5")
    with open(os.path.join(bank_dir, "tilebank.json")) as fh:
        man = json.load(fh)
    for e in man["tiles"]:
        e["prior"] = cals[e["tile"]].to_dict()
    with open(os.path.join(bank_dir, "tilebank.json"), "w") as fh:
        json.dump(man, fh, indent=1)


if __name__ == "__main__":
    main()
