"""Shipped 7-tile bank + one grid tile (128x128x128g144) whose filters hold only the sizes where
that tile beat every shipped config by more than 2% in the pass-1 records of the 10-tile sweep
(profiles/round2/session5/sweep_s5_grid_records.*).  The seven shipped banks are unchanged, so a
query's candidates are a superset of the shipped bank's; selection quality is evaluated on the
sweep's independent pass-2 records (held-out run).

usage: python tools/build_union_bank.py [--install]
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2408_11417_b200 import tiles as tl  # noqa: E402
from paper_2408_11417_b200.sieve import SieveBank  # noqa: E402

SWEEP = os.path.join(ROOT, "profiles", "round2", "session5")
TILES10 = ["128x128x64", "128x64x128", "128x128x128", "256x256x64", "256x256x128", "128x128x128b16",
           "256x256x128b16", "128x128x128g128", "128x128x128g144", "128x64x128g128"]
GRID_TILE = "128x128x128g144"
MARGIN = 1.02


def main() -> None:
    shipped = tl.TileBank.load(tl.default_bank_dir())
    shipped_labels = [tl.tile_label(t) for t in shipped.tiles]
    recs = tl.joint_records_from_csvs([(tl.parse_tile(t), os.path.join(SWEEP, f"sweep_s5_grid_records.{t}.csv"))
                                       for t in TILES10])
    val = tl.joint_records_from_csvs([(tl.parse_tile(t), os.path.join(SWEEP, "validate", f"sweep_s5_grid_validate.{t}.csv"))
                                      for t in TILES10])
    gt = tl.parse_tile(GRID_TILE)
    gbank = SieveBank()
    inserted = []
    for r in sorted(recs, key=lambda r: (r.size.m, r.size.n, r.size.k)):
        best7 = min(e.makespan for t, rec in r.per_tile if tl.tile_label(t) in shipped_labels for _, e in rec.costs)
        pol, best_g = min(((p, e.makespan) for t, rec in r.per_tile if t == gt for p, e in rec.costs),
                          key=lambda pe: (pe[1], pe[0].sort_key()))
        if best7 > MARGIN * best_g:
            gbank.insert(r.size, pol)
            inserted.append((r.size.m, r.size.n, r.size.k, pol.label, round(best7 / best_g, 3)))
    union = tl.TileBank(shipped.tiles + [gt], shipped.banks + [gbank])
    union.priors = shipped.priors + [None]
    out = {"grid_tile": GRID_TILE, "margin": MARGIN, "inserted": len(inserted),
           "inserted_examples": inserted[:20],
           "shipped_on_pass2": tl.evaluate_selection(shipped, val),
           "union_on_pass2": tl.evaluate_selection(union, val)}
    print(json.dumps(out, indent=1))
    if "--install" in sys.argv:
        union.save(tl.default_bank_dir())
        with open(os.path.join(SWEEP, "union_bank.json"), "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
