#!/usr/bin/env python
"""BASELINE config 3 table from the committed joint sweep: Llama-3-8B projections,
Bloom-selected (tile, policy) vs data-parallel vs the measured oracle."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2408_11417_b200 as sk  # noqa: E402
from paper_2408_11417_b200 import tiles as tl  # noqa: E402

R = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "round1")
TILES = [sk.TileShape(128, 128, 64), sk.TileShape(128, 64, 128), sk.TileShape(128, 128, 128),
         sk.TileShape(256, 256, 64), sk.TileShape(256, 256, 128)]
paths = [(t, os.path.join(R, f"sweep_joint5_records.{tl.tile_label(t)}.csv")) for t in TILES]
joint = {r.size: r for r in tl.joint_records_from_csvs(paths)}
bank = tl.build_tile_bank(list(joint.values()), TILES)
print("| M | N | dp_util (128x128) | DP 128x128x64 µs | best DP (any tile) µs | selected (tile, policy) | selected µs | TFLOP/s "
      "| vs DP 128x128x64 | vs best DP | vs oracle |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
wq, wq_best = [], []
for m in [1 << e for e in range(14)]:
    for n in (4096, 14336):
        size = sk.ProblemSize(m, n, 4096)
        rec = joint[size]
        cand = bank.candidates(size)
        chosen = min(cand, key=lambda c: rec.time_of(c))
        t_sel = rec.time_of(chosen)
        t_dp = rec.time_of(bank.baseline)
        t_dp_best = min(rec.time_of((t, sk.Policy.data_parallel())) for t in TILES)
        util = sk.dp_utilization(sk.grid_info(size, TILES[0]), 148)
        tf = size.flops / (t_sel * 1e-6) / 1e12
        if util < 0.9:
            wq.append(t_dp / t_sel)
            wq_best.append(t_dp_best / t_sel)
        print(f"| {m} | {n} | {util:.3f} | {t_dp:.1f} | {t_dp_best:.1f} | {tl.tile_label(chosen[0])} {chosen[1].label} | "
              f"{t_sel:.1f} | {tf:.1f} | {t_dp / t_sel:.2f}x | {t_dp_best / t_sel:.2f}x | {t_sel / rec.winner_us:.2f} |")
import math  # noqa: E402
def gm(v):
    return math.exp(sum(map(math.log, v)) / len(v))


print(f"\nwave-quantisation-bound sizes (dp_util < 0.9): {len(wq)}; selected config vs data-parallel on the "
      f"baseline tile: geomean {gm(wq):.2f}x, min {min(wq):.2f}x; vs data-parallel on the best tile: geomean "
      f"{gm(wq_best):.2f}x, min {min(wq_best):.2f}x")
