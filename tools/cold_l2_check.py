#!/usr/bin/env python
"""Does warm-L2 timing pick different winners than cold-L2 timing?

The sweep times every (size, policy) with CUDA-graph replays on ONE operand set, so sizes
whose operands fit in the 126 MB L2 are timed warm.  For every grid size whose operand set
(2(MK + KN) + 4MN bytes) lies in [--min-mb, 126 MB], this re-measures all seven policies of
the size's warm joint-winner tile COLD: each graph replay cycles through R distinct operand
sets with R x set bytes > 4 x L2 (R <= --max-sets), and reports how many winners change and
what keeping the warm winner costs under cold timing.

    python tools/cold_l2_check.py --records profiles/round2/sweep_r2_records --out gpurun_out/cold
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
L2 = 126 * 1024 * 1024


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", default=os.path.join(ROOT, "profiles", "round2", "sweep_r2_records"))
    ap.add_argument("--tiles", default="128x128x64,128x64x128,128x128x128,256x256x64,256x256x128,"
                                      "128x128x128b16,256x256x128b16")
    ap.add_argument("--min-mb", type=float, default=2.0)
    ap.add_argument("--max-sets", type=int, default=128)
    ap.add_argument("--limit", type=int, default=0, help="check only the first N eligible sizes")
    ap.add_argument("--out", default="gpurun_out/cold")
    args = ap.parse_args()

    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import tiles as tl
    from paper_2408_11417_b200.scheduler import schedule_signature

    tiles = [tl.parse_tile(t) for t in args.tiles.split(",")]
    joint = tl.joint_records_from_csvs([(t, f"{args.records}.{tl.tile_label(t)}.csv") for t in tiles])
    eligible = []
    for rec in joint:
        z = rec.size
        b = 2 * (z.m * z.k + z.k * z.n) + 4 * z.m * z.n
        if args.min_mb * 1e6 <= b <= L2:
            eligible.append((rec, b))
    if args.limit:
        eligible = eligible[: args.limit]
    os.makedirs(args.out, exist_ok=True)
    rows = []
    t_start = time.perf_counter()
    for rec, set_bytes in eligible:
        z = rec.size
        tile = rec.winner[0]
        r_sets = min(args.max_sets, max(2, math.ceil(4 * L2 / set_bytes)))
        sets = [(torch.randn(z.m, z.k, device="cuda").to(torch.bfloat16),
                 torch.randn(z.k, z.n, device="cuda").to(torch.bfloat16),
                 torch.empty(z.m, z.n, device="cuda")) for _ in range(r_sets)]
        warm = {p: e.makespan for t, r in rec.per_tile if t == tile for p, e in r.costs}
        cold: dict = {}
        by_sig: dict = {}
        for pol in sk.canonical_policies():
            plans = [sk.GemmPlan(a, b, c, pol, tile) for a, b, c in sets]
            sig = schedule_signature(plans[0].sched_c)
            if sig in by_sig:
                cold[pol] = by_sig[sig]
                continue
            side = torch.cuda.Stream()
            for p in plans:
                p.prepare_for_capture(side)
            side.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                for p in plans:
                    p.launch()  # warm-up outside the graph
                g.capture_begin()
                for p in plans:
                    p.launch()
                g.capture_end()
            torch.cuda.current_stream().wait_stream(side)
            g.replay()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / len(plans))
            cold[pol] = by_sig[sig] = statistics.median(ts)
            del g
        warm_w = min(warm, key=lambda p: (warm[p], p.sort_key()))
        cold_w = min(cold, key=lambda p: (cold[p], p.sort_key()))
        rows.append({"m": z.m, "n": z.n, "k": z.k, "tile": tl.tile_label(tile), "set_mb": round(set_bytes / 1e6, 2),
                     "sets": r_sets, "warm_winner": warm_w.label, "cold_winner": cold_w.label,
                     "warm_winner_cold_us": round(cold[warm_w], 3), "cold_best_us": round(cold[cold_w], 3),
                     "regret": round(cold[warm_w] / cold[cold_w], 4),
                     "warm_us": round(warm[warm_w], 3)})
        del sets
    changed = [r for r in rows if r["warm_winner"] != r["cold_winner"]]
    summary = {
        "sizes_checked": len(rows), "criterion": f"operand set in [{args.min_mb} MB, 126 MB] (fits in L2)",
        "winners_changed": len(changed),
        "changed_with_regret_over_5pct": sum(1 for r in changed if r["regret"] > 1.05),
        "changed_with_regret_over_20pct": sum(1 for r in changed if r["regret"] > 1.20),
        "max_regret": max((r["regret"] for r in rows), default=1.0),
        "median_cold_over_warm_of_winner": statistics.median(r["warm_winner_cold_us"] / r["warm_us"] for r in rows)
        if rows else None,
        "seconds": round(time.perf_counter() - t_start, 1),
        "method": "all 7 policies of the size's warm joint-winner tile; one CUDA graph per schedule cycling "
                  "through R operand sets (R x set > 4 x L2, R <= max-sets), median of 5 replays",
    }
    with open(os.path.join(args.out, "cold_l2_check.json"), "w") as fh:
        json.dump({"summary": summary, "rows": rows}, fh, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
