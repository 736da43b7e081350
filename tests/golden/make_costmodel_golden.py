#!/usr/bin/env python
"""Generate tests/golden/costmodel_golden.json by running the REFERENCE cost model.

Run in the build container only (the GPU box has no /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_costmodel_golden.py

``gemmsched.costmodel.estimate`` / ``pick_winner`` (costmodel.py:91-164) on seeded
random (size, tile, g, policy, CostParams) instances -- including DP-first and
non-canonical hybrids, where the overlap discount differs -- plus the reference's own
worked examples (tests/test_costmodel.py).  The fixtures pin the analytic model that
paper_2408_11417_b200.costmodel restates (item-wise and in closed form) and calibrates.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import gemmsched as G  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "costmodel_golden.json")


def pol_tuple(p):
    return [p.kind.value, p.sk_batches, bool(p.sk_first)]


def main():
    rng = np.random.default_rng(2408)
    policies = G.canonical_policies() + [G.Policy.hybrid(2, False), G.Policy.hybrid(4, False), G.Policy.hybrid(7)]
    cases = []
    for i in range(400):
        size = G.ProblemSize(*(int(2 ** rng.uniform(0, 13)) for _ in range(3)))
        tile = G.TileShape(int(rng.choice([16, 64, 128, 256])), int(rng.choice([16, 64, 128, 256])),
                           int(rng.choice([8, 32, 64, 128])))
        g = int(rng.choice([1, 3, 5, 37, 104, 148, int(rng.integers(1, 300))]))
        params = G.CostParams(c_mac=float(rng.choice([1.0, 0.5, 2.0])), c_store=float(rng.choice([0.0, 1.0, 4.0, 7.5])),
                              c_atomic=float(rng.choice([0.0, 4.0, 16.0, 40.0])),
                              overlap=float(rng.choice([0.0, 0.25, 0.75, 1.0])))
        pol = policies[i % len(policies)]
        hw = G.HardwareModel(g, 1)
        est = G.estimate(G.build_schedule(size, tile, hw, pol), params)
        cases.append({"m": size.m, "n": size.n, "k": size.k, "tile": [tile.blk_m, tile.blk_n, tile.blk_k], "g": g,
                      "policy": pol_tuple(pol), "params": [params.c_mac, params.c_store, params.c_atomic, params.overlap],
                      "makespan": est.makespan, "utilization": est.utilization, "atomic_writes": est.atomic_writes,
                      "full_stores": est.full_stores,
                      "per_wg_cost": list(est.per_wg_cost) if len(est.per_wg_cost) <= 8 else None,
                      "per_wg_sum": float(sum(est.per_wg_cost))})
    winners = []
    for i in range(120):
        size = G.ProblemSize(*(int(2 ** rng.uniform(0, 14)) for _ in range(3)))
        tile = G.TileShape(*[int(v) for v in rng.choice([[128, 128, 64], [256, 128, 32], [128, 256, 64]])])
        g = int(rng.choice([104, 148, 74]))
        params = G.CostParams() if i % 2 == 0 else G.CostParams(1.0, float(rng.uniform(0, 10)),
                                                                float(rng.uniform(0, 60)), float(rng.uniform(0, 1)))
        rec = G.pick_winner(size, tile, G.HardwareModel(g, 1), G.canonical_policies(), params)
        winners.append({"m": size.m, "n": size.n, "k": size.k, "tile": [tile.blk_m, tile.blk_n, tile.blk_k], "g": g,
                        "params": [params.c_mac, params.c_store, params.c_atomic, params.overlap],
                        "winner": pol_tuple(rec.winner), "runner_up": pol_tuple(rec.runner_up), "gain": rec.gain,
                        "makespans": [e.makespan for _, e in rec.costs]})
    bad_params = []
    for kw in ({"c_mac": -1.0}, {"c_store": -0.5}, {"c_atomic": -2.0}, {"overlap": 1.5}, {"overlap": -0.1}):
        try:
            G.CostParams(**kw)
            bad_params.append({"kwargs": kw, "error": None})
        except ValueError as e:
            bad_params.append({"kwargs": kw, "error": str(e)})
    try:
        G.CostParams.from_dict({"c_mac": 1.0, "bogus": 2.0})
        unknown = None
    except ValueError as e:
        unknown = str(e)
    out = {"generator": "tests/golden/make_costmodel_golden.py", "reference": "gemmsched.costmodel (costmodel.py:26-164)",
           "defaults": [G.CostParams().c_mac, G.CostParams().c_store, G.CostParams().c_atomic, G.CostParams().overlap],
           "estimate": cases, "pick_winner": winners, "bad_params": bad_params, "unknown_key_error": unknown}
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=0)
    print("wrote", OUT, len(cases), len(winners))


if __name__ == "__main__":
    main()
