#!/usr/bin/env python
"""A/B: cooperative launch of Stream-K grids (skpp_set_cooperative) vs a plain launch.

Per shape, K back-to-back launches (PDL on) rotating over cold operand sets between one
CUDA-event pair, interleaved off/on rounds; prints the median us/launch of each mode.
"""

from __future__ import annotations

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import _lib
    from paper_2408_11417_b200.tiles import parse_tile

    cases = [(512, 512, 16384, "128x128x128", sk.Policy.hybrid(1)),
             (8192, 14336, 4096, "256x256x128b16", sk.Policy.hybrid(1)),
             (16, 4096, 4096, "128x128x128", sk.Policy.hybrid(1)),
             (1024, 1024, 1024, "128x128x64", sk.Policy.hybrid(1))]
    out = []
    for m, n, k, tl, pol in cases:
        tile = parse_tile(tl)
        set_bytes = 2 * (m * k + k * n) + 4 * m * n
        n_sets = max(2, -(-(512 << 20) // set_bytes))
        plans = []
        for _ in range(n_sets):
            a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
            b = torch.randn(k, n, device="cuda").to(torch.bfloat16)
            c = torch.empty(m, n, device="cuda")
            plans.append(sk.GemmPlan(a, b, c, pol, tile))
        steps = max(50, int(200000 / max(1.0, 2 * m * n * k / 1e12 * 1e6 / 1000)))
        steps = min(steps, 5000)
        res = {0: [], 1: []}
        for rnd in range(6):
            for coop in (0, 1):
                _lib.lib.skpp_set_cooperative(coop)
                for i in range(20):
                    plans[i % n_sets].launch()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for i in range(steps):
                    plans[i % n_sets].launch()
                e1.record()
                torch.cuda.synchronize()
                res[coop].append(e0.elapsed_time(e1) * 1e3 / steps)
        _lib.lib.skpp_set_cooperative(1)
        row = {"shape": f"{m}x{n}x{k}", "tile": tl, "policy": pol.label, "steps": steps,
               "plain_us": round(statistics.median(res[0]), 3), "coop_us": round(statistics.median(res[1]), 3)}
        row["coop_over_plain"] = round(row["coop_us"] / row["plain_us"], 4)
        print(json.dumps(row), flush=True)
        out.append(row)


if __name__ == "__main__":
    main()
