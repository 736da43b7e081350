#!/usr/bin/env python
"""Host-side cost of the drop-in path: GemmPlan creation, and the per-call breakdown of
execute_schedule with pinned host inputs (H2D, kernel, D2H) for cfg2 and cfg3 shapes."""

from __future__ import annotations

import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200.tiles import parse_tile

    from paper_2408_11417_b200 import executor as ex

    for m, n, k, tl, pol in [(16, 4096, 4096, "128x128x128", sk.Policy.hybrid(1)),
                             (512, 512, 16384, "128x128x128", sk.Policy.hybrid(1)),
                             (8192, 14336, 4096, "256x256x128b16", sk.Policy.hybrid(3))]:
        tile = parse_tile(tl)
        a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        b = torch.randn(k, n, device="cuda").to(torch.bfloat16)
        c = torch.empty(m, n, device="cuda")
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            sk.GemmPlan(a, b, c, pol, tile)
            ts.append(time.perf_counter() - t0)
        size = sk.ProblemSize(m, n, k)
        sched = sk.build_schedule(size, tile, sk.HardwareModel(sk.executor.default_g(tile), 1), pol)
        a_h, b_h = a.cpu().pin_memory(), b.cpu().pin_memory()
        calls = []
        for i in range(40):
            t0 = time.perf_counter()
            out = sk.execute_schedule(a_h, b_h, sched, tile, size)
            calls.append(time.perf_counter() - t0)
        calls = calls[3:]
        print(json.dumps({"shape": f"{m}x{n}x{k}", "tile": tl, "plan_create_us_median": round(statistics.median(ts) * 1e6, 1),
                          "execute_schedule_ms": {"median": round(statistics.median(calls) * 1e3, 3),
                                                  "min": round(min(calls) * 1e3, 3), "max": round(max(calls) * 1e3, 3),
                                                  "p90": round(sorted(calls)[int(0.9 * len(calls))] * 1e3, 3)},
                          "h2d_bytes": 2 * (m * k + k * n), "d2h_bytes": 4 * m * n,
                          "plan_cache": dict(ex._plan_cache_stats)}), flush=True)
        del out


if __name__ == "__main__":
    main()
