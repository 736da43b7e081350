#!/usr/bin/env python
"""A/B of skpp_set_raster (G-row tile bands) vs the reference row-major order: bitwise
equality of C, then bench-style timing (rotating operand sets), interleaved rounds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import _lib
    from tools.profile_gemm import parse_policy

    cases = [(8192, 8192, 8192, "dp", "256x256x128"), (4096, 14336, 4096, "dp", "256x256x128"),
             (4096, 14336, 4096, "hybrid1", "256x256x128"), (4096, 4096, 4096, "dp", "256x256x128"),
             (2048, 14336, 4096, "hybrid1", "256x256x128"), (8192, 8192, 8192, "dp", "128x256x64"),
             (1000, 3000, 5000, "hybrid1", "128x128x64"), (512, 512, 16384, "hybrid1", "128x128x128")]
    rasters = [int(v) for v in os.environ.get("RASTERS", "0,4,8,16").split(",")]
    for m, n, k, pol, t in cases:
        tile = sk.TileShape(*(int(v) for v in t.split("x")))
        policy = parse_policy(sk, pol)
        set_bytes = 2 * (m * k + k * n) + 2 * m * n
        sets = max(2, min(32, (512 << 20) // set_bytes))
        ops = [(torch.randn(m, k, device="cuda").to(torch.bfloat16), torch.randn(k, n, device="cuda").to(torch.bfloat16),
                torch.empty(m, n, device="cuda", dtype=torch.bfloat16)) for _ in range(sets)]
        ref = None
        for r in rasters:
            _lib.lib.skpp_set_raster(r)
            a, b, _ = ops[0]
            c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            sk.GemmPlan(a, b, c, policy, tile).launch()
            torch.cuda.synchronize()
            if ref is None:
                ref = c
            elif not torch.equal(ref, c):
                print(f"MISMATCH raster={r} {m}x{n}x{k} {pol} {t}", flush=True)
        flops = 2.0 * m * n * k
        steps = max(sets, int(min(2000, max(20, 0.2e6 / (flops / 1e12 / 1000 * 1e6 + 5)))) // sets * sets)
        res = {}
        for rnd in range(3):
            for r in rasters:
                _lib.lib.skpp_set_raster(r)
                plans = [sk.GemmPlan(a, b, c, policy, tile) for a, b, c in ops]
                for p in plans * 2:
                    p.launch()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for i in range(steps):
                    plans[i % sets].launch()
                e1.record()
                torch.cuda.synchronize()
                res.setdefault(r, []).append(e0.elapsed_time(e1) * 1e3 / steps)
        _lib.lib.skpp_set_raster(0)
        line = " ".join(f"G{r}: {sorted(v)[1]:8.2f}us ({flops / sorted(v)[1] / 1e6:6.1f}TF)" for r, v in res.items())
        print(f"{m}x{n}x{k} {pol} {t}: {line}", flush=True)


if __name__ == "__main__":
    main()
