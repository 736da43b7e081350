#!/usr/bin/env python
"""Wall time of sweep.measure_size for a few sizes, repeated (finds slow measurement paths)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import sweep

    spec = os.environ.get("SIZES", "8192x2048x32,8192x1024x512,1024x1024x1024,4x4096x1024,64x64x64")
    sizes = [sk.ProblemSize(*(int(v) for v in z.split("x"))) for z in spec.split(",")]
    tiles = [sk.TileShape(*(int(v) for v in t.split("x")))
             for t in os.environ.get("TILES", "128x128x128,256x256x128").split(",")]
    params = sweep.MeasureParams(warmup=3, reps=10)
    pool = sweep.OperandPool(sizes, params.in_dtype, params.out_dtype)
    for tile in tiles:
        g = sk.executor.default_g(tile)
        for size in sizes:
            ts = []
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rec = sweep.measure_size(size, tile, g, sk.canonical_policies(), params, pool)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            us = {p.label: round(e.makespan, 1) for p, e in rec.costs}
            print(tile.blk_m, tile.blk_n, tile.blk_k, size.m, size.n, size.k, [round(t, 3) for t in ts], us, flush=True)


if __name__ == "__main__":
    main()
