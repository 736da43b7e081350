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

    sizes = [sk.ProblemSize(*v) for v in [(8192, 2048, 32), (8192, 1024, 512), (1024, 1024, 1024),
                                          (8192, 2048, 65536), (8192, 8192, 65536), (64, 64, 64)]]
    params = sweep.MeasureParams(warmup=3, reps=10)
    pool = sweep.OperandPool(sizes, params.in_dtype, params.out_dtype)
    for tile in (sk.TileShape(128, 128, 128), sk.TileShape(256, 256, 128)):
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
