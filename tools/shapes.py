#!/usr/bin/env python
"""Per-shape TFLOP/s of every canonical policy on one B200 (CUDA-graph timing, L2 warm or flushed).

Writes one JSON object per shape to stdout; used for the BASELINE config table.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {
    "cfg1": [(1024, 1024, 1024)],
    "cfg2": [(512, 512, 16384)],
    "square": [(4096, 4096, 4096), (8192, 8192, 8192)],
    "llama": [(m, n, 4096) for m in (1, 16, 64, 128, 256, 512, 1024, 2048, 4096, 8192) for n in (4096, 14336)],
}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="cfg1,cfg2,square,llama")
    ap.add_argument("--tiles", default="128x128x64,128x256x64")
    ap.add_argument("--dtype", default="bf16")
    args = ap.parse_args()

    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import sweep

    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float16
    shapes = [s for name in args.set.split(",") for s in SHAPES[name]]
    sizes = [sk.ProblemSize(*s) for s in shapes]
    pool = sweep.OperandPool(sizes, dt, torch.float32)
    params = sweep.MeasureParams(warmup=3, reps=10, in_dtype=dt)
    for tile_s in args.tiles.split(","):
        tile = sk.TileShape(*(int(v) for v in tile_s.split("x")))
        g = sk.executor.default_g(tile)
        for size in sizes:
            rec = sweep.measure_size(size, tile, g, sk.canonical_policies(), params, pool)
            out = {
                "m": size.m, "n": size.n, "k": size.k, "tile": tile_s,
                "tflops": {p.label: round(size.flops / (e.makespan * 1e-6) / 1e12, 1) for p, e in rec.costs},
                "us": {p.label: round(e.makespan, 2) for p, e in rec.costs},
                "winner": rec.winner.label,
                "dp_utilization": round(sk.dp_utilization(sk.grid_info(size, tile), g), 3),
            }
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
