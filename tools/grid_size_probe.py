"""Per-launch time of fixup-bound shapes as a function of the persistent grid size g (the
reference's HardwareModel.num_cus x occupancy), bench protocol: back-to-back launches over rotating
operand sets larger than L2, one event pair.  Every (tile, policy, g) schedule is the reference's
schedule for that g; g only changes how the MAC iterations are split.

usage: python tools/grid_size_probe.py   (one JSON line per (shape, tile, policy, g))
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2408_11417_b200 as sk

SHAPES = [(16, 4096, 4096), (128, 4096, 4096), (512, 512, 16384), (1024, 1024, 1024)]
TILES = ["128x128x128", "128x64x128"]
POLICIES = {"hybrid1": sk.Policy.hybrid(1), "all-streamk": sk.Policy.all_stream_k()}
GS = [148, 144, 128, 112, 96, 74, 64]


def main() -> None:
    torch.cuda.set_device(0)
    for m, n, k in SHAPES:
        sets = min(64, max(2, (512 << 20) // (2 * (m * k + k * n) + 4 * m * n)))
        ops = [(torch.randn(m, k, device="cuda").to(torch.bfloat16), torch.randn(k, n, device="cuda").to(torch.bfloat16),
                torch.empty(m, n, device="cuda")) for _ in range(sets)]
        steps = max(sets, 1000 // sets * sets)
        for tl in TILES:
            tile = sk.TileShape(*(int(v) for v in tl.split("x")))
            for pname, pol in POLICIES.items():
                for g in GS:
                    plans = [sk.GemmPlan(a, b, c, pol, tile, g) for a, b, c in ops]
                    for p in plans * 2:
                        p.launch()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for i in range(steps):
                        plans[i % sets].launch()
                    e1.record()
                    torch.cuda.synchronize()
                    us = e0.elapsed_time(e1) * 1e3 / steps
                    print(json.dumps({"m": m, "n": n, "k": k, "tile": tl, "policy": pname, "g": g,
                                      "us": round(us, 3)}), flush=True)


if __name__ == "__main__":
    main()
