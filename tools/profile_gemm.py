#!/usr/bin/env python
"""Launch one Stream-K++ GEMM repeatedly (no graphs) — a short target for ncu.

    ncu --set full -k regex:streamk_gemm -s 3 -c 1 -o prof python tools/profile_gemm.py --m 512 --n 512 --k 16384
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def parse_policy(sk, name: str):
    name = name.lower()
    if name in ("dp", "data-parallel"):
        return sk.Policy.data_parallel()
    if name in ("ask", "all-streamk", "sk"):
        return sk.Policy.all_stream_k()
    if name.startswith("hybrid"):
        rest = name[len("hybrid"):]
        first = not rest.endswith("-dpfirst")
        return sk.Policy.hybrid(int(rest.replace("-dpfirst", "")), first)
    raise SystemExit(f"unknown policy {name}")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=512)
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--k", type=int, default=16384)
    ap.add_argument("--tile", default="128x128x64")
    ap.add_argument("--policy", default="ask")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--out", default="fp32")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--flush", action="store_true", help="write 256 MiB between launches")
    ap.add_argument("--b3d", type=int, default=1, help="one 3-D TMA box for B per stage")
    args = ap.parse_args()

    import torch

    import paper_2408_11417_b200 as sk

    from paper_2408_11417_b200 import _lib

    if os.environ.get("SKPP_DEBUG"):
        _lib.lib.skpp_set_debug(int(os.environ["SKPP_DEBUG"]))
    if os.environ.get("SKPP_L2_HINTS"):
        _lib.lib.skpp_set_l2_hints(int(os.environ["SKPP_L2_HINTS"]))

    _lib.lib.skpp_set_b3d(args.b3d)
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float16
    od = {"fp32": torch.float32, "bf16": torch.bfloat16, "fp16": torch.float16}[args.out]
    tile = sk.tiles.parse_tile(args.tile)  # "MxNxK" or "MxNxKbG" (banded tile order)
    a = torch.randn(args.m, args.k, device="cuda").to(dt)
    b = torch.randn(args.k, args.n, device="cuda").to(dt)
    c = torch.empty(args.m, args.n, device="cuda", dtype=od)
    plan = sk.GemmPlan(a, b, c, parse_policy(sk, args.policy), tile)
    flush = torch.empty(64 << 20, device="cuda") if args.flush else None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.iters)]
    for i in range(args.iters):
        if flush is not None:
            flush.zero_()
        ev[2 * i].record()
        plan.launch()
        ev[2 * i + 1].record()
    torch.cuda.synchronize()
    us = [ev[2 * i].elapsed_time(ev[2 * i + 1]) * 1e3 for i in range(args.iters)]
    fl = 2.0 * args.m * args.n * args.k
    best = min(us)
    print(f"{args.m}x{args.n}x{args.k} {args.policy} tile {args.tile} b3d={args.b3d}: min {best:.2f} us "
          f"median {sorted(us)[len(us)//2]:.2f} us -> {fl / best / 1e6:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
