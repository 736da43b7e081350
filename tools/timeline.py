#!/usr/bin/env python
"""Per-CTA phase timeline of one Stream-K++ launch (skpp_debug_timeline, %globaltimer ns)."""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

EVENTS = ["start", "first_tma", "first_full", "mma_done", "phase1", "waited", "phase2", "end", "epi_first", "part_issued", "part_flag", "sum1", "sum2", "-", "-", "-",
          "p2_stored", "p2_synced", "p2_loop", "p2_clean", "waited0"]
NEV = 32  # TL_EVENTS


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=512)
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--k", type=int, default=16384)
    ap.add_argument("--tile", default="128x128x64")
    ap.add_argument("--policy", default="ask")
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--out", default="fp32", help="fp32 | bf16")
    ap.add_argument("--per-cta", type=int, default=0, help="print the first N CTAs")
    ap.add_argument("--kstamps", type=int, default=0, help="print CTA 0's first N k-block stamps")
    args = ap.parse_args()

    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import _lib

    if os.environ.get("SKPP_DEBUG"):
        _lib.lib.skpp_set_debug(int(os.environ["SKPP_DEBUG"]))
    from tools.profile_gemm import parse_policy

    from paper_2408_11417_b200.tiles import parse_tile

    tile = parse_tile(args.tile)  # "256x256x128b16" = banded tile order 16
    a = torch.randn(args.m, args.k, device="cuda").to(torch.bfloat16)
    b = torch.randn(args.k, args.n, device="cuda").to(torch.bfloat16)
    c = torch.empty(args.m, args.n, device="cuda",
                    dtype=torch.bfloat16 if args.out == "bf16" else torch.float32)
    plan = sk.GemmPlan(a, b, c, parse_policy(sk, args.policy), tile)
    grid = plan.g * (tile.blk_m // 128)
    tl = torch.zeros(grid * NEV + 512, dtype=torch.int64, device="cuda")
    flush = torch.empty(64 << 20, device="cuda")
    for _ in range(3):
        plan.launch()
    if args.flush:
        flush.zero_()
        flush.sum()
    torch.cuda.synchronize()
    _lib.lib.skpp_debug_timeline(tl.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.launch()
    e1.record()
    torch.cuda.synchronize()
    _lib.lib.skpp_debug_timeline(None)
    raw = tl.cpu().numpy().astype("float64")
    t = raw[: grid * NEV].reshape(grid, NEV)
    ks = raw[grid * NEV:].reshape(256, 2)
    base = t[:, 0][t[:, 0] > 0].min()
    print(f"{args.m}x{args.n}x{args.k} {args.policy} tile {args.tile} flush={args.flush}: "
          f"event time {e0.elapsed_time(e1) * 1e3:.1f} us, "
          f"kernel span {(t[:, :13].max() - base) / 1e3:.2f} us")
    for i, name in enumerate(EVENTS):
        if name == "-":
            continue
        col = t[:, i]
        col = col[col > 0] - base
        if len(col):
            print(f"  {name:>10}: min {col.min() / 1e3:8.2f}  med {sorted(col)[len(col) // 2] / 1e3:8.2f}  "
                  f"max {col.max() / 1e3:8.2f} us  (n={len(col)})")
    bs = t[:, 13:16]
    ok = (bs[:, 0] > 0) & (bs[:, 1] > 0) & (bs[:, 2] > 0)
    if ok.any():
        lat, tot = bs[ok, 1] - bs[ok, 0], bs[ok, 2] - bs[ok, 0]
        print(f"  band_sum (thread 128, SM cycles): first loads back med {sorted(lat)[len(lat) // 2]:.0f} "
              f"max {lat.max():.0f}; whole pass med {sorted(tot)[len(tot) // 2]:.0f} max {tot.max():.0f}  (n={ok.sum()})")
    if args.kstamps:
        n = int((ks[:, 1] > 0).sum())
        c0 = ks[0, 0]
        print(f"  CTA 0 k-blocks: {n}; SM cycles relative to the first issue:")
        for k in range(min(n, args.kstamps)):
            lat = ks[k, 1] - ks[k, 0]
            gap = ks[k, 1] - ks[k - 1, 1] if k else 0.0
            igap = ks[k, 0] - ks[k - 1, 0] if k else 0.0
            print(f"    k {k:3d}: issue {ks[k, 0] - c0:8.0f} (+{igap:5.0f}) arrive {ks[k, 1] - c0:8.0f} "
                  f"(+{gap:5.0f}) lat {lat:6.0f}")
        if n > 8:
            print(f"  mean arrival spacing k>=8: {(ks[n - 1, 1] - ks[8, 1]) / (n - 9):.0f} cycles")
    cols = [0, 3, 8, 10, 4, 20, 5, 11, 12, 16, 17, 18, 19, 6, 7]  # start mma_done epi_first part_flag phase1 waited0 waited sum1 sum2 p2_stored p2_synced p2_loop p2_clean phase2 end
    if args.per_cta:
        print("  cta      " + " ".join(f"{EVENTS[i][:7]:>7s}" for i in cols))
    for x in range(min(args.per_cta, grid)):
        row = [(t[x, i] - base) / 1e3 if t[x, i] > 0 else float('nan') for i in cols]
        print(f"  cta {x:3d}: " + " ".join(f"{v:7.2f}" for v in row))


if __name__ == "__main__":
    main()
