#!/usr/bin/env python
"""Per-CTA phase timeline of two consecutive launches in the bench's steady state.

The bench times K back-to-back launches over rotating operand sets (cold L2, PDL overlap
between launches).  This records the %globaltimer stamps (skpp_debug_timeline) of launches
S-1 and S of such a sequence, so the critical path of a step — previous grid's tail, this
grid's start, mainloop, partial publish, flag wait, reduction, end — can be read off, all
relative to the first CTA start of launch S-1.

    python tools/steady_timeline.py --m 16 --n 4096 --k 4096 --tile 128x128x128 --policy hybrid1
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

NEV = 32  # TL_EVENTS (skpp_gemm.cu)
EV = {"entry": 21, "start": 0, "first_tma": 1, "first_full": 2, "mma_done": 3, "phase1": 4, "waited": 5, "phase2": 6, "end": 7,
      "epi_first": 8, "part_issued": 9, "part_flag": 10, "sum1": 11, "sum2": 12, "p2_stored": 16, "p2_loop": 18}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--tile", default="128x128x128")
    ap.add_argument("--policy", default="hybrid1")
    ap.add_argument("--steps", type=int, default=40)
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import _lib
    from tools.profile_gemm import parse_policy

    if os.environ.get("SKPP_DEBUG"):
        _lib.lib.skpp_set_debug(int(os.environ["SKPP_DEBUG"]))
    for kv in filter(None, os.environ.get("SKPP_SET", "").split(",")):  # e.g. SKPP_SET=l2_prefetch=4,pdl=0
        name, val = kv.split("=")
        getattr(_lib.lib, "skpp_set_" + name)(int(val))
    from paper_2408_11417_b200.tiles import parse_tile

    tile = parse_tile(args.tile)  # "256x256x128b16" = banded tile order 16
    m, n, k = args.m, args.n, args.k
    set_bytes = 2 * (m * k + k * n) + 4 * m * n
    n_sets = max(2, -(-(512 << 20) // set_bytes))
    pol = parse_policy(sk, args.policy)
    plans = [sk.GemmPlan(torch.randn(m, k, device="cuda").to(torch.bfloat16),
                         torch.randn(k, n, device="cuda").to(torch.bfloat16),
                         torch.empty(m, n, device="cuda"), pol, tile) for _ in range(n_sets)]
    grid = plans[0].g * (tile.blk_m // 128)
    bufs = [torch.zeros(grid * NEV + 512, dtype=torch.int64, device="cuda") for _ in range(2)]
    for i in range(50):
        plans[i % n_sets].launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        if i == args.steps - 2:
            _lib.lib.skpp_debug_timeline(bufs[0].data_ptr())
        elif i == args.steps - 1:
            _lib.lib.skpp_debug_timeline(bufs[1].data_ptr())
        plans[i % n_sets].launch()
    e1.record()
    _lib.lib.skpp_debug_timeline(None)
    torch.cuda.synchronize()
    us_step = e0.elapsed_time(e1) * 1e3 / args.steps
    raw = [b.cpu().numpy().astype(np.float64) for b in bufs]
    t = [r[: grid * NEV].reshape(grid, NEV) for r in raw]
    base = t[0][:, 0][t[0][:, 0] > 0].min()
    print(f"{m}x{n}x{k} {args.policy} tile {args.tile}: "
          f"{us_step:.2f} us/step over {args.steps} back-to-back launches ({n_sets} operand sets)")
    for li, tt in enumerate(t):
        print("  launch S-1" if li == 0 else "  launch S")
        for name, i in EV.items():
            col = tt[:, i]
            col = col[col > 0]
            if len(col):
                col = (col - base) / 1e3
                print(f"    {name:>11}: min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
    for li, tt in enumerate(t):
        pro = [tt[:, c] for c in (25, 26, 28, 27)]
        if all((v > 0).any() for v in pro):
            print(f"  launch {'S-1' if li == 0 else 'S'} prologue (SM cycles since entry, med/max): "
                  + ", ".join(f"{nm} {np.median(v[v > 0]):.0f}/{v.max():.0f}"
                              for nm, v in zip(("barriers", "tmem+sync", "decoded", "prefetched"), pro)))
        c_tma = tt[:, 22]
        if (c_tma > 0).any():
            print(f"  launch {'S-1' if li == 0 else 'S'}: SM cycles griddepcontrol.wait -> first A load "
                  f"med {np.median(c_tma[c_tma > 0]):.0f} max {c_tma.max():.0f}")
    for li, tt in enumerate(t):
        bs = tt[:, 13:16]
        okb = (bs[:, 0] > 0) & (bs[:, 1] > 0) & (bs[:, 2] > 0)
        if okb.any():
            lat, tot = bs[okb, 1] - bs[okb, 0], bs[okb, 2] - bs[okb, 0]
            print(f"  launch {'S-1' if li == 0 else 'S'} band_sum (thread 128, SM cycles): first loads back med "
                  f"{np.median(lat):.0f} max {lat.max():.0f}; whole pass med {np.median(tot):.0f} max {tot.max():.0f}")
    ks = raw[1][grid * NEV: grid * NEV + 512].reshape(256, 2)  # CTA 0 of launch S: (issue, arrival) clock64
    nk = int((ks[:, 1] > 0).sum())
    if nk:
        c0 = t[1][0, 24]  # clock64 at CTA 0's entry
        print("  launch S, CTA 0 k-blocks (SM cycles since entry: issue / arrival / latency): " + "; ".join(
            f"{k}: {ks[k, 0] - c0:.0f}/{ks[k, 1] - c0:.0f}/{ks[k, 1] - ks[k, 0]:.0f}" for k in range(min(nk, 16))))
    end_prev = (t[0][:, 7][t[0][:, 7] > 0].max() - base) / 1e3
    start_next = (t[1][:, 0][t[1][:, 0] > 0].min() - base) / 1e3
    start_next_med = (np.median(t[1][:, 0][t[1][:, 0] > 0]) - base) / 1e3
    print(f"  S-1 last CTA end {end_prev:.2f} us; S first CTA past griddepcontrol.wait {start_next:.2f} us "
          f"(median {start_next_med:.2f}); S-1 -> S start to start "
          f"{(t[1][:, 0][t[1][:, 0] > 0].min() - base) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
