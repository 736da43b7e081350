#!/usr/bin/env python
"""Every canonical policy of one (size, tile), timed bench-style (K back-to-back launches
over rotating operand sets > L2), interleaved over rounds.  argv: M N K TILE [ROUNDS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    import paper_2408_11417_b200 as sk

    m, n, k = (int(v) for v in sys.argv[1:4])
    tile = sk.TileShape(*(int(v) for v in sys.argv[4].split("x")))
    rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    set_bytes = 2 * (m * k + k * n) + 2 * m * n
    sets = max(2, min(32, (512 << 20) // set_bytes))
    ops = [(torch.randn(m, k, device="cuda").to(torch.bfloat16), torch.randn(k, n, device="cuda").to(torch.bfloat16),
            torch.empty(m, n, device="cuda", dtype=torch.bfloat16)) for _ in range(sets)]
    flops = 2.0 * m * n * k
    steps = max(sets, int(min(2000, max(20, 0.2e6 / (flops / 1e12 / 1000 * 1e6 + 5)))) // sets * sets)
    res = {}
    for r in range(rounds):
        for pol in sk.canonical_policies():
            plans = [sk.GemmPlan(a, b, c, pol, tile) for a, b, c in ops]
            for p in plans * 2:
                p.launch()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(steps):
                plans[i % sets].launch()
            e1.record()
            torch.cuda.synchronize()
            res.setdefault(pol.label, []).append(e0.elapsed_time(e1) * 1e3 / steps)
    for lab, v in res.items():
        v = sorted(v)
        print(f"{m}x{n}x{k} {sys.argv[4]} {lab:14s} med {v[len(v) // 2]:9.2f} us  min {v[0]:9.2f}  "
              f"{flops / v[len(v) // 2] / 1e6:7.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
