#!/usr/bin/env python
"""Per-step time of cfg2 under three launch modes: isolated (flush + event pair),
back-to-back stream launches over rotating operand sets, and a CUDA graph of
the rotating launches replayed.  PDL on/off for the last two."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("SKPP_PKG_ROOT"):  # A/B against another build of the package
    sys.path.insert(0, os.environ["SKPP_PKG_ROOT"])


def main():
    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import _lib

    if os.environ.get("SKPP_PF"):
        _lib.lib.skpp_set_l2_prefetch(int(os.environ["SKPP_PF"]))
    if os.environ.get("SKPP_A3D"):
        _lib.lib.skpp_set_a3d(int(os.environ["SKPP_A3D"]))
    if os.environ.get("SKPP_DEBUG"):
        _lib.lib.skpp_set_debug(int(os.environ["SKPP_DEBUG"]))
    if os.environ.get("SKPP_L2_HINTS"):
        _lib.lib.skpp_set_l2_hints(int(os.environ["SKPP_L2_HINTS"]))
    from tools.profile_gemm import parse_policy

    m, n, k = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (512, 512, 16384)))
    pol = sys.argv[4] if len(sys.argv) > 4 else "ask"
    tile = sk.TileShape(*(int(v) for v in (sys.argv[5] if len(sys.argv) > 5 else "128x128x64").split("x")))
    sets = min(64, max(2, (512 << 20) // (2 * (m * k + k * n) + 4 * m * n)))
    ops = [(torch.randn(m, k, device="cuda").to(torch.bfloat16), torch.randn(k, n, device="cuda").to(torch.bfloat16),
            torch.empty(m, n, device="cuda")) for _ in range(sets)]
    steps = 2000 // sets * sets
    for pdl in (1, 0):
        _lib.lib.skpp_set_pdl(pdl)
        plans = [sk.GemmPlan(a, b, c, parse_policy(sk, pol), tile) for a, b, c in ops]
        for p in plans * 3:
            p.launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            plans[i % sets].launch()
        e1.record()
        torch.cuda.synchronize()
        stream_us = e0.elapsed_time(e1) * 1e3 / steps
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                for p in plans:
                    p.launch()
        torch.cuda.current_stream().wait_stream(side)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps // sets):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph_us = e0.elapsed_time(e1) * 1e3 / steps
        print(f"{m}x{n}x{k} {pol} {sys.argv[5] if len(sys.argv) > 5 else '128x128x64'} sets={sets} pdl={pdl}: "
              f"stream {stream_us:.2f} us/step  graph {graph_us:.2f} us/step", flush=True)


if __name__ == "__main__":
    main()
