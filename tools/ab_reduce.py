#!/usr/bin/env python
"""Time fixup-heavy shapes (graph replays); SKPP_PKG_ROOT=<dir> times another build of the package (A/B)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("SKPP_PKG_ROOT"):  # A/B against another build of the package
    sys.path.insert(0, os.environ["SKPP_PKG_ROOT"])


def main():
    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import sweep
    from tools.profile_gemm import parse_policy

    cases = [(512, 512, 16384, "ask", "128x128x64"), (512, 512, 16384, "ask", "256x256x64"),
             (512, 512, 16384, "ask", "256x128x64"), (1024, 1024, 1024, "ask", "128x128x64"),
             (1024, 1024, 1024, "hybrid1", "256x256x64"), (128, 4096, 4096, "ask", "128x128x64"),
             (2048, 2048, 2048, "hybrid1", "128x128x64"), (256, 14336, 4096, "ask", "256x256x64")]
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    params = sweep.MeasureParams(warmup=5, reps=25)
    for m, n, k, pol, t in cases:
        tile = sk.TileShape(*(int(v) for v in t.split("x")))
        a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        b = torch.randn(k, n, device="cuda").to(torch.bfloat16)
        c = torch.empty(m, n, device="cuda")
        plan = sk.GemmPlan(a, b, c, parse_policy(sk, pol), tile)
        res = [f"{sweep.time_plan(plan, params):7.2f} us" for _ in range(reps)]
        print(f"{m}x{n}x{k} {pol:8s} {t:11s} " + "  ".join(res), flush=True)


if __name__ == "__main__":
    main()
