#!/usr/bin/env python
"""Host-side cost of one GemmPlan.launch() vs a torch kernel launch (no sync in the loop)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2408_11417_b200 as sk

    a = torch.randn(128, 64, device="cuda").to(torch.bfloat16)
    b = torch.randn(64, 128, device="cuda").to(torch.bfloat16)
    c = torch.empty(128, 128, device="cuda")
    from paper_2408_11417_b200 import _lib

    for pdl, pol in [(p, q) for p in (0, 1) for q in (sk.Policy.data_parallel(), sk.Policy.all_stream_k())]:
        _lib.lib.skpp_set_pdl(pdl)
        plan = sk.GemmPlan(a, b, c, pol)
        for _ in range(20):
            plan.launch()
        torch.cuda.synchronize()
        n = 2000
        t0 = time.perf_counter()
        for _ in range(n):
            plan.launch()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"pdl={pdl} {pol.label}: host {1e6 * (t1 - t0) / n:.2f} us/launch, device-bound {1e6 * (t2 - t0) / n:.2f} us/launch")
    x = torch.empty(1024, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        x.add_(1.0)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"torch add_: host {1e6 * (t1 - t0) / 2000:.2f} us/launch")


if __name__ == "__main__":
    main()
