#!/usr/bin/env python
"""Where the end-to-end execute_schedule time goes (host operands -> device GEMM -> host result)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def t_us(fn, n=20):
    import torch
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


def main():
    import torch

    import paper_2408_11417_b200 as sk

    m, n, k = 512, 512, 16384
    a_h = torch.randn(m, k).to(torch.bfloat16).pin_memory()
    b_h = torch.randn(k, n).to(torch.bfloat16).pin_memory()
    a_d = a_h.cuda()
    b_d = b_h.cuda()
    c_d = torch.empty(m, n, device="cuda")
    c_h = torch.empty(m, n).pin_memory()
    size, tile = sk.ProblemSize(m, n, k), sk.TileShape(128, 128, 128)
    pol = sk.Policy.hybrid(1)
    sched = sk.build_schedule(size, tile, sk.HardwareModel(148, 1), pol)
    print("H2D A+B pinned      %.1f us" % t_us(lambda: (a_d.copy_(a_h, non_blocking=True), b_d.copy_(b_h, non_blocking=True))))
    s2 = torch.cuda.Stream()
    def two_streams():
        ev = torch.cuda.Event()
        with torch.cuda.stream(s2):
            b_d.copy_(b_h, non_blocking=True)
            ev.record(s2)
        a_d.copy_(a_h, non_blocking=True)
        torch.cuda.current_stream().wait_event(ev)
    print("H2D A|B two streams %.1f us" % t_us(two_streams))
    print("D2H C pageable      %.1f us" % t_us(lambda: c_d.cpu()))
    print("D2H C pinned        %.1f us" % t_us(lambda: c_h.copy_(c_d, non_blocking=True)))
    print("GemmPlan create     %.1f us" % t_us(lambda: sk.GemmPlan(a_d, b_d, c_d, pol, tile, 148)))
    plan = sk.GemmPlan(a_d, b_d, c_d, pol, tile, 148)
    print("launch only         %.1f us" % t_us(lambda: plan.launch(), 200))
    print("execute_schedule    %.1f us" % t_us(lambda: sk.execute_schedule(a_h, b_h, sched, tile, size)))


if __name__ == "__main__":
    main()
