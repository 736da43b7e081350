#!/usr/bin/env python
"""Which H2D copy is slow: A alone, B alone, A then B, B then A (pinned host bf16, 16 MiB each)."""
import sys
import time

import torch

sys.path.insert(0, ".")


def t_us(fn, n=20):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


a_h = torch.randn(512, 16384).to(torch.bfloat16).pin_memory()
b_h = torch.randn(16384, 512).to(torch.bfloat16).pin_memory()
print("pinned:", a_h.is_pinned(), b_h.is_pinned())
a_d = torch.empty_like(a_h, device="cuda")
b_d = torch.empty_like(b_h, device="cuda")
print("A      %.1f us" % t_us(lambda: a_d.copy_(a_h, non_blocking=True)))
print("B      %.1f us" % t_us(lambda: b_d.copy_(b_h, non_blocking=True)))
print("A,B    %.1f us" % t_us(lambda: (a_d.copy_(a_h, non_blocking=True), b_d.copy_(b_h, non_blocking=True))))
print("B,A    %.1f us" % t_us(lambda: (b_d.copy_(b_h, non_blocking=True), a_d.copy_(a_h, non_blocking=True))))
big_h = torch.empty(2 * a_h.numel(), dtype=torch.bfloat16).pin_memory()
big_d = torch.empty_like(big_h, device="cuda")
print("1x32MB %.1f us" % t_us(lambda: big_d.copy_(big_h, non_blocking=True)))
s2 = torch.cuda.Stream()
def two():
    ev = torch.cuda.Event()
    with torch.cuda.stream(s2):
        b_d.copy_(b_h, non_blocking=True)
        ev.record(s2)
    a_d.copy_(a_h, non_blocking=True)
    torch.cuda.current_stream().wait_event(ev)
print("A|B 2 streams %.1f us" % t_us(two))
