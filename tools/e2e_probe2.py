#!/usr/bin/env python
"""H2D variants for execute_schedule's host-operand path (cfg2 operands, 2 x 16 MiB pinned)."""
import sys
import time

import torch

sys.path.insert(0, '.')


def t_us(fn, n=30):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


m, n, k = 512, 512, 16384
a_h = torch.randn(m, k).to(torch.bfloat16).pin_memory()
b_h = torch.randn(k, n).to(torch.bfloat16).pin_memory()
a_d = torch.empty_like(a_h, device="cuda")
b_d = torch.empty_like(b_h, device="cuda")
print("to(cuda) x2          %.1f us" % t_us(lambda: (a_h.to("cuda", non_blocking=True), b_h.to("cuda", non_blocking=True))))
print("copy_ prealloc x2    %.1f us" % t_us(lambda: (a_d.copy_(a_h, non_blocking=True), b_d.copy_(b_h, non_blocking=True))))
print("empty+copy_ x2       %.1f us" % t_us(lambda: (torch.empty_like(a_h, device="cuda").copy_(a_h, non_blocking=True),
                                                    torch.empty_like(b_h, device="cuda").copy_(b_h, non_blocking=True))))
print("to(cuda) A only      %.1f us" % t_us(lambda: a_h.to("cuda", non_blocking=True)))
print("copy_ A only         %.1f us" % t_us(lambda: a_d.copy_(a_h, non_blocking=True)))
print("cudaMemcpyAsync-like %.1f us" % t_us(lambda: torch.cuda.current_stream() and a_d.copy_(a_h, non_blocking=True)))
