#!/usr/bin/env python
"""execute_schedule with host operands: concurrent A|B upload (current) vs sequential, interleaved."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2408_11417_b200 as sk  # noqa: E402
from paper_2408_11417_b200 import executor as ex  # noqa: E402

m, n, k = 512, 512, 16384
a_h = torch.randn(m, k).to(torch.bfloat16).pin_memory()
b_h = torch.randn(k, n).to(torch.bfloat16).pin_memory()
size, tile = sk.ProblemSize(m, n, k), sk.TileShape(128, 128, 128)
sched = sk.build_schedule(size, tile, sk.HardwareModel(148, 1), sk.Policy.hybrid(1))
concurrent = ex._upload_pair


def sequential(a, b, dev):
    return a.to(f"cuda:{dev}", non_blocking=True), b.to(f"cuda:{dev}", non_blocking=True)


res = {"concurrent": [], "sequential": []}
for rnd in range(6):
    for name, fn in (("concurrent", concurrent), ("sequential", sequential)):
        ex._upload_pair = fn
        for _ in range(5):
            sk.execute_schedule(a_h, b_h, sched, tile, size)
        ts = []
        for _ in range(40):
            t0 = time.perf_counter()
            sk.execute_schedule(a_h, b_h, sched, tile, size)
            ts.append(time.perf_counter() - t0)
        res[name].append(statistics.median(ts) * 1e6)
for name, v in res.items():
    print(f"{name:10s} median per call (us) by round: " + " ".join(f"{x:7.1f}" for x in v))
