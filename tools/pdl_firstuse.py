"""Can a GEMM launched with programmatic dependent launch read an operand before the torch kernel
that wrote it (the first use of that kernel in the process) has finished?

In a fresh process, each event writes A with a torch kernel used for the first time and launches a
data-parallel GEMM (no fixup workspace) right behind it, then checks C against float64.
usage: python tools/pdl_firstuse.py   (one JSON line: per event ok)
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2408_11417_b200 as sk


def main() -> None:
    torch.cuda.set_device(0)
    m, n, k = 384, 256, 1536
    rng = np.random.default_rng(7)
    a = rng.integers(-8, 9, size=(m, k)).astype(np.float32)
    b = rng.integers(-8, 9, size=(k, n)).astype(np.float32)
    want = torch.from_numpy(a.astype(np.float64) @ b.astype(np.float64)).cuda()
    af = torch.from_numpy(a).cuda()
    bt = torch.from_numpy(b).cuda().to(torch.bfloat16)
    bh = torch.from_numpy(b).cuda().to(torch.float16)
    tile = sk.TileShape(128, 128, 64)
    events = {
        "f32_to_bf16": lambda: af.to(torch.bfloat16),
        "f32_to_f16": lambda: af.half(),
        "mul_then_bf16": lambda: (af * 1.0).to(torch.bfloat16),
        "neg_neg_bf16": lambda: torch.neg(torch.neg(af)).to(torch.bfloat16),
        "where_bf16": lambda: torch.where(af > 100.0, af, af).to(torch.bfloat16),
    }
    out = {}
    for name, make in events.items():
        c = torch.empty(m, n, device="cuda")
        torch.cuda.synchronize()
        at = make()  # first use of this kernel in the process, then the PDL GEMM right behind it
        plan = sk.GemmPlan(at, bh if at.dtype == torch.float16 else bt, c, sk.Policy.data_parallel(), tile)
        plan.launch()
        torch.cuda.synchronize()
        out[name] = bool(torch.equal(c.double(), want))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
