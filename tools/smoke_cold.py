"""smoke()'s exact sequence in a fresh process (DP, hybrid1, all-streamk on 384x256x1536,
tile 128x128x64), without asserting: on a mismatch print the differing C blocks/rows and the
fixup workspace's control block (epoch header, started/abandon counters, band states, flags).

usage: python tools/smoke_cold.py [--timeline]   (one JSON line)
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2408_11417_b200 as sk
from paper_2408_11417_b200 import executor
from oracle import gemm as ogemm


def main() -> None:
    torch.cuda.set_device(0)
    m, n, k = 384, 256, 1536
    rng = np.random.default_rng(2024)
    a = ogemm.random_int_matrix(m, k, rng)
    b = ogemm.random_int_matrix(k, n, rng)
    want = ogemm.reference_gemm(a, b)
    tile = sk.TileShape(128, 128, 64)
    at = torch.from_numpy(a).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
    out = {}
    for pol in (sk.Policy.data_parallel(), sk.Policy.hybrid(1), sk.Policy.all_stream_k()):
        c = torch.empty(m, n, dtype=torch.float32, device="cuda")
        plan = sk.GemmPlan(at, bt, c, pol, tile, trace_cap=16)
        plan.launch()
        torch.cuda.synchronize()
        got = c.double().cpu().numpy()
        rec = {"ok": bool(np.array_equal(got, want)), "g": plan.g}
        if not rec["ok"]:
            bad = got != want
            blocks = []
            for tm in range(3):
                for tn in range(2):
                    blk = bad[tm * 128:(tm + 1) * 128, tn * 128:(tn + 1) * 128]
                    if blk.any():
                        rows = np.nonzero(blk.any(axis=1))[0].tolist()
                        cols = np.nonzero(blk.any(axis=0))[0].tolist()
                        blocks.append({"tile": [tm, tn], "rows": rows, "ncols": len(cols),
                                       "max_abs": float(np.abs(got - want)[tm * 128:(tm + 1) * 128,
                                                                          tn * 128:(tn + 1) * 128].max())})
            rec["blocks"] = blocks
            if plan.ws_bytes:
                ws = next(iter(plan._ws_cache.values()))[2]
                ctl = ws[:32768].view(torch.int32).cpu().numpy()
                rec["hdr"] = ctl[:32].tolist()
                flags = ctl[256:256 + 2 * plan.g]
                rec["flags_distinct"] = sorted(set(int(v) for v in flags))
                st = ctl[(1024 + 8192) // 4:(1024 + 8192) // 4 + 2048]
                rec["bstate_nonzero"] = [(i, int(v)) for i, v in enumerate(st) if v != 0][:64]
        out[pol.label] = rec
    print(json.dumps(out))


if __name__ == "__main__":
    main()
