"""Repeat the smoke() GEMM (384x256x1536, tile 128x128x64, every CTA of a 148-CTA grid
taking one k-iteration) and count launches whose C differs from the float64 oracle.

usage: SKPP_LIB=... python tools/smoke_diag.py [--reps N] [--debug FLAGS] [--fresh-plan]
Prints one JSON line: failures per policy and, for the first failure, the differing
(tile_m, tile_n) blocks and row ranges.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2408_11417_b200 as sk
from paper_2408_11417_b200 import _lib
from oracle import gemm as ogemm


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--debug", type=int, default=0)
    ap.add_argument("--fresh-plan", action="store_true")
    ap.add_argument("--m", type=int, default=384)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--k", type=int, default=1536)
    ap.add_argument("--bk", type=int, default=64)
    args = ap.parse_args()
    if args.debug:
        _lib.lib.skpp_set_debug(args.debug)
    m, n, k = args.m, args.n, args.k
    rng = np.random.default_rng(2024)
    a = ogemm.random_int_matrix(m, k, rng)
    b = ogemm.random_int_matrix(k, n, rng)
    want = torch.from_numpy(ogemm.reference_gemm(a, b)).cuda()
    tile = sk.TileShape(128, 128, args.bk)
    at = torch.from_numpy(a).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
    out = {"lib": os.environ.get("SKPP_LIB", "in-tree"), "debug": args.debug, "reps": args.reps,
           "fresh_plan": args.fresh_plan}
    for pol in (sk.Policy.hybrid(1), sk.Policy.all_stream_k(), sk.Policy.hybrid(2)):
        c = torch.empty(m, n, dtype=torch.float32, device="cuda")
        plan = None
        fails, first = 0, None
        for r in range(args.reps):
            if plan is None or args.fresh_plan:
                plan = sk.GemmPlan(at, bt, c, pol, tile)
            c.fill_(float("nan"))
            plan.launch()
            torch.cuda.synchronize()
            bad = c.double() != want
            if bool(bad.any()):
                fails += 1
                if first is None:
                    blocks = []
                    for tm in range(-(-m // 128)):
                        for tn in range(-(-n // 128)):
                            blk = bad[tm * 128:(tm + 1) * 128, tn * 128:(tn + 1) * 128]
                            if bool(blk.any()):
                                rows = blk.any(dim=1).nonzero().flatten().tolist()
                                nan = bool(torch.isnan(c[tm * 128:(tm + 1) * 128, tn * 128:(tn + 1) * 128]).any())
                                blocks.append({"tile": [tm, tn], "rows": [rows[0], rows[-1]], "nrows": len(rows),
                                               "nan": nan})
                    first = {"rep": r, "blocks": blocks,
                             "max_abs": float((c.double() - want).abs().nan_to_num(1e30).max())}
        out[pol.label] = {"fails": fails, "first": first, "g": plan.g}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
