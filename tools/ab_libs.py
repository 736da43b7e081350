#!/usr/bin/env python
"""Same-box A/B of kernel builds: per shape, back-to-back launches over cold operand sets
(the bench's timed-region protocol), one subprocess per (library, round), libraries
interleaved round by round.  Prints one JSON line per shape with the median us per build.

    python tools/ab_libs.py --libs tools/ab_libs/libskpp_base.so,paper_2408_11417_b200/libskpp.so

An entry may carry a debug switch of the build: ``path@DEBUG`` calls skpp_set_debug(DEBUG) before
the plans are made.  SKPP_AB_CASES="m:n:k:tile:policy,..." replaces the default shapes.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(512, 512, 16384, "128x128x128", "hybrid1"), (16, 4096, 4096, "128x128x128", "hybrid1"),
         (128, 4096, 4096, "128x128x128", "hybrid1"), (1024, 1024, 1024, "128x128x64", "hybrid1"),
         (1024, 1024, 1024, "128x64x128", "data-parallel"), (8192, 14336, 4096, "256x256x128b16", "hybrid1")]


def worker(cases) -> None:
    sys.path.insert(0, ROOT)
    import torch

    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import _lib
    from paper_2408_11417_b200.tiles import parse_tile
    from tools.profile_gemm import parse_policy

    if hasattr(_lib.lib, "skpp_set_cooperative"):
        _lib.lib.skpp_set_cooperative(0)
    if os.environ.get("SKPP_DEBUG"):
        _lib.lib.skpp_set_debug(int(os.environ["SKPP_DEBUG"]))
    for kv in filter(None, os.environ.get("SKPP_SET", "").split(",")):  # e.g. SKPP_SET=l2_prefetch=4,pdl=0
        name, val = kv.split("=")
        getattr(_lib.lib, "skpp_set_" + name)(int(val))
    if os.environ.get("SKPP_AB_CASES"):
        cases = [tuple(int(v) if v.isdigit() else v for v in c.split(":")) for c in os.environ["SKPP_AB_CASES"].split(",")]
    out = {}
    for m, n, k, tl, pol in cases:
        tile, policy = parse_tile(tl), parse_policy(sk, pol)
        set_bytes = 2 * (m * k + k * n) + 4 * m * n
        n_sets = max(2, -(-(512 << 20) // set_bytes))
        plans = [sk.GemmPlan(torch.randn(m, k, device="cuda").to(torch.bfloat16),
                             torch.randn(k, n, device="cuda").to(torch.bfloat16),
                             torch.empty(m, n, device="cuda"), policy, tile) for _ in range(n_sets)]
        steps = min(5000, max(100, int(0.1 / max(2 * m * n * k / 1.2e15, 15e-6))))
        for i in range(50):
            plans[i % n_sets].launch()
        res = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for i in range(steps):
                plans[i % n_sets].launch()
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) * 1e3 / steps)
        out[f"{m}x{n}x{k}/{tl}/{pol}"] = statistics.median(res)
        del plans
    print("RESULT " + json.dumps(out), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--worker", action="store_true")
    args = ap.parse_args()
    if args.worker:
        worker(CASES)
        return
    libs = args.libs.split(",")
    per = {lib: [] for lib in libs}
    for _ in range(args.rounds):
        for lib in libs:
            path, *sw = lib.split("@")
            env = dict(os.environ, SKPP_LIB=os.path.abspath(path))
            if sw:
                env["SKPP_DEBUG"] = sw[0]
            r = subprocess.run([sys.executable, __file__, "--libs", lib, "--worker"], env=env, capture_output=True,
                               text=True, timeout=900)
            line = next((ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")), None)
            if line is None:
                print(r.stdout[-2000:], r.stderr[-2000:], file=sys.stderr)
                raise SystemExit(f"worker failed for {lib}")
            per[lib].append(json.loads(line[7:]))
    for key in per[libs[0]][0]:
        row = {"case": key}
        for lib in libs:
            row[os.path.basename(lib)] = round(statistics.median(d[key] for d in per[lib]), 3)
        base = row[os.path.basename(libs[0])]
        for lib in libs[1:]:
            row[f"{os.path.basename(lib)}/{os.path.basename(libs[0])}"] = round(row[os.path.basename(lib)] / base, 4)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
