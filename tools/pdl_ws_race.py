"""Does a Stream-K launch race the zero-fill of a freshly allocated fixup workspace?

Each trial allocates a NEW workspace of --ws-mib MiB through executor._new_workspace (torch.zeros
on the launch stream), binds it to the plan and launches the smoke GEMM (384x256x1536, tile
128x128x64, hybrid1) right behind it with no host sync; then checks C against the float64 oracle
and the workspace header (epoch must be 1 and started[1] = g after the launch).  A large
workspace makes the fill long, so a launch that overlaps it shows up reliably.

usage: python tools/pdl_ws_race.py --mode {default,nopdl,sync} [--trials N] [--ws-mib MiB]
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
from paper_2408_11417_b200 import _lib, executor
from oracle import gemm as ogemm


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="default")
    ap.add_argument("--trials", type=int, default=30)
    ap.add_argument("--ws-mib", type=int, default=1024)
    ap.add_argument("--stream", default="default", help="default | side (a created stream)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    if args.mode == "nopdl":
        _lib.lib.skpp_set_pdl(0)
    m, n, k = 384, 256, 1536
    rng = np.random.default_rng(2024)
    a = ogemm.random_int_matrix(m, k, rng)
    b = ogemm.random_int_matrix(k, n, rng)
    want = torch.from_numpy(ogemm.reference_gemm(a, b)).cuda()
    at = torch.from_numpy(a).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
    c = torch.empty(m, n, device="cuda")
    plan = sk.GemmPlan(at, bt, c, sk.Policy.hybrid(1), sk.TileShape(128, 128, 64))
    st = torch.cuda.Stream() if args.stream == "side" else torch.cuda.current_stream()
    handle = st.cuda_stream
    bad_c = bad_hdr = 0
    hdrs = []
    for t in range(args.trials):
        c.fill_(float("nan"))
        torch.cuda.synchronize()
        buf = executor._new_workspace(args.ws_mib << 20, 0, handle)
        if args.mode == "sync":
            torch.cuda.synchronize()
        plan._ws_cache[handle] = (buf.data_ptr(), buf.numel(), buf)
        plan.launch(stream=st)
        torch.cuda.synchronize()
        ok = torch.equal(c.double(), want)
        hdr = buf[:64].view(torch.int32).cpu().tolist()
        hok = hdr[0] == 1 and hdr[9] == plan.g
        bad_c += not ok
        bad_hdr += not hok
        if not hok and len(hdrs) < 3:
            hdrs.append(hdr[:20])
        del buf
    print(json.dumps({"mode": args.mode, "stream": args.stream, "handle": handle, "ws_mib": args.ws_mib,
                      "trials": args.trials, "c_mismatch": bad_c, "hdr_mismatch": bad_hdr, "bad_hdrs": hdrs}))


if __name__ == "__main__":
    main()
