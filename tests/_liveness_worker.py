"""Workers for tests/test_gpu_liveness.py (run as subprocesses so that a hang is contained).

``streams R S SEED ROOT``: Stream-K launches on S streams of different priorities at once,
R rounds (concurrent Stream-K grids, and another process under the two-process test).

``partial R HOLD SEED ROOT``: a grid of HOLD single-warp CTAs with ~120 KiB of shared memory
each occupies HOLD SMs until a release flag is set; a Stream-K GEMM launched next on another
stream is then only partially resident (148 - HOLD SMs free; with HOLD = 140 the 148-CTA grid
runs 8 CTAs at a time, ~30x its normal duration).  The flag is set by a kernel
that waits for the GEMM to finish, so the GEMM must complete while partially resident — the
case the phase-2 abandon protocol exists for (a cooperative launch would deadlock here).

Both exit 0 when every result is bitwise equal to the float64 product of integer inputs.
"""

import os
import sys
import time

import torch


def _operands(seed, m=512, n=512, k=8192):
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    a = torch.randint(-8, 9, (m, k), generator=gen, device="cuda", dtype=torch.int8)
    b = torch.randint(-8, 9, (k, n), generator=gen, device="cuda", dtype=torch.int8)
    return a.to(torch.bfloat16), b.to(torch.bfloat16), a.double() @ b.double()


def streams(rounds: int, n_streams: int, seed: int) -> int:
    import paper_2408_11417_b200 as sk

    ab, bb, want = _operands(seed)
    lo, hi = torch.cuda.Stream.priority_range()
    sts = [torch.cuda.Stream(priority=lo if i % 2 else hi) for i in range(n_streams)]
    plans = [sk.GemmPlan(ab, bb, torch.zeros_like(want, dtype=torch.float32),
                         sk.Policy.all_stream_k() if i % 2 else sk.Policy.hybrid(1),
                         sk.TileShape(128, 128, 64) if i % 2 else sk.TileShape(256, 256, 64))
             for i in range(n_streams)]
    for st in sts:
        st.wait_stream(torch.cuda.current_stream())
    for _ in range(rounds):
        for p, st in zip(plans, sts):
            p.launch(stream=st)
    torch.cuda.synchronize()
    return 0 if all(torch.equal(p.c.double(), want) for p in plans) else 1


def partial(rounds: int, hold: int, seed: int) -> int:
    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import _lib

    shape = os.environ.get("SKPP_LIVENESS_SHAPE")  # "m,n,k" (diagnostics; default 512x512x8192)
    ab, bb, want = _operands(seed, *map(int, shape.split(","))) if shape else _operands(seed)
    s_hold, s_gemm, s_rel = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    cases = [(sk.Policy.all_stream_k(), sk.TileShape(128, 128, 64)),
             (sk.Policy.hybrid(1), sk.TileShape(128, 128, 128)),
             (sk.Policy.all_stream_k(), sk.TileShape(256, 256, 64))]
    total_abandoned = 0
    for r in range(rounds):
        pol, tile = cases[r % len(cases)]
        c = torch.zeros_like(want, dtype=torch.float32)
        plan = sk.GemmPlan(ab, bb, c, pol, tile)
        plan.launch(stream=s_gemm)  # warm: workspace, module load
        s_gemm.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s_gemm)
        plan.launch(stream=s_gemm)
        a1.record(s_gemm)
        a1.synchronize()
        alone_us = a0.elapsed_time(a1) * 1e3
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        _lib.check(_lib.lib.skpp_test_hold_sms(hold, 120 * 1024, flag.data_ptr(), s_hold.cuda_stream))
        time.sleep(0.02)  # the holding CTAs are resident before the GEMM is launched
        c.zero_()
        torch.cuda.current_stream().synchronize()
        t0 = time.perf_counter()
        g0, done = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(s_gemm)
        plan.launch(stream=s_gemm)
        done.record(s_gemm)
        s_rel.wait_event(done)
        with torch.cuda.stream(s_rel):
            flag.fill_(1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ok = torch.equal(c.double(), want)
        # workspace header of the launch: [0] epoch, [16 + (epoch & 1)] bands abandoned by
        # reducers that timed out while CTAs had not started (reduced by the last starter)
        ws = plan._ws_cache[s_gemm.cuda_stream][2]
        hdr = ws[:256].view(torch.int32).cpu()
        abandoned = int(hdr[16 + (int(hdr[0]) & 1)])
        if os.environ.get("SKPP_LIVENESS_DEBUG"):
            st = ws[1024 + 8192:1024 + 8192 + 8192].view(torch.int32).view(2, 1024).cpu()
            print("hdr", hdr[:24].tolist(), "states(par)", st[int(hdr[0]) & 1, :148].tolist(), flush=True)
        total_abandoned += abandoned
        print(f"round {r}: {pol.label} {tile} with {hold} SMs held: GEMM {g0.elapsed_time(done) * 1e3:.1f} us "
              f"(alone {alone_us:.1f} us), wall {dt * 1e3:.2f} ms, bitwise={ok}, "
              f"bands abandoned={abandoned}", flush=True)
        if not ok:
            return 1
    print(f"abandoned_total={total_abandoned}", flush=True)
    return 0


if __name__ == "__main__":
    sys.path.insert(0, sys.argv[5])
    mode = sys.argv[1]
    rc = (streams if mode == "streams" else partial)(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
    print("ok" if rc == 0 else "mismatch", flush=True)
    sys.exit(rc)
