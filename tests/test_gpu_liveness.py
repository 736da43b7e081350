"""Liveness of Stream-K grids that share the GPU (run on a B200 via gpurun).

Phase-2 reducers wait for peer flags at most ~20 us; then, if some CTA of the launch has not
started yet (its SM is held by another grid), the reducer marks its band abandoned and exits,
and the last CTA to start reduces it; if every CTA has started, waiting is safe and it keeps
waiting.  So no CTA ever waits on a CTA that is not resident.
These tests drive that: concurrent Stream-K grids on prioritised streams, two processes on
one GPU, a GEMM that runs while 140 (or 100) of the 148 SMs are held by another grid, and a
zero wait bound on every phase-2 wait (skpp_set_debug bit 1) — all bitwise.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "_liveness_worker.py")


def _run_workers(args_list, timeout=240):
    procs = [subprocess.Popen([sys.executable, WORKER, *map(str, args), ROOT], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True, cwd=ROOT) for args in args_list]
    outs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=timeout)
            outs.append((p.returncode, out))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    return outs


def test_concurrent_streamk_grids_on_prioritised_streams():
    (rc, out), = _run_workers([("streams", 200, 4, 11)])
    assert rc == 0 and out.strip().endswith("ok"), out[-2000:]


def test_two_processes_share_one_gpu():
    for rc, out in _run_workers([("streams", 200, 3, 12), ("streams", 200, 3, 13)]):
        assert rc == 0 and out.strip().endswith("ok"), out[-2000:]


def test_gemm_completes_while_partially_resident():
    """With 140 of 148 SMs held, the 148-CTA grid runs 8 CTAs at a time: reducers time out while
    CTAs have not started, abandon their bands, and the last CTA to start reduces them — the
    path must actually be taken (abandoned bands are counted in the workspace header).  With
    100 SMs held (the CTA-pair tile included) the grid also completes, bitwise."""
    (rc, out), = _run_workers([("partial", 2, 140, 14)], timeout=180)
    assert rc == 0 and out.strip().endswith("ok"), out[-2000:]
    total = int(out.split("abandoned_total=")[1].split()[0])
    assert total > 0, out[-2000:]
    (rc, out), = _run_workers([("partial", 3, 100, 15)], timeout=180)
    assert rc == 0 and out.strip().endswith("ok"), out[-2000:]


@pytest.mark.parametrize("debug", [2, 3])
@pytest.mark.parametrize("tile,shape", [((128, 128, 64), (512, 512, 8192)), ((128, 128, 128), (16, 4096, 4096)),
                                        ((256, 256, 128), (600, 392, 4096)), ((128, 64, 128), (1, 4096, 65536))])
def test_abandon_path_bit_identical(debug, tile, shape):
    """Bound 0 on every phase-2 wait: every wait that is not already satisfied goes through the
    timeout decision (keep waiting when every CTA has started, else abandon to the last starter);
    every policy stays bitwise on integer inputs and bit-identical to the normal path on randn."""
    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import _lib
    from oracle import gemm as ogemm

    m, n, k = shape
    rng = np.random.default_rng(m + n + k)
    a = ogemm.random_int_matrix(m, k, rng)
    b = ogemm.random_int_matrix(k, n, rng)
    want = ogemm.reference_gemm(a, b)
    at, bt = torch.from_numpy(a).to(torch.bfloat16).cuda(), torch.from_numpy(b).to(torch.bfloat16).cuda()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    ar = torch.randn(m, k, generator=gen, device="cuda").to(torch.bfloat16)
    br = torch.randn(k, n, generator=gen, device="cuda").to(torch.bfloat16)
    t = sk.TileShape(*tile)
    for pol in (sk.Policy.all_stream_k(), sk.Policy.hybrid(1), sk.Policy.hybrid(2, sk_first=False)):
        ref = torch.empty(m, n, device="cuda")
        sk.GemmPlan(ar, br, ref, pol, t).launch()
        try:
            _lib.lib.skpp_set_debug(debug)
            c = torch.full((m, n), float("nan"), device="cuda")
            sk.GemmPlan(at, bt, c, pol, t).launch()
            cr = torch.empty(m, n, device="cuda")
            for _ in range(3):
                sk.GemmPlan(ar, br, cr, pol, t).launch()
            torch.cuda.synchronize()
        finally:
            _lib.lib.skpp_set_debug(0)
        assert np.array_equal(c.double().cpu().numpy(), want), (pol.label, debug)
        assert torch.equal(cr, ref), (pol.label, debug)
