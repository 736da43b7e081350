"""GPU parity at the BASELINE configurations' full sizes (run on a B200 via gpurun).

The reference's bar is every policy bitwise against ``reference_gemm``
(``tests/test_executor.py:51-57``; ``executor.py:51-124``).  Integer inputs in
[-8, 8] are exact in fp16/bf16 and every partial sum stays below 2^24, so the fp32
device result must equal the float64 product bit for bit.  The float64 product is
computed with a torch float64 matmul on the device (the same ``A @ B`` as the oracle's
``reference_gemm``, exact on these inputs in any summation order), which keeps the
8192 x 14336 x 4096 cases to seconds.

* cfg3 (Llama-3-8B projections): M in {1, 16, 128, 512, 1024, 4096, 8192} x N in
  {4096, 14336} x K = 4096 under the (tile, policy) the Stream-K++ selection picks from
  the committed tile bank, and under the banded CTA-pair tile 256x256x128b16
  (``streamk_gemm_kernel<256, 128, 2, true>``) for DP / hybrid1 / all-Stream-K, with the
  device trace's C tiles checked against the oracle's banded order.
* cfg2: 512 x 512 x 16384 (full K), all seven canonical policies.
* cfg1: fp16 1024^3, DP and hybrid1.
"""

import os

import pytest

from oracle import schedule as osched

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sk():
    import paper_2408_11417_b200 as sk

    return sk


def _int_operands(m, n, k, seed, dtype=torch.bfloat16):
    """random_int_matrix-style operands in [-8, 8], drawn on the device (A then B)."""
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    a = torch.randint(-8, 9, (m, k), generator=gen, device="cuda", dtype=torch.int8)
    b = torch.randint(-8, 9, (k, n), generator=gen, device="cuda", dtype=torch.int8)
    want = a.double() @ b.double()
    return a.to(dtype), b.to(dtype), want


def _check(a, b, want, policy, tile, trace_cap=0):
    sk = _sk()
    c = torch.full(want.shape, float("nan"), dtype=torch.float32, device="cuda")
    plan = sk.GemmPlan(a, b, c, policy, tile, trace_cap=trace_cap)
    plan.launch()
    torch.cuda.synchronize()
    bad = (c.double() != want)
    if bool(bad.any()):
        idx = bad.nonzero()[0].tolist()
        raise AssertionError(f"{policy.label} on {sk.tiles.tile_label(tile)}: {int(bad.sum())} elements differ, "
                             f"first at {idx}: got {c[idx[0], idx[1]].item()} want {want[idx[0], idx[1]].item()}")
    return plan


def _selector():
    sk = _sk()
    from paper_2408_11417_b200 import tiles as tl

    return tl.Selector(tl.TileBank.load(sk.default_bank_dir()))


CFG3 = [(m, n) for n in (4096, 14336) for m in (1, 16, 128, 512, 1024, 4096, 8192)]


@pytest.mark.parametrize("m,n", CFG3, ids=[f"{m}x{n}x4096" for m, n in CFG3])
def test_cfg3_selected_config_and_banded_pair_bitwise(m, n):
    sk = _sk()
    k = 4096
    a, b, want = _int_operands(m, n, k, seed=m * 7 + n)
    size = sk.ProblemSize(m, n, k)
    # the configuration the selection layer runs for this size (Bloom candidates, timed once)
    out = torch.empty(m, n, device="cuda")
    tile, pol = _selector().config(size, a, b, out)
    _check(a, b, want, pol, tile)
    # the banded CTA-pair tile behind the large-shape numbers, with its trace
    banded = sk.kernel_tile(256, 256, 128, 16)
    for p in (sk.Policy.data_parallel(), sk.Policy.hybrid(1), sk.Policy.all_stream_k()):
        plan = _check(a, b, want, p, banded, trace_cap=64)
        ref = osched.build_schedule(m, n, k, 256, 256, 128, plan.g, p.kind.value, p.sk_batches, p.sk_first)
        dev = plan.trace_items()
        assert [[row[:5] for row in wg] for wg in dev] == ref, p.label
        want_coords = osched.trace_coords(ref, -(-m // 256), -(-n // 256), 16)
        assert [[tuple(row[6:8]) for row in wg] for wg in dev] == want_coords, p.label


def test_cfg3_reference_order_trace_equals_locate_iter():
    """Parity mode (tile order 0) on the largest cfg3 shape: every item's C tile is the
    reference's locate_iter (scheduler.py:155-165), and the output is bitwise."""
    sk = _sk()
    m, n, k = 8192, 14336, 4096
    a, b, want = _int_operands(m, n, k, seed=5)
    tile = sk.TileShape(256, 256, 128)
    grid = sk.grid_info(sk.ProblemSize(m, n, k), tile)
    for p in (sk.Policy.data_parallel(), sk.Policy.hybrid(2, sk_first=False)):
        plan = _check(a, b, want, p, tile, trace_cap=64)
        for wg in plan.trace_items():
            for row in wg:
                loc = sk.locate_iter(row[0] * grid.iters_per_tile + row[1], grid)
                assert (loc.tile_m, loc.tile_n) == tuple(row[6:8])


@pytest.mark.parametrize("tile", [(128, 128, 64), (128, 128, 128), (128, 64, 128), (256, 256, 128)])
def test_cfg2_full_k_every_policy_bitwise(tile):
    sk = _sk()
    a, b, want = _int_operands(512, 512, 16384, seed=2)
    for p in sk.canonical_policies():
        _check(a, b, want, p, sk.TileShape(*tile))


def test_cfg2_selected_config_bitwise():
    sk = _sk()
    a, b, want = _int_operands(512, 512, 16384, seed=3)
    tile, pol = _selector().config(sk.ProblemSize(512, 512, 16384), a, b, torch.empty(512, 512, device="cuda"))
    _check(a, b, want, pol, tile)


@pytest.mark.parametrize("tile", [(128, 128, 64), (128, 128, 128), (256, 256, 64)])
def test_cfg1_fp16_1024_dp_and_hybrid1_bitwise(tile):
    sk = _sk()
    a, b, want = _int_operands(1024, 1024, 1024, seed=1, dtype=torch.float16)
    for p in (sk.Policy.data_parallel(), sk.Policy.hybrid(1)):
        _check(a, b, want, p, sk.TileShape(*tile))
