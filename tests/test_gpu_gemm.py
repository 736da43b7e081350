"""GPU parity of the sm_100a Stream-K++ GEMM (run on a B200 via gpurun).

Integer inputs in [-8, 8] (executor.py:44-48 ``random_int_matrix``) are exact
in fp16/bf16 and every partial sum is an integer below 2^24, so the fp32
device result must equal the float64 oracle bit for bit under every policy
and every fixup order.  Random-normal inputs are checked against a float64
product of the same rounded operands with the tolerance stated per test.
"""

import os

import numpy as np
import pytest

from oracle import gemm as ogemm
from oracle import schedule as osched

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _sk():
    import paper_2408_11417_b200 as sk

    return sk


def _int_case(m, n, k, seed):
    rng = np.random.default_rng(seed)
    a = ogemm.random_int_matrix(m, k, rng)
    b = ogemm.random_int_matrix(k, n, rng)
    return a, b


def _run(a, b, policy, tile, g=None, in_dtype=torch.bfloat16, out_dtype=torch.float32, trace_cap=0):
    sk = _sk()
    at = torch.from_numpy(a).to(in_dtype).cuda()
    bt = torch.from_numpy(b).to(in_dtype).cuda()
    c = torch.full((a.shape[0], b.shape[1]), float("nan"), dtype=out_dtype, device="cuda")
    plan = sk.GemmPlan(at, bt, c, policy, tile, g, trace_cap=trace_cap)
    plan.launch()
    torch.cuda.synchronize()
    return c, plan


def _assert_trace(plan, m, n, k, tile, policy, band=0):
    """Device trace == the oracle's build_schedule item for item (tile, kb, ke, write mode,
    phase), and every item's C tile == locate_iter (band 0, the reference's order) or the
    oracle's enumerated banded order."""
    sk = _sk()
    ref = osched.build_schedule(m, n, k, tile[0], tile[1], tile[2], plan.g, policy.kind.value,
                                policy.sk_batches, policy.sk_first)
    dev = plan.trace_items()
    assert [[row[:5] for row in wg] for wg in dev] == ref, policy.label
    mt, nt = -(-m // tile[0]), -(-n // tile[1])
    want = osched.trace_coords(ref, mt, nt, band)
    assert [[tuple(row[6:8]) for row in wg] for wg in dev] == want, (policy.label, band)
    if band == 0:
        grid = sk.grid_info(sk.ProblemSize(m, n, k), sk.TileShape(*tile[:3]))
        for wg in dev:
            for row in wg:
                loc = sk.locate_iter(row[0] * grid.iters_per_tile + row[1], grid)
                assert (loc.tile_m, loc.tile_n) == tuple(row[6:8])




def _policies():
    sk = _sk()
    return sk.canonical_policies() + [sk.Policy.hybrid(2, sk_first=False), sk.Policy.hybrid(7)]


@pytest.mark.parametrize(
    "m,n,k,blk_n,blk_k",
    [
        (128, 128, 64, 128, 64),      # one tile, one k-block
        (256, 256, 256, 128, 64),
        (1024, 1024, 1024, 128, 64),  # BASELINE cfg 1
        (512, 512, 4096, 128, 64),    # cfg 2 shape at reduced K
        (384, 640, 1088, 256, 64),
        (200, 136, 520, 64, 32),      # ragged M/N/K, BK=32
        (130, 72, 48, 64, 16),        # ragged, BK=16
        (512, 512, 4096, 128, 128),   # BK=128: two A boxes per stage
        (1024, 1024, 1024, 256, 128),
        (200, 136, 520, 64, 128),     # ragged, K tail inside the second A box
        (136, 264, 72, 128, 128),     # K < BK: second A box entirely out of bounds
    ],
)
def test_integer_inputs_bitwise_every_policy(m, n, k, blk_n, blk_k):
    _bitwise_every_policy(m, n, k, 128, blk_n, blk_k)


@pytest.mark.parametrize(
    "m,n,k,blk_n,blk_k",
    [
        (256, 256, 256, 256, 64),     # one pair tile
        (1024, 1024, 1024, 256, 64),
        (512, 512, 8192, 128, 64),    # fixup-heavy
        (600, 392, 1000, 256, 64),    # ragged: half-empty second CTA rows / columns
        (300, 200, 520, 128, 32),
        (512, 512, 8192, 256, 128),   # BK=128 pair
        (600, 392, 1000, 128, 128),
    ],
)
def test_cta_pair_tiles_bitwise_every_policy(m, n, k, blk_n, blk_k):
    """cta_group::2 tiles (256 rows over a CTA pair, g = SMs/2 workgroups)."""
    _bitwise_every_policy(m, n, k, 256, blk_n, blk_k)


def _bitwise_every_policy(m, n, k, blk_m, blk_n, blk_k):
    sk = _sk()
    a, b = _int_case(m, n, k, seed=m + n + k)
    want = ogemm.reference_gemm(a, b)
    tile = sk.TileShape(blk_m, blk_n, blk_k)
    for pol in _policies():
        got, _ = _run(a, b, pol, tile)
        g = got.double().cpu().numpy()
        assert np.array_equal(g, want), (pol.label, float(np.nanmax(np.abs(g - want))))


@pytest.mark.parametrize("g", [1, 5, 37, 148])
def test_grid_sizes(g):
    sk = _sk()
    a, b = _int_case(256, 384, 640, seed=g)
    want = ogemm.reference_gemm(a, b)
    for pol in (sk.Policy.data_parallel(), sk.Policy.hybrid(1), sk.Policy.all_stream_k()):
        got, _ = _run(a, b, pol, sk.TileShape(128, 128, 64), g=g)
        assert np.array_equal(got.double().cpu().numpy(), want), (g, pol.label)


def test_device_trace_matches_closed_form_and_oracle():
    sk = _sk()
    size = sk.ProblemSize(1024, 1024, 1024)
    tile = sk.TileShape(128, 128, 64)
    a, b = _int_case(1024, 1024, 1024, seed=1)
    for pol in _policies():
        _, plan = _run(a, b, pol, tile, trace_cap=64)
        _assert_trace(plan, size.m, size.n, size.k, (128, 128, 64), pol)


def test_cta_pair_trace_matches_oracle():
    sk = _sk()
    size = sk.ProblemSize(1024, 2048, 2048)
    a, b = _int_case(size.m, size.n, size.k, seed=3)
    want = ogemm.reference_gemm(a, b)
    for pol in _policies():
        got, plan = _run(a, b, pol, sk.TileShape(256, 256, 64), trace_cap=64)
        assert plan.g == 74
        assert np.array_equal(got.double().cpu().numpy(), want), pol.label
        _assert_trace(plan, size.m, size.n, size.k, (256, 256, 64), pol)


def test_fp16_and_output_dtypes():
    sk = _sk()
    a, b = _int_case(512, 256, 1024, seed=7)
    want = ogemm.reference_gemm(a, b)
    for tile in (sk.TileShape(128, 128, 64), sk.TileShape(256, 256, 64)):
        for in_dt in (torch.float16, torch.bfloat16):
            for out_dt in (torch.float32, torch.bfloat16, torch.float16):
                for pol in (sk.Policy.data_parallel(), sk.Policy.all_stream_k()):
                    got, _ = _run(a, b, pol, tile, in_dtype=in_dt, out_dtype=out_dt)
                    ref = torch.from_numpy(want).to(out_dt).double().numpy()
                    assert np.array_equal(got.double().cpu().numpy(), ref), (tile, in_dt, out_dt, pol.label)


def test_randn_within_tolerance_and_deterministic():
    sk = _sk()
    m, n, k = 512, 512, 16384  # BASELINE cfg 2
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)
    a = torch.randn(m, k, generator=gen, device="cuda").to(torch.bfloat16)
    b = torch.randn(k, n, generator=gen, device="cuda").to(torch.bfloat16)
    ref = (a.double() @ b.double())
    tol = 1e-5 * ref.abs().max().item() * (k / 1024) ** 0.5
    outs = []
    for pol in sk.canonical_policies():
        c = sk.gemm(a, b, pol)
        torch.cuda.synchronize()
        err = (c.double() - ref).abs().max().item()
        assert err <= tol, (pol.label, err, tol)
        if pol == sk.Policy.all_stream_k():
            outs.append(c)
    base = outs[0]
    for _ in range(10):
        again = sk.gemm(a, b, sk.Policy.all_stream_k())
        torch.cuda.synchronize()
        assert torch.equal(again, base)


@pytest.mark.parametrize("tile", [(128, 128, 64), (128, 128, 128), (256, 256, 128)])
def test_fixup_one_pass_and_two_pass_paths_bit_identical(tile):
    """The phase-2 fixup sums (((0 + p1) + p2) ... ) + p0 whether the owner's partial is
    added in the same pass (owner already published) or in a second pass (owner late);
    skpp_set_debug(1) forces the second path.  randn inputs, so rounding would show."""
    sk = _sk()
    from paper_2408_11417_b200 import _lib

    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    m, n, k = 512, 768, 8192
    a = torch.randn(m, k, generator=gen, device="cuda").to(torch.bfloat16)
    b = torch.randn(k, n, generator=gen, device="cuda").to(torch.bfloat16)
    t = sk.TileShape(*tile)
    outs = []
    try:
        for flags in (0, 1):
            _lib.lib.skpp_set_debug(flags)
            for pol in (sk.Policy.all_stream_k(), sk.Policy.hybrid(2, sk_first=False)):
                c = torch.empty(m, n, device="cuda")
                sk.GemmPlan(a, b, c, pol, t).launch()
                torch.cuda.synchronize()
                outs.append(c)
    finally:
        _lib.lib.skpp_set_debug(0)
    assert torch.equal(outs[0], outs[2]) and torch.equal(outs[1], outs[3])


@pytest.mark.parametrize("tile", [(128, 128, 64), (128, 128, 128), (256, 256, 128)])
def test_multi_wave_serpentine_k_bitwise(tile):
    """Several data-parallel waves per workgroup (odd waves walk K backwards), ragged K
    tail inside the first reversed k-block; integer inputs => exact in any order."""
    sk = _sk()
    m, n, k = 2048, 2560, 1096
    a, b = _int_case(m, n, k, seed=11)
    want = ogemm.reference_gemm(a, b)
    for pol in (sk.Policy.data_parallel(), sk.Policy.hybrid(1), sk.Policy.hybrid(2, sk_first=False)):
        got, _ = _run(a, b, pol, sk.TileShape(*tile))
        assert np.array_equal(got.double().cpu().numpy(), want), pol.label


@pytest.mark.parametrize("m,n,k,tile", [
    (1, 4096, 4096, (128, 128, 128)),     # decode-like: partials hold one 32-row chunk
    (16, 1096, 2048, (128, 128, 64)),     # skinny M with a last column tile over half full
    (33, 4136, 1024, (128, 128, 128)),    # N % 128 = 40: last column tile skips chunks
    (20, 600, 4096, (256, 256, 128)),     # CTA pair: rank-1 half entirely past M
])
def test_skinny_and_narrow_edge_tiles_bitwise_every_policy(m, n, k, tile):
    """Stream-K partials and reduction bands bounded to the valid 32-row / 32-column chunks
    (GemmParams.ragged) stay bitwise equal to the float64 oracle on integer inputs."""
    _bitwise_every_policy(m, n, k, *tile)


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (1, 8, 8), (7, 9, 5), (1, 4096, 8), (300, 1, 700), (2, 3, 70000)])
@pytest.mark.parametrize("tile", [(128, 128, 64), (128, 64, 128), (128, 128, 128), (256, 256, 128)])
def test_degenerate_shapes_bitwise(m, n, k, tile):
    """Tiny / degenerate extents (K, N below a TMA box, M = 1, very long K) through the
    padding host path: bitwise vs the float64 oracle for DP and all-Stream-K."""
    sk = _sk()
    a, b = _int_case(m, n, k, seed=m * 31 + n * 7 + k)
    want = ogemm.reference_gemm(a, b)
    size, t = sk.ProblemSize(m, n, k), sk.TileShape(*tile)
    g = sk.executor.default_g(t)
    for pol in (sk.Policy.data_parallel(), sk.Policy.all_stream_k()):
        sched = sk.build_schedule(size, t, sk.HardwareModel(g, 1), pol)
        got = sk.execute_schedule(a, b, sched, t, size)
        assert np.array_equal(got, want), (pol.label, float(np.abs(got - want).max()))


# Seeded fuzz over the whole device surface: random shapes (M arbitrary, N and K
# multiples of 8 as TMA needs), every implemented tile, canonical and non-canonical
# policies (hybrid s up to 9, DP-first), random grid sizes.  Each case is checked
# bitwise against the float64 oracle and its device item trace against the oracle's
# build_schedule, so any schedule/fixup disagreement shows up as a named case.
_FUZZ_TILES = [(128, bn, bk) for bn in (64, 128, 256) for bk in (16, 32, 64, 128)] + \
              [(256, bn, bk) for bn in (128, 256) for bk in (32, 64, 128)]


def _fuzz_cases(n_cases=100, seed=2408):
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n_cases):
        tile = _FUZZ_TILES[int(rng.integers(len(_FUZZ_TILES)))]
        m = int(rng.integers(1, 1400))
        n = 8 * int(rng.integers(1, 180))
        k = 8 * int(rng.integers(1, 700))
        gmax = 148 // (tile[0] // 128)
        g = int(rng.choice([gmax, gmax, int(rng.integers(1, gmax + 1))]))
        kind = int(rng.integers(3))
        pol = ("dp",) if kind == 0 else ("ask",) if kind == 1 else ("hybrid", int(rng.integers(1, 10)), bool(rng.integers(2)))
        cases.append((i, m, n, k, tile, g, pol))
    return cases


@pytest.mark.parametrize("case", _fuzz_cases(int(os.environ.get("SKPP_FUZZ_CASES", "100"))), ids=lambda c: f"fuzz{c[0]}-{c[1]}x{c[2]}x{c[3]}-{c[4][0]}x{c[4][1]}x{c[4][2]}-g{c[5]}-{c[6][0]}")
def test_fuzz_bitwise_and_trace(case):
    sk = _sk()
    i, m, n, k, tile, g, pol = case
    policy = (sk.Policy.data_parallel() if pol[0] == "dp" else sk.Policy.all_stream_k() if pol[0] == "ask"
              else sk.Policy.hybrid(pol[1], sk_first=pol[2]))
    a, b = _int_case(m, n, k, seed=1000 + i)
    got, plan = _run(a, b, policy, sk.TileShape(*tile), g=g, trace_cap=512)
    want = ogemm.reference_gemm(a, b)
    gd = got.double().cpu().numpy()
    assert np.array_equal(gd, want), float(np.nanmax(np.abs(gd - want)))
    ref = osched.build_schedule(m, n, k, tile[0], tile[1], tile[2], g, policy.kind.value, policy.sk_batches,
                                policy.sk_first)
    if max(len(w) for w in ref) <= 512:
        _assert_trace(plan, m, n, k, tile, policy)


@pytest.mark.parametrize("band", [0, 3, 8, 16])
@pytest.mark.parametrize("m,n,k,tile", [
    (2304, 3000, 1000, (256, 256, 64)),   # 9 x 12 = 108 pair tiles on 74 pairs: 1.5 waves
    (1500, 2600, 704, (128, 64, 64)),     # 12 x 41 = 492 tiles: >= 3 waves of 148
    (4000, 4104, 520, (128, 128, 128)),   # 32 x 33 = 1056 tiles: 7 waves
    (700, 9000, 304, (256, 128, 32)),     # 3 x 71 tile rows fewer than the band
])
def test_banded_tile_order_bitwise_every_policy(band, m, n, k, tile):
    """The banded tile order (KernelTile band_rows, skpp_tile_t.tile_order) is a bijection:
    every policy stays bit-exact against the oracle, the device trace is still the reference
    schedule, and each item's C tile is the oracle's enumerated banded order (band 0: the
    reference's locate_iter)."""
    sk = _sk()
    a, b = _int_case(m, n, k, seed=m ^ n ^ k)
    want = ogemm.reference_gemm(a, b)
    t = sk.kernel_tile(*tile, band)
    for pol in (sk.Policy.data_parallel(), sk.Policy.hybrid(1), sk.Policy.hybrid(2, sk_first=False),
                sk.Policy.all_stream_k()):
        got, plan = _run(a, b, pol, t, trace_cap=64)
        assert np.array_equal(got.double().cpu().numpy(), want), (band, pol.label)
        _assert_trace(plan, m, n, k, tile, pol, band)


@pytest.mark.parametrize("grid", [64, 128, 144])
@pytest.mark.parametrize("m,n,k,tile", [
    (512, 512, 16384, (128, 128, 128)),   # cfg2: 16 tiles x 128 k-iterations
    (16, 4096, 4096, (128, 128, 128)),    # decode-like
    (1024, 1024, 1024, (128, 64, 128)),   # 128 tiles x 8 k-iterations
])
def test_declared_grid_bitwise_every_policy(grid, m, n, k, tile):
    """KernelTile.grid: a launch on g = grid workgroups (default_g honours the tile) runs the
    reference's schedule for HardwareModel(grid, 1) item for item and stays bit-exact."""
    sk = _sk()
    a, b = _int_case(m, n, k, seed=m ^ n ^ k ^ grid)
    want = ogemm.reference_gemm(a, b)
    t = sk.kernel_tile(*tile, 0, grid)
    for pol in (sk.Policy.data_parallel(), sk.Policy.hybrid(1), sk.Policy.all_stream_k()):
        got, plan = _run(a, b, pol, t, trace_cap=64)
        assert plan.g == grid
        assert np.array_equal(got.double().cpu().numpy(), want), (grid, pol.label)
        _assert_trace(plan, m, n, k, tile, pol)


@pytest.mark.parametrize("out", ["fp32", "bf16"])
@pytest.mark.parametrize("m,n,k,tile,pol", [
    (2048, 2560, 1096, (128, 128, 64), ("hybrid", 2, True)),      # multi-wave, two-contributor split tiles
    (1024, 14336, 1024, (256, 256, 128, 16), ("hybrid", 3, True)),  # banded CTA pair (cfg3-like hybrid)
    (1536, 2048, 4096, (128, 128, 128), ("hybrid", 2, False)),    # DP-first: Stream-K items last
])
def test_owner_reduction_bit_identical_to_phase2_path(m, n, k, tile, pol, out):
    """Owner reduction: a split tile with two contributors whose owner item is the owner's last
    Stream-K item is finished in the owner's epilogue ((0 + p[x+1]) + p[x]) instead of in phase 2.
    The path must be taken (slot flags carry epoch | 0x80000000), give the same bits as the
    phase-2 reduction (skpp_set_debug bit 4 disables it) on randn inputs, and be exact on
    integer inputs."""
    sk = _sk()
    from paper_2408_11417_b200 import _lib

    t = sk.kernel_tile(*tile) if len(tile) == 4 else sk.TileShape(*tile)
    policy = sk.Policy.hybrid(pol[1], sk_first=pol[2])
    gen = torch.Generator(device="cuda")
    gen.manual_seed(m + n)
    ar = torch.randn(m, k, generator=gen, device="cuda").to(torch.bfloat16)
    br = torch.randn(k, n, generator=gen, device="cuda").to(torch.bfloat16)
    outs = []
    try:
        for flags in (16, 0):
            _lib.lib.skpp_set_debug(flags)
            c = torch.full((m, n), float("nan"), device="cuda",
                           dtype=torch.float32 if out == "fp32" else torch.bfloat16)
            plan = sk.GemmPlan(ar, br, c, policy, t)
            plan.launch()
            torch.cuda.synchronize()
            outs.append(c)
            if flags == 0:
                ws = next(iter(plan._ws_cache.values()))[2]
                hdr = ws[:64].view(torch.int32).cpu()
                epoch = int(hdr[0])
                n_slots = 2 * plan.g * (tile[0] // 128)
                words = ws[1024:1024 + 4 * n_slots].view(torch.int32).cpu().numpy().view(np.uint32)
                assert int((words == (epoch | 0x80000000)).sum()) > 0, "owner reduction never taken"
    finally:
        _lib.lib.skpp_set_debug(0)
    assert torch.equal(outs[0].view(torch.int16 if out == "bf16" else torch.int32),
                       outs[1].view(torch.int16 if out == "bf16" else torch.int32))  # bits, incl. signed zeros
    if out == "fp32":
        a, b = _int_case(m, n, k, seed=k)
        got, _ = _run(a, b, policy, t)
        assert np.array_equal(got.double().cpu().numpy(), ogemm.reference_gemm(a, b))
