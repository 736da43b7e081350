"""GPU tests of the public drop-in API (execute_schedule / run_equivalence / gemm).

Mirrors the reference's executor tests (tests/test_executor.py in gemmsched):
every canonical policy bitwise-equal to the float64 oracle on integer inputs,
ragged edges, shuffled-order and threaded arguments, error messages — plus the
device-specific contracts: CUDA-graph replays, workspace reuse, unaligned
operands, and that the native library is what actually runs.
"""

import numpy as np
import pytest

from oracle import gemm as ogemm

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def sk():
    import paper_2408_11417_b200 as m

    return m


def instance(size, tile, g, policy, seed=0):
    rng = np.random.default_rng(seed)
    a = ogemm.random_int_matrix(size.m, size.k, rng)
    b = ogemm.random_int_matrix(size.k, size.n, rng)
    sched = sk().build_schedule(size, tile, sk().HardwareModel(g, 1), policy)
    return a, b, sched


def test_native_library_is_loaded():
    from paper_2408_11417_b200 import _lib

    maps = open("/proc/self/maps").read()
    assert str(_lib.LIB_PATH) in maps


def test_every_canonical_policy_matches_reference_numpy_path():
    m = sk()
    size, tile = m.ProblemSize(384, 256, 640), m.TileShape(128, 128, 64)
    for policy in m.canonical_policies():
        a, b, sched = instance(size, tile, 148, policy, seed=11)
        got = m.execute_schedule(a, b, sched, tile, size)
        assert got.dtype == np.float64
        assert np.array_equal(got, m.reference_gemm(a, b)), policy


def test_ragged_unaligned_k_and_n_are_padded_transparently():
    m = sk()
    size, tile = m.ProblemSize(100, 75, 53), m.TileShape(128, 64, 16)
    for policy in (m.Policy.data_parallel(), m.Policy.hybrid(3), m.Policy.all_stream_k()):
        a, b, sched = instance(size, tile, 7, policy, seed=4)
        got = m.execute_schedule(a, b, sched, tile, size)
        assert np.array_equal(got, m.reference_gemm(a, b)), policy


def test_shuffled_and_threaded_arguments_are_accepted_and_exact():
    m = sk()
    size, tile = m.ProblemSize(256, 256, 512), m.TileShape(128, 128, 64)
    a, b, sched = instance(size, tile, 148, m.Policy.hybrid(2), seed=5)
    base = m.execute_schedule(a, b, sched, tile, size)
    for trial in range(3):
        shuffled = m.execute_schedule(a, b, sched, tile, size, order="shuffled", rng=np.random.default_rng(trial))
        assert shuffled.tobytes() == base.tobytes()
    assert np.array_equal(m.execute_schedule(a, b, sched, tile, size, workers=4), base)


def test_error_messages_match_reference():
    m = sk()
    size, tile = m.ProblemSize(128, 128, 64), m.TileShape(128, 128, 64)
    a, b, sched = instance(size, tile, 148, m.Policy.data_parallel())
    with pytest.raises(ValueError, match="rng"):
        m.execute_schedule(a, b, sched, tile, size, order="shuffled")
    with pytest.raises(ValueError, match="order"):
        m.execute_schedule(a, b, sched, tile, size, order="sideways")
    with pytest.raises(ValueError, match="do not match"):
        m.execute_schedule(a[:8], b, sched, tile, size)
    other = m.ProblemSize(128, 128, 128)
    a2, b2, _ = instance(other, tile, 148, m.Policy.data_parallel())
    with pytest.raises(ValueError, match="different problem"):
        m.execute_schedule(a2, b2, sched, tile, other)
    with pytest.raises(ValueError, match="inner dimensions"):
        m.reference_gemm(np.zeros((2, 3)), np.zeros((4, 2)))
    with pytest.raises(ValueError, match="not implemented"):
        t2 = m.TileShape(64, 64, 32)
        m.execute_schedule(a, b, m.build_schedule(size, t2, m.HardwareModel(148, 1), m.Policy.data_parallel()), t2, size)


def test_hand_edited_schedule_is_rejected():
    m = sk()
    size, tile = m.ProblemSize(256, 256, 256), m.TileShape(128, 128, 64)
    a, b, sched = instance(size, tile, 148, m.Policy.all_stream_k())
    items = [list(wg) for wg in sched.assignments]
    first = next(i for i, wg in enumerate(items) if wg)
    del items[first][0]
    bad = m.Schedule(sched.grid, sched.g, sched.policy, tuple(tuple(w) for w in items))
    assert not m.validate_schedule(bad).covered_once
    with pytest.raises(ValueError, match="closed form"):
        m.execute_schedule(a, b, bad, tile, size)


@pytest.mark.parametrize("policy_idx", range(7))
def test_run_equivalence_like_reference(policy_idx):
    m = sk()
    policy = m.canonical_policies()[policy_idx]
    for size in (m.ProblemSize(1, 64, 16), m.ProblemSize(100, 100, 100), m.ProblemSize(256, 256, 256)):
        rep = m.run_equivalence(size, m.TileShape(128, 128, 64), m.HardwareModel(104, 1), policy, rng_seed=42)
        assert rep.exact_match and rep.max_abs_diff == 0.0, (size, policy)


def test_torch_cuda_and_host_tensors():
    m = sk()
    size, tile = m.ProblemSize(512, 384, 2048), m.TileShape(256, 256, 64)
    a, b, sched = instance(size, tile, 74, m.Policy.hybrid(1), seed=9)
    want = ogemm.reference_gemm(a, b)
    at, bt = torch.from_numpy(a).to(torch.bfloat16), torch.from_numpy(b).to(torch.bfloat16)
    dev = m.execute_schedule(at.cuda(), bt.cuda(), sched, tile, size)
    assert dev.is_cuda and np.array_equal(dev.double().cpu().numpy(), want)
    host = m.execute_schedule(at.pin_memory(), bt.pin_memory(), sched, tile, size)
    assert not host.is_cuda and np.array_equal(host.double().numpy(), want)


def test_unaligned_output_uses_direct_stores():
    m = sk()
    size = m.ProblemSize(256, 200, 512)
    a, b, _ = instance(size, m.TileShape(128, 128, 64), 148, m.Policy.data_parallel(), seed=2)
    at = torch.from_numpy(a).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
    big = torch.zeros(256, 203, device="cuda")  # row stride 203 floats: not 16-byte aligned
    c = big[:, 1:201]
    for pol in (m.Policy.data_parallel(), m.Policy.all_stream_k()):
        c.zero_()
        m.GemmPlan(at, bt, c, pol, m.TileShape(128, 128, 64)).launch()
        torch.cuda.synchronize()
        assert np.array_equal(c.double().cpu().numpy(), ogemm.reference_gemm(a, b)), pol
        assert float(big[:, 0].abs().sum()) == 0.0 and float(big[:, 201:].abs().sum()) == 0.0


def test_cuda_graph_replays_and_workspace_reuse():
    """Epoch-tagged flags keep graph replays (frozen parameters) correct."""
    m = sk()
    rng = np.random.default_rng(8)
    shapes = [(512, 512, 4096), (384, 256, 2048)]
    plans, wants = [], []
    for mm, nn, kk in shapes:
        a = ogemm.random_int_matrix(mm, kk, rng)
        b = ogemm.random_int_matrix(kk, nn, rng)
        at = torch.from_numpy(a).to(torch.bfloat16).cuda()
        bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
        c = torch.zeros(mm, nn, device="cuda")
        plans.append(m.GemmPlan(at, bt, c, m.Policy.all_stream_k(), m.TileShape(128, 128, 64)))
        wants.append(ogemm.reference_gemm(a, b))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        for p in plans:
            p.launch()  # warm the per-stream workspace outside capture
        side.synchronize()
        with torch.cuda.graph(graph, stream=side):
            for _ in range(3):
                for p in plans:
                    p.launch()
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(5):
        for p in plans:
            p.c.zero_()
        graph.replay()
        torch.cuda.synchronize()
        for p, want in zip(plans, wants):
            assert np.array_equal(p.c.double().cpu().numpy(), want)


def test_graphs_captured_on_one_stream_replay_concurrently():
    """Captured launches use a plan-private workspace (GemmPlan.prepare_for_capture), so two
    graphs captured on the same stream can be replayed at the same time on two streams."""
    m = sk()
    rng = np.random.default_rng(9)
    a = ogemm.random_int_matrix(512, 4096, rng)
    b = ogemm.random_int_matrix(4096, 512, rng)
    want = ogemm.reference_gemm(a, b)
    at = torch.from_numpy(a).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
    plans = [m.GemmPlan(at, bt, torch.zeros(512, 512, device="cuda"), m.Policy.all_stream_k(),
                        m.TileShape(128, 128, 64)) for _ in range(2)]
    side = torch.cuda.Stream()
    graphs = []
    for i, p in enumerate(plans):
        if i == 0:
            p.prepare_for_capture(side)  # the other plan allocates inside its capture
        g = torch.cuda.CUDAGraph()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=side):
            for _ in range(4):
                p.launch()
        graphs.append(g)
    assert plans[0]._private_ws.data_ptr() != plans[1]._private_ws.data_ptr()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for _ in range(10):
        for p in plans:
            p.c.zero_()
        torch.cuda.synchronize()
        for g, s in zip(graphs, streams):
            with torch.cuda.stream(s):
                g.replay()
        torch.cuda.synchronize()
        for p in plans:
            assert np.array_equal(p.c.double().cpu().numpy(), want)


def test_first_launch_on_a_non_current_stream():
    """The eager workspace of a new stream is allocated and zeroed on that stream, so a
    plan launched with stream=s (s not torch's current stream) sees initialised flags."""
    m = sk()
    rng = np.random.default_rng(10)
    a = ogemm.random_int_matrix(256, 8192, rng)
    b = ogemm.random_int_matrix(8192, 384, rng)
    want = ogemm.reference_gemm(a, b)
    at = torch.from_numpy(a).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
    for _ in range(3):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        c = torch.zeros(256, 384, device="cuda")
        plan = m.GemmPlan(at, bt, c, m.Policy.all_stream_k(), m.TileShape(128, 128, 128))
        for _ in range(3):
            plan.launch(stream=s)
        s.synchronize()
        assert np.array_equal(c.double().cpu().numpy(), want)


def test_device_schedule_trace_kernel_matches_host():
    m = sk()
    from paper_2408_11417_b200 import _lib, scheduler

    for size, tile, g, pol in [
        (m.ProblemSize(8192, 14336, 4096), m.TileShape(128, 128, 64), 148, m.Policy.hybrid(3)),
        (m.ProblemSize(1, 64, 65536), m.TileShape(128, 128, 64), 148, m.Policy.all_stream_k()),
        (m.ProblemSize(4096, 4096, 4096), m.TileShape(256, 256, 64), 74, m.Policy.hybrid(2, False)),
    ]:
        sc = scheduler.closed_form(size, tile, g, pol)
        items, offsets = scheduler.schedule_arrays(sc)
        cap = int(max(offsets[x + 1] - offsets[x] for x in range(g)))
        trace = torch.full((g, cap, _lib.TRACE_FIELDS), -1, dtype=torch.int64, device="cuda")
        counts = torch.zeros(g, dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib.skpp_schedule_trace_device(
            _lib.Problem(size.m, size.n, size.k), _lib.Tile(tile.blk_m, tile.blk_n, tile.blk_k),
            scheduler.policy_to_c(pol), g, trace.data_ptr(), cap, counts.data_ptr(),
            torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        tr, cn = trace.cpu().numpy(), counts.cpu().numpy()
        for x in range(g):
            lo, hi = int(offsets[x]), int(offsets[x + 1])
            assert cn[x] == hi - lo
            assert np.array_equal(tr[x, : hi - lo], items[lo:hi])


@pytest.mark.gpu
def test_selector_measures_candidates_and_runs_the_selected_config():
    """tiles.Selector on the device: Bloom candidates timed once, result bitwise vs the oracle."""
    import numpy as np
    import torch

    import paper_2408_11417_b200 as sk
    from oracle import gemm as ogemm
    from paper_2408_11417_b200 import tiles as tl

    t0, t1 = sk.TileShape(128, 128, 64), sk.TileShape(128, 128, 128)
    bank = tl.TileBank([t0, t1])
    size = sk.ProblemSize(512, 384, 2048)
    bank.insert(size, (t1, sk.Policy.all_stream_k()))
    rng = np.random.default_rng(5)
    a = ogemm.random_int_matrix(size.m, size.k, rng)
    b = ogemm.random_int_matrix(size.k, size.n, rng)
    at = torch.from_numpy(a).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
    sel = tl.Selector(bank)
    c = sel.gemm(at, bt)
    torch.cuda.synchronize()
    assert sel.measured == 1 and len(sel.cache) == 1
    assert sel.config(size, at, bt, c) in bank.candidates(size)
    assert np.array_equal(c.double().cpu().numpy(), ogemm.reference_gemm(a, b))


def test_joint_sweep_end_to_end_with_calibrated_priors(tmp_path):
    """sweep.main over two tiles on a tiny grid: per-tile records, tile bank with a
    calibrated cost-model prior per tile, and the off-grid selection summaries."""
    import json
    import os

    from paper_2408_11417_b200 import sweep
    from paper_2408_11417_b200 import tiles as tl

    out = str(tmp_path / "sw")
    rc = sweep.main(["--out", out, "--grid", "small", "--tiles", "128x128x64,128x128x128", "--reps", "2",
                     "--warmup", "1", "--max-gflop", "0.002", "--heldout", "8"])
    assert rc == 0
    summary = json.load(open(os.path.join(out, "summary.json")))
    assert set(summary["costmodel_priors"]) == {"128x128x64", "128x128x128"}
    assert "selection_offgrid_corners_and_model" in summary
    bank = tl.TileBank.load(os.path.join(out, "tilebank"))
    assert all(p is not None for p in bank.priors)
    size = sk().ProblemSize(3000, 5000, 7000)
    assert bank.prior_pick(size) in bank.query(size, nearest="corners+model")


def test_concurrent_streams_each_with_its_own_workspace():
    """Stream-K launches on three streams at once, no cross-stream ordering: each stream
    has its own fixup workspace and flags (per-stream cache), and every result stays
    bit-exact.  Persistent grids from different streams are dispatched in launch order,
    so a later grid never holds SMs an earlier grid's fixup waits on."""
    m = sk()
    rng = np.random.default_rng(21)
    streams = [torch.cuda.Stream() for _ in range(3)]
    cases = [((512, 512, 8192), m.Policy.all_stream_k(), m.TileShape(128, 128, 64)),
             ((300, 704, 5000), m.Policy.hybrid(1), m.TileShape(128, 128, 128)),
             ((600, 392, 4000), m.Policy.hybrid(2), m.TileShape(256, 256, 128))]
    plans, wants = [], []
    for s, ((mm, nn, kk), pol, tile) in zip(streams, cases):
        a = ogemm.random_int_matrix(mm, kk, rng)
        b = ogemm.random_int_matrix(kk, nn, rng)
        at = torch.from_numpy(a).to(torch.bfloat16).cuda()
        bt = torch.from_numpy(b).to(torch.bfloat16).cuda()
        c = torch.zeros(mm, nn, device="cuda")
        with torch.cuda.stream(s):
            plans.append(m.GemmPlan(at, bt, c, pol, tile))
        wants.append(ogemm.reference_gemm(a, b))
    torch.cuda.synchronize()
    for _ in range(40):
        for s, p in zip(streams, plans):
            with torch.cuda.stream(s):
                p.launch()
    torch.cuda.synchronize()
    for p, want in zip(plans, wants):
        assert np.array_equal(p.c.double().cpu().numpy(), want)


def test_sweep_cold_timing_rotates_operand_sets():
    """MeasureParams(cold=True): sizes whose operands fit in L2 are timed rotating over
    distinct operand sets (> 4 x L2 in total); the record is a normal ranked TuneRecord, and a
    rotated plan computes the same product as the pool's plan (views carved from the cold pool)."""
    import paper_2408_11417_b200 as m
    from paper_2408_11417_b200 import sweep

    size = m.ProblemSize(512, 2048, 2048)
    params = sweep.MeasureParams(warmup=2, reps=5, cold=True)
    n = sweep.cold_sets(size, params)
    assert 2 <= n <= params.cold_max_sets
    tile = m.TileShape(128, 128, 128)
    rec, = sweep.tune_sizes([size], tile, None, None, params)
    assert len(rec.costs) == 7 and all(e.makespan > 0 for _, e in rec.costs)
    warm, = sweep.tune_sizes([size], tile, None, None, sweep.MeasureParams(warmup=2, reps=5))
    best = lambda r: min(e.makespan for _, e in r.costs)  # noqa: E731
    assert best(rec) >= 0.7 * best(warm)  # cold is not (much) faster than warm
    pool = sweep._cold_pool(params)
    (a, b, c), = pool.sets(size, 1)
    a.copy_(torch.randint(-8, 9, a.shape, device="cuda").to(a.dtype))
    b.copy_(torch.randint(-8, 9, b.shape, device="cuda").to(b.dtype))
    m.GemmPlan(a, b, c, m.Policy.hybrid(1), tile).launch()
    torch.cuda.synchronize()
    assert torch.equal(c.double(), a.double() @ b.double())


def test_execute_schedule_reuses_plans_for_repeated_shapes():
    """Repeated execute_schedule calls of one shape skip the plan build (the cached plan is keyed
    by the operands' device addresses, strides and dtypes, and holds no tensor references);
    results stay exact, and a different shape or policy builds its own plan."""
    m = sk()
    from paper_2408_11417_b200 import executor as ex

    size, tile = m.ProblemSize(256, 512, 1024), m.TileShape(128, 128, 64)
    a, b, sched = instance(size, tile, 148, m.Policy.hybrid(1), seed=21)
    want = ogemm.reference_gemm(a, b)
    at, bt = torch.from_numpy(a).to(torch.bfloat16).pin_memory(), torch.from_numpy(b).to(torch.bfloat16).pin_memory()
    before = dict(ex._plan_cache_stats)
    for _ in range(5):
        got = m.execute_schedule(at, bt, sched, tile, size)
        assert np.array_equal(got.double().numpy(), want)
    assert ex._plan_cache_stats["hits"] - before["hits"] >= 3
    size2 = m.ProblemSize(256, 384, 1024)
    a2, b2, sched2 = instance(size2, tile, 148, m.Policy.all_stream_k(), seed=22)
    got2 = m.execute_schedule(a2, b2, sched2, tile, size2)
    assert np.array_equal(got2, ogemm.reference_gemm(a2, b2))
    assert len(ex._PLAN_CACHE) <= ex._PLAN_CACHE_MAX
