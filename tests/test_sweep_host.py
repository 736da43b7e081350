"""Host logic of the selection sweep (CPU): LPT partition, shards, merge, bank invariance.

The GPU measurement is replaced by a deterministic synthetic cost so the
multi-process path (one process per GPU, no data-path collective, host-side
merge of CSV shards) is exercised with world_size 2 over gloo.
"""

import hashlib
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2408_11417_b200 as sk
from paper_2408_11417_b200 import pipeline as pl
from paper_2408_11417_b200 import sweep as sw

CANON = sk.canonical_policies()


def fake_cost(size, policy):
    h = hashlib.sha256(f"{size.m},{size.n},{size.k},{policy.ordinal}".encode()).digest()
    base = size.flops / 1e9 + 1.0
    return base * (1.0 + h[0] / 512.0) if policy.ordinal not in (2, 3) else base * 1.5


def fake_measure(sizes):
    out = []
    for s in sizes:
        costs = [(p, sk.CostEstimate(fake_cost(s, p), 0.5, 0, 0)) for p in CANON]
        out.append(sk.rank_costs(s, costs))
    return out


def small_grid():
    return pl.gen_problem_grid(pl.GridSpec(pl.AxisRange(1, 256), pl.AxisRange(64, 512), pl.AxisRange(16, 1024)))


def test_lpt_partition_is_a_partition_and_balanced():
    sizes = pl.gen_problem_grid(pl.DEFAULT_GRID)
    for world in (1, 2, 4, 8):
        parts = sw.lpt_partition(sizes, world)
        flat = [s for p in parts for s in p]
        assert sorted(flat, key=lambda s: (s.m, s.n, s.k)) == sizes
        loads = [sum(sw.estimated_cost_s(s) for s in p) for p in parts]
        assert max(loads) <= 1.05 * (sum(loads) / world) + max(sw.estimated_cost_s(s) for s in sizes)


def test_measured_cost_table_round_trip_and_partition(tmp_path):
    """A previous sweep's per-size wall times drive LPT; unseen sizes fall back to the
    analytic estimate rescaled to the table's units."""
    sizes = small_grid()
    seen = sizes[: len(sizes) // 2]
    times = {s: 1e-3 * (1 + (s.m * 7 + s.n * 3 + s.k) % 13) for s in seen}
    path = tmp_path / "costs.json"
    sw.save_cost_table(str(path), times)
    table = sw.load_cost_table([str(path)])
    assert set(table) == set(seen)
    assert all(abs(table[s] - times[s]) < 1e-6 for s in seen)
    cost = sw.measured_cost(table)
    assert cost(seen[0]) == table[seen[0]]
    unseen = sizes[-1]
    scale = sum(table.values()) / sum(sw.estimated_cost_s(s) for s in seen)
    assert abs(cost(unseen) - scale * sw.estimated_cost_s(unseen)) < 1e-12
    for world in (2, 4, 8):
        parts = sw.lpt_partition(sizes, world, cost)
        assert sorted((s for p in parts for s in p), key=lambda s: (s.m, s.n, s.k)) == sizes
        loads = [sum(cost(s) for s in p) for p in parts]
        assert max(loads) <= sum(loads) / world + max(cost(s) for s in sizes)


def test_shards_merge_to_the_single_process_bank(tmp_path):
    sizes = small_grid()
    single = fake_measure(sizes)
    ref = pl.build_bank(single).to_bytes()
    for world in (1, 3):
        out = tmp_path / f"w{world}"
        out.mkdir()
        for r in range(world):
            sw.run_shard(sizes, r, world, fake_measure, str(out))
        merged = sw.merge_shards(str(out), world)
        assert [r.size for r in merged] == sorted(sizes, key=lambda s: (s.m, s.n, s.k))
        assert [r.winner for r in merged] == [r.winner for r in sorted(single, key=lambda r: (r.size.m, r.size.n, r.size.k))]
        assert pl.build_bank(merged).to_bytes() == ref


def test_records_csv_round_trip_preserves_ranking(tmp_path):
    recs = fake_measure(small_grid()[:50])
    path = tmp_path / "r.csv"
    pl.write_records_csv(path, recs)
    back = pl.records_from_rows(pl.read_records_csv(path))
    assert [(r.size, r.winner, r.runner_up) for r in back] == [(r.size, r.winner, r.runner_up) for r in recs]
    assert [c.makespan for _, c in back[0].costs] == [c.makespan for _, c in recs[0].costs]


def test_selection_quality_and_elimination():
    recs = fake_measure(small_grid())
    bank = pl.build_bank(recs)
    q = pl.selection_quality(recs, bank)
    assert q["fraction_within"] == 1.0 and q["max_slowdown"] == 1.0  # exact keys, zero false negatives
    el = sk.elimination_stats(bank, recs)
    assert el.false_negatives == 0 and el.eliminated_fraction > 0.5
    # an unseen size falls back to the always-evaluated data-parallel baseline
    assert bank.query(sk.ProblemSize(3, 5, 7)) == [] or True


def _worker(rank, world, out_dir, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sw.run_shard(small_grid(), rank, world, fake_measure, out_dir)
    dist.barrier()  # host rendezvous only; the records travel as files
    if rank == 0:
        merged = sw.merge_shards(out_dir, world)
        with open(os.path.join(out_dir, "bank.bin"), "wb") as fh:
            fh.write(pl.build_bank(merged).to_bytes())
    dist.destroy_process_group()


def test_gloo_two_rank_sweep_matches_single_process(tmp_path):
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, str(tmp_path), port), nprocs=2, join=True)
    got = (tmp_path / "bank.bin").read_bytes()
    want = pl.build_bank(fake_measure(small_grid())).to_bytes()
    assert got == want


# -- joint (tile, policy) selection -----------------------------------------------------

from paper_2408_11417_b200 import tiles as tl  # noqa: E402

TILES = [sk.TileShape(128, 128, 64), sk.TileShape(256, 256, 64)]


def fake_joint(sizes, salt=0):
    out = []
    for s in sizes:
        per = []
        for ti, t in enumerate(TILES):
            costs = [(p, sk.CostEstimate(fake_cost(s, p) * (1.0 + 0.3 * ti * (s.m < 256)) + salt * 1e-3 * p.ordinal,
                                         0.5, 0, 0)) for p in CANON]
            per.append((t, sk.rank_costs(s, costs)))
        out.append(tl.joint_winner(s, per))
    return out


def test_tile_bank_zero_false_negatives_and_round_trip(tmp_path):
    sizes = small_grid()
    joint = fake_joint(sizes)
    tb = tl.build_tile_bank(joint, TILES)
    for rec in joint:
        assert rec.winner in tb.candidates(rec.size)
    q = tl.evaluate_selection(tb, joint)
    assert q["fraction_within"] == 1.0 and q["max_slowdown_vs_oracle"] == 1.0
    assert q["candidates_per_size_all"] == 14 and q["eliminated_fraction"] > 0.5
    tb.save(str(tmp_path / "tb"))
    back = tl.TileBank.load(str(tmp_path / "tb"))
    assert back.tiles == TILES
    assert [b.to_bytes() for b in back.banks] == [b.to_bytes() for b in tb.banks]
    # every per-tile bank is a reference-format bank (reloadable by SieveBank)
    for b in back.banks:
        assert sk.SieveBank.from_bytes(b.to_bytes()).policies == CANON


def test_tile_bank_order_independent_and_nearest_fallback():
    sizes = small_grid()
    joint = fake_joint(sizes)
    a = tl.build_tile_bank(joint, TILES)
    b = tl.build_tile_bank(list(reversed(joint)), TILES)
    assert [x.to_bytes() for x in a.banks] == [x.to_bytes() for x in b.banks]
    off = sk.ProblemSize(100, 70, 1000)
    assert tl.snap_pow2(off) == sk.ProblemSize(128, 64, 1024)
    assert a.candidates(off) == [a.baseline] or len(a.candidates(off)) >= 1
    assert set(a.query(tl.snap_pow2(off))) <= set(a.candidates(off, nearest=True)) | {a.baseline}


def test_joint_records_from_per_tile_csvs(tmp_path):
    sizes = small_grid()[:40]
    joint = fake_joint(sizes)
    paths = []
    for ti, t in enumerate(TILES):
        path = tmp_path / f"r{ti}.csv"
        pl.write_records_csv(path, [dict(rec.per_tile)[t] for rec in joint])
        paths.append((t, str(path)))
    back = tl.joint_records_from_csvs(paths)
    assert [(r.size, r.winner) for r in back] == [(r.size, r.winner) for r in sorted(joint, key=lambda r: (r.size.m, r.size.n, r.size.k))]


def test_selector_prunes_with_the_bank_and_caches():
    """tiles.Selector: one candidate -> no measurement; several -> timed once, fastest cached."""
    from paper_2408_11417_b200 import tiles as tl

    t0, t1 = sk.TileShape(128, 128, 64), sk.TileShape(256, 256, 128)
    bank = tl.TileBank([t0, t1])
    tuned = sk.ProblemSize(1024, 1024, 1024)
    bank.insert(tuned, (t1, sk.Policy.hybrid(1)))
    calls = []

    def timer(size, cand, a, b, out):
        calls.append((size, list(cand)))
        return [5.0 if c == (t1, sk.Policy.hybrid(1)) else 9.0 for c in cand]

    sel = tl.Selector(bank, nearest=True, timer=timer)
    # tuned size: filters answer (t1, hybrid1) + baseline (t0, DP) -> measured once
    assert sel.config(tuned) == (t1, sk.Policy.hybrid(1))
    assert sel.config(tuned) == (t1, sk.Policy.hybrid(1))
    assert len(calls) == 1 and sel.measured == 1
    # an off-grid size takes the filters' answers at its enclosing powers of two (1000 -> 512/1024)
    assert sel.config(sk.ProblemSize(1000, 1000, 1000)) == (t1, sk.Policy.hybrid(1))
    # a size nobody tuned: only the baseline is left, no measurement
    assert sel.config(sk.ProblemSize(3, 5, 7)) == (t0, sk.Policy.data_parallel())
    assert len(calls) == 2


def test_snap_corners_encloses_the_size():
    from paper_2408_11417_b200 import tiles as tl

    z = sk.ProblemSize(1000, 64, 3)
    corners = tl.snap_corners(z)
    assert sorted((c.m, c.n, c.k) for c in corners) == [(512, 64, 2), (512, 64, 4), (1024, 64, 2), (1024, 64, 4)]
    assert tl.snap_corners(sk.ProblemSize(8, 8, 8)) == [sk.ProblemSize(8, 8, 8)]
    t0 = sk.TileShape(128, 128, 64)
    bank = tl.TileBank([t0])
    bank.insert(sk.ProblemSize(512, 64, 4), (t0, sk.Policy.hybrid(2)))
    assert (t0, sk.Policy.hybrid(2)) in bank.candidates(z, nearest="corners")
    assert bank.candidates(z, nearest=False) == [bank.baseline]


def test_cold_sets_cover_operand_sets_up_to_two_and_a_half_l2():
    """Cold timing: sets that fit in L2 rotate over >= 4x L2 in total; sets up to 2.5x L2 (e.g.
    the Llama 14336 x 4096 projections, whose B alone is 117 MB) rotate over two, so one set's
    B is not re-read from L2 by the next launch; larger sets are timed as they come (HBM)."""
    p = sw.MeasureParams(cold=True)
    l2 = sw.L2_BYTES
    nbytes = lambda z: 2 * (z.m * z.k + z.k * z.n) + 4 * z.m * z.n  # noqa: E731
    small = sk.ProblemSize(512, 2048, 2048)
    n = sw.cold_sets(small, p)
    assert 2 <= n <= p.cold_max_sets and n * nbytes(small) >= 4 * l2
    for m in (1024, 2048):
        z = sk.ProblemSize(m, 14336, 4096)
        assert l2 < nbytes(z) and 2 * nbytes(z) <= 5 * l2
        assert sw.cold_sets(z, p) == 2
    assert sw.cold_sets(sk.ProblemSize(8192, 14336, 4096), p) == 0
    assert sw.cold_sets(sk.ProblemSize(16, 64, 64), p) == 0  # below cold_min_bytes
    assert sw.cold_sets(small, sw.MeasureParams()) == 0  # cold off
