#!/usr/bin/env python
"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Run in the build container only (the GPU box has no /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every value below is produced by ``gemmsched`` itself (the reference package,
pkg/src/gemmsched) — murmur hashes, filter sizing, schedules, coverage audits,
bank bytes, query answers, parse errors, elimination statistics — so the
committed fixtures pin both the oracle restatement (tests/test_oracle_golden.py)
and the product (tests/test_host_parity.py, tests/test_gpu_*.py) to the
reference's behaviour.  Literal known-answer vectors from the reference's own
tests are included verbatim under "kat".
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import gemmsched as G  # noqa: E402
from gemmsched import hashing as GH  # noqa: E402
from gemmsched import sieve as GS  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def pol_tuple(p):
    return [p.kind.value, p.sk_batches, bool(p.sk_first)]


def pol_from(t):
    kind, s, first = t
    if kind == "data-parallel":
        return G.Policy.data_parallel()
    if kind == "all-streamk":
        return G.Policy.all_stream_k()
    return G.Policy.hybrid(s, first)


def sched_rows(sched):
    rows = []
    for wg in sched.assignments:
        rows.append([[it.tile_idx, it.local_iter_begin, it.local_iter_end,
                      0 if it.write_mode is G.WriteMode.FULL_STORE else 1,
                      0 if it.phase is G.Phase.STREAM_K else 1] for it in wg])
    return rows


def sched_digest(rows) -> str:
    txt = "|".join(";".join(",".join(str(v) for v in item) for item in wg) for wg in rows)
    return hashlib.sha256(txt.encode()).hexdigest()


def _tmp_csv(text: str) -> str:
    import tempfile

    fd, path = tempfile.mkstemp(suffix=".csv")
    with os.fdopen(fd, "w") as fh:
        fh.write(text)
    return path


def main() -> None:
    rng = np.random.default_rng(20240821)
    out: dict = {"generator": "tests/golden/make_golden.py", "reference": "gemmsched 0.1.0 (pkg/src/gemmsched)"}

    # -- literal KATs from the reference's own tests (tests/test_hashing.py:12-41, test_sieve.py:41-45)
    out["kat"] = {
        "murmur": [
            ["", 0, [0, 0]],
            ["", 42, [17305828677633410339, 15060430851467758521]],
            ["a", 0, [9607679276477937801, 16624257681780017498]],
            ["foo", 0, [16316970633193145697, 9128664383759220103]],
            ["hello", 0, [14688674573012802306, 6565844092913065241]],
            ["hello", 123, [3016954156110693643, 1043184066639555970]],
            ["hello, world", 321, [7533679572817601133, 11811685183640001006]],
            ["The quick brown fox jumps over the lazy dog", 0, [16378391709484522348, 8809951995912426311]],
            ["0123456789abcdef0123456789abcdefABCDEFGHIJKL", 99, [1941902248655048229, 2676132337890212611]],
            ["abcdefghijklmnop", 7, [4448784618183325535, 4093737273664872544]],
            ["abcdefghijklmnopqrstuvwx", 7, [15408725433791075941, 5189007623493139958]],
        ],
        "triple": [
            [[1, 1, 1], 0, [10952789098337097608, 13281419438922705407]],
            [[1, 64, 16], 0, [12576440658899820686, 240203222842308453]],
            [[256, 512, 128], 1, [8542782460663049281, 8187488057708540397]],
            [[1024, 1024, 1024], 2654435769, [13467307367258508987, 8586790828570743759]],
            [[8192, 8192, 65536], 305419896, [14184364134445420777, 10821718848681073201]],
        ],
        "smhasher_x64_128": 0x6384BA69,
        "filter_params": [[10000, 0.01, 95872, 7], [1, 0.5, 64, 1]],
        "key_256_512_128_hex": G.encode_key(G.ProblemSize(256, 512, 128)).hex(),
        "bank_file_bytes_default": 8 + 7 * (28 + 11984) + 4,
    }
    for lit, seed, want in out["kat"]["murmur"]:
        assert list(GH.murmur3_x64_128(lit.encode(), seed)) == want
    for triple, seed, want in out["kat"]["triple"]:
        assert list(GH.murmur3_x64_128(G.encode_key(G.ProblemSize(*triple)), seed)) == want

    # -- murmur on random data (all block/tail combinations) and 24-byte keys incl. u64 extremes
    mm = []
    for _ in range(300):
        data = rng.bytes(int(rng.integers(0, 80)))
        seed = int(rng.integers(0, 2**32))
        mm.append([data.hex(), seed, list(GH.murmur3_x64_128(data, seed))])
    out["murmur_random"] = mm
    h24 = []
    hi = 2**64 - 1
    for m, n, k in [(hi, 1, 1), (1, hi, 1), (hi, hi, hi)] + [
        tuple(int(v) for v in rng.integers(1, 2**63, size=3, dtype=np.uint64)) for _ in range(100)
    ]:
        seed = int(rng.integers(0, 2**32))
        h24.append([[m, n, k], seed, list(GH.hash24(m, n, k, seed))])
    out["hash24"] = h24

    # -- filter sizing / seeds / probes
    fp = []
    for _ in range(300):
        cap = int(rng.integers(1, 10**6))
        f = float(rng.uniform(1e-6, 0.5))
        fp.append([cap, f, *GS.filter_params(cap, f)])
    out["filter_params"] = fp
    out["filter_seeds"] = [GS.filter_seed(i) for i in range(16)]
    pr = []
    for _ in range(100):
        m, n, k = (int(v) for v in rng.integers(1, 2**40, size=3))
        seed = int(rng.integers(0, 2**32))
        mb = int(rng.choice([64, 1024, 95872, 1 << 20]))
        kh = int(rng.integers(1, 33))
        pr.append([[m, n, k], seed, mb, kh, GS.hash_probes(G.encode_key(G.ProblemSize(m, n, k)), seed, mb, kh)])
    out["probes"] = pr

    # -- schedules: BASELINE configs at the B200 geometry plus random instances
    canon = G.canonical_policies()
    extra = [G.Policy.hybrid(2, sk_first=False), G.Policy.hybrid(7), G.Policy.hybrid(3, sk_first=False)]
    scheds = []

    def add_sched(m, n, k, bm, bn, bk, g, pol, keep_items):
        s = G.build_schedule(G.ProblemSize(m, n, k), G.TileShape(bm, bn, bk), G.HardwareModel(g, 1), pol)
        rows = sched_rows(s)
        rec = {"size": [m, n, k], "tile": [bm, bn, bk], "g": g, "policy": pol_tuple(pol),
               "n_items": sum(len(w) for w in rows), "digest": sched_digest(rows)}
        if keep_items:
            rec["items"] = rows
        scheds.append(rec)

    for (m, n, k) in [(1024, 1024, 1024), (512, 512, 16384)]:
        for tile in [(128, 128, 64), (128, 256, 64)]:
            for pol in canon + extra:
                add_sched(m, n, k, *tile, 148, pol, keep_items=(tile == (128, 128, 64)))
    for (m, n, k) in [(8192, 14336, 4096), (4096, 4096, 4096), (1, 64, 65536), (100, 75, 53), (1, 14336, 4096)]:
        for pol in canon + extra:
            add_sched(m, n, k, 128, 128, 64, 148, pol, keep_items=False)
    for i in range(400):
        m, n, k = (int(2 ** rng.uniform(0, 12)) for _ in range(3))
        bm, bn = (int(rng.choice([16, 32, 64, 128, 256])) for _ in range(2))
        bk = int(rng.choice([8, 16, 32, 64]))
        g = int(rng.integers(1, 513))
        pol = (canon + extra)[i % 10]
        add_sched(m, n, k, bm, bn, bk, g, pol, keep_items=(i < 40))
    out["schedules"] = scheds

    # -- coverage audits of mutated schedules (scheduler.py:257-291)
    cov = []
    for i in range(60):
        m, n, k = (int(2 ** rng.uniform(2, 10)) for _ in range(3))
        g = int(rng.integers(1, 40))
        pol = canon[i % 7]
        tile = G.TileShape(32, 32, 16)
        s = G.build_schedule(G.ProblemSize(m, n, k), tile, G.HardwareModel(g, 1), pol)
        rows = sched_rows(s)
        flat = [(w, j) for w, wg in enumerate(rows) for j in range(len(wg))]
        mode = ["none", "drop", "dup", "shift"][i % 4]
        if mode != "none" and flat:
            w, j = flat[int(rng.integers(0, len(flat)))]
            item = rows[w][j]
            if mode == "drop":
                del rows[w][j]
            elif mode == "dup":
                rows[(w + 1) % len(rows)].append(list(item))
            else:
                t, kb, ke, wm, ph = item
                if ke - kb > 1:
                    rows[w][j] = [t, kb, ke - 1, wm, ph]
                else:
                    rows[w][j] = [t, kb, ke + 1, wm, ph]
        items = tuple(tuple(G.WorkItem(t, kb, ke, G.WriteMode.FULL_STORE if wm == 0 else G.WriteMode.ATOMIC_PARTIAL,
                                       G.Phase.STREAM_K if ph == 0 else G.Phase.DATA_PARALLEL)
                            for t, kb, ke, wm, ph in wg) for wg in rows)
        rep = G.validate_schedule(G.Schedule(s.grid, s.g, s.policy, items))
        cov.append({"grid": [s.grid.m_tiles, s.grid.n_tiles, s.grid.iters_per_tile, s.grid.total_tiles,
                             s.grid.total_iters], "g": g, "policy": pol_tuple(pol), "items": rows,
                    "report": [rep.covered_once, rep.duplicates, rep.gaps]})
    out["coverage"] = cov

    # -- banks: a small bank with full bytes, queries on members and non-members
    bank = G.SieveBank(canon, capacity=200, fp_target=0.01)
    inserted = []
    for _ in range(150):
        size = [int(v) for v in rng.integers(1, 2**20, size=3)]
        pol = canon[int(rng.integers(0, 7))]
        bank.insert(G.ProblemSize(*size), pol)
        inserted.append([size, pol.ordinal])
    probes = [s for s, _ in inserted] + [[int(v) for v in rng.integers(1, 2**20, size=3)] for _ in range(300)]
    out["small_bank"] = {
        "capacity": 200, "fp_target": 0.01, "inserts": inserted, "hex": bank.to_bytes().hex(),
        "queries": [[s, [p.ordinal for p in bank.query(G.ProblemSize(*s))]] for s in probes],
    }

    # -- the reference's default CLI artefact: cost-model winners over the paper grid
    sizes = G.gen_problem_grid(G.DEFAULT_GRID)
    recs = G.tune_grid(sizes, G.DEFAULT_TILE, G.DEFAULT_HW)
    big = G.build_bank(recs)
    el = G.elimination_stats(big, recs)
    out["default_tune"] = {
        "grid_len": len(sizes), "first": [sizes[0].m, sizes[0].n, sizes[0].k],
        "last": [sizes[-1].m, sizes[-1].n, sizes[-1].k],
        "winners": [r.winner.ordinal for r in recs],
        "bank_sha256": hashlib.sha256(big.to_bytes()).hexdigest(),
        "bank_bytes": len(big.to_bytes()),
        "elimination": [el.eliminated_fraction, el.false_negatives, el.evaluations_saved],
        "query_masks_first_200": [[p.ordinal for p in big.query(s)] for s in sizes[:200]],
    }

    # -- malformed files and the exception class the reference raises
    good = bank.to_bytes()
    bad_cases = []

    def expect(data: bytes, label: str):
        try:
            G.SieveBank.from_bytes(data)
            err = None
        except GS.SieveFormatError as exc:
            err = type(exc).__name__
        except ValueError as exc:
            err = "ValueError:" + str(exc)
        bad_cases.append([label, data.hex(), err])

    expect(good, "good")
    expect(good[:11], "short")
    expect(b"XKPS" + good[4:], "magic")
    expect(good[:4] + (2).to_bytes(2, "little") + good[6:], "version")
    expect(good[:6] + (0).to_bytes(2, "little") + good[8:], "count0")
    expect(good[:-1], "truncated-crc")
    expect(good[:40], "truncated-bits")
    expect(good[:20], "truncated-header")
    expect(good + b"\0", "trailing")
    flipped = bytearray(good)
    flipped[100] ^= 0x10
    expect(bytes(flipped), "bitflip")
    reserved = bytearray(good)
    reserved[8 + 3] = 1
    expect(bytes(reserved), "reserved")
    tagbad = bytearray(good)
    tagbad[8] = 3  # tag 3 with sk_batches 0 -> unrecognized parameterless tag (DP filter is first)
    expect(bytes(tagbad), "tag")
    out["parse_cases"] = bad_cases

    # -- ranking rule on synthetic costs (costmodel.py:158)
    ranks = []
    for _ in range(100):
        costs = [(canon[i], float(rng.choice([1.0, 2.0, 3.0, float(rng.uniform(1, 3))]))) for i in range(7)]
        ordered = sorted(costs, key=lambda pc: (pc[1], pc[0].sort_key()))
        ranks.append([[c for _, c in costs], ordered[0][0].ordinal, ordered[1][0].ordinal])
    out["ranking"] = ranks

    # -- records CSV + report of a small cost-model tune (reference pipeline.py:149-313)
    small = G.gen_problem_grid(G.GridSpec(G.AxisRange(1, 256), G.AxisRange(64, 256), G.AxisRange(16, 1024)))
    recs_small = G.tune_grid(small, G.TileShape(64, 64, 32), G.HardwareModel(13, 1))
    out["report_case"] = {
        "records_csv": G.records_csv_text(recs_small),
        "report": G.build_report(G.read_records_csv(_tmp_csv(G.records_csv_text(recs_small)))),
        "report_tol": G.build_report(G.read_records_csv(_tmp_csv(G.records_csv_text(recs_small))), [0.0, 0.3]),
    }

    with open(OUT, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
