"""Pin the oracle restatement against the reference's golden vectors (CPU).

The fixtures in tests/golden/golden.json were produced by running the
reference package itself (tests/golden/make_golden.py) plus the literal
known-answer vectors of its own test-suite; passing here means the oracle
used by the GPU parity tests behaves like the reference.
"""

import hashlib
import json
import os
import struct

import numpy as np
import pytest

from oracle import gemm as og
from oracle import schedule as osc
from oracle import sieve as osv

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def digest(rows):
    txt = "|".join(";".join(",".join(str(v) for v in item) for item in wg) for wg in rows)
    return hashlib.sha256(txt.encode()).hexdigest()


def test_murmur_kats():
    for lit, seed, want in GOLD["kat"]["murmur"]:
        assert list(osv.murmur3_x64_128(lit.encode(), seed)) == want
    for triple, seed, want in GOLD["kat"]["triple"]:
        assert list(osv.murmur3_x64_128(osv.key(*triple), seed)) == want


def test_murmur_smhasher_verification():
    # tests/test_hashing.py:70-81 (SMHasher VerificationTest)
    buf = bytearray()
    for i in range(256):
        h1, h2 = osv.murmur3_x64_128(bytes(range(i)), 256 - i)
        buf += struct.pack("<QQ", h1, h2)
    assert osv.murmur3_x64_128(bytes(buf), 0)[0] & 0xFFFFFFFF == GOLD["kat"]["smhasher_x64_128"]


def test_murmur_random_and_hash24():
    for hexdata, seed, want in GOLD["murmur_random"]:
        assert list(osv.murmur3_x64_128(bytes.fromhex(hexdata), seed)) == want
    for (m, n, k), seed, want in GOLD["hash24"]:
        assert list(osv.murmur3_x64_128(osv.key(m, n, k), seed)) == want


def test_filter_params_seeds_probes():
    for cap, fp, mb, kh in GOLD["kat"]["filter_params"] + GOLD["filter_params"]:
        assert osv.filter_params(cap, fp) == (mb, kh)
    assert [osv.filter_seed(i) for i in range(16)] == GOLD["filter_seeds"]
    for (m, n, k), seed, mb, kh, want in GOLD["probes"]:
        assert osv.probes(osv.key(m, n, k), seed, mb, kh) == want


def _pol(t):
    return t[0], t[1], t[2]


def test_schedules_match_reference():
    for rec in GOLD["schedules"]:
        m, n, k = rec["size"]
        bm, bn, bk = rec["tile"]
        kind, s, first = rec["policy"]
        rows = osc.build_schedule(m, n, k, bm, bn, bk, rec["g"], kind, s, first)
        rows = [[list(it) for it in wg] for wg in rows]
        assert sum(len(w) for w in rows) == rec["n_items"], rec
        assert digest(rows) == rec["digest"], rec
        if "items" in rec:
            assert rows == rec["items"]


def test_coverage_audit_matches_reference():
    for rec in GOLD["coverage"]:
        _, _, ipt, _, total = rec["grid"]
        got = osc.validate(rec["items"], ipt, total)
        assert list(got) == rec["report"]


def test_small_bank_bytes_and_queries():
    sb = GOLD["small_bank"]
    bank = osv.Bank(osv.CANONICAL, sb["capacity"], sb["fp_target"])
    for (m, n, k), ordinal in sb["inserts"]:
        bank.insert(m, n, k, osv.CANONICAL[ordinal])
    assert bank.to_bytes().hex() == sb["hex"]
    for (m, n, k), want in sb["queries"]:
        assert [osv.CANONICAL.index(p) for p in bank.query(m, n, k)] == want


def test_default_tune_bank_sha():
    dt = GOLD["default_tune"]
    ms = [1 << e for e in range(14)]
    ns = [1 << e for e in range(6, 14)]
    ks = [1 << e for e in range(4, 17)]
    sizes = [(m, n, k) for m in ms for n in ns for k in ks]
    assert len(sizes) == dt["grid_len"]
    bank = osv.Bank(osv.CANONICAL)
    for (m, n, k), w in sorted(zip(sizes, dt["winners"])):
        bank.insert(m, n, k, osv.CANONICAL[w])
    data = bank.to_bytes()
    assert len(data) == dt["bank_bytes"] == GOLD["kat"]["bank_file_bytes_default"]
    assert hashlib.sha256(data).hexdigest() == dt["bank_sha256"]


def test_ranking_rule():
    for costs, win, run in GOLD["ranking"]:
        w, r, _ = osv.pick_winner(list(zip(osv.CANONICAL, costs)))
        assert (osv.CANONICAL.index(w), osv.CANONICAL.index(r)) == (win, run)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_executor_bitwise(seed):
    rng = np.random.default_rng(seed)
    m, n, k = 100, 75, 53
    a = og.random_int_matrix(m, k, rng)
    b = og.random_int_matrix(k, n, rng)
    for kind, s, first in [("data-parallel", 0, False), ("hybrid", 3, True), ("all-streamk", 0, False)]:
        rows = osc.build_schedule(m, n, k, 64, 32, 16, 7, kind, s, first)
        got = og.execute_schedule(a, b, rows, m, n, k, 64, 32, 16, -(-n // 32))
        assert np.array_equal(got, og.reference_gemm(a, b))
