"""Oracle restatement of the reference hashing and Bloom sieve (gemmsched hashing.py, sieve.py).

Pure Python (arbitrary-precision ints masked to 64 bits), zlib for CRC32.
"""

from __future__ import annotations

import math
import struct
import zlib

M64 = (1 << 64) - 1
C1, C2 = 0x87C37B91114253D5, 0x4CF5AD432745937F


def _rotl(v, r):
    return ((v << r) | (v >> (64 - r))) & M64


def _fmix(k):
    k ^= k >> 33
    k = (k * 0xFF51AFD7ED558CCD) & M64
    k ^= k >> 33
    k = (k * 0xC4CEB9FE1A85EC53) & M64
    k ^= k >> 33
    return k


def murmur3_x64_128(data: bytes, seed: int):
    """hashing.py:41-91 (Appleby's MurmurHash3_x64_128; seed zero-extended to both halves)."""
    h1 = h2 = seed & 0xFFFFFFFF
    n = len(data)
    nb = n // 16
    for i in range(nb):
        k1, k2 = struct.unpack_from("<QQ", data, 16 * i)
        k1 = (_rotl((k1 * C1) & M64, 31) * C2) & M64
        h1 ^= k1
        h1 = (_rotl(h1, 27) + h2) & M64
        h1 = (h1 * 5 + 0x52DCE729) & M64
        k2 = (_rotl((k2 * C2) & M64, 33) * C1) & M64
        h2 ^= k2
        h2 = (_rotl(h2, 31) + h1) & M64
        h2 = (h2 * 5 + 0x38495AB5) & M64
    tail = data[16 * nb:]
    if len(tail) > 8:
        k2 = int.from_bytes(tail[8:], "little")
        h2 ^= (_rotl((k2 * C2) & M64, 33) * C1) & M64
    if tail:
        k1 = int.from_bytes(tail[:8], "little")
        h1 ^= (_rotl((k1 * C1) & M64, 31) * C2) & M64
    h1 ^= n
    h2 ^= n
    h1 = (h1 + h2) & M64
    h2 = (h2 + h1) & M64
    h1, h2 = _fmix(h1), _fmix(h2)
    h1 = (h1 + h2) & M64
    h2 = (h2 + h1) & M64
    return h1, h2


def key(m: int, n: int, k: int) -> bytes:
    """types.py:48-55."""
    return struct.pack("<QQQ", m, n, k)


def filter_params(capacity: int, fp: float):
    """sieve.py:63-78 (code, not SPEC.md:377 — see SURVEY Appendix B.1)."""
    m_raw = math.ceil(-capacity * math.log(fp) / (math.log(2) ** 2))
    kh = math.floor((m_raw / capacity) * math.log(2) + 0.5)
    return ((m_raw + 63) // 64) * 64, max(1, min(32, kh))


def filter_seed(index: int) -> int:
    """sieve.py:81-83 — by bank position."""
    return (0x9E3779B9 * (index + 1)) & 0xFFFFFFFF


def probes(k24: bytes, seed: int, m_bits: int, k_hashes: int):
    """sieve.py:86-97."""
    h1, h2 = murmur3_x64_128(k24, seed)
    return [((h1 + i * h2) & M64) % m_bits for i in range(k_hashes)]


def bloom_insert(bits: bytearray, k24: bytes, seed: int, m_bits: int, k_hashes: int) -> None:
    """sieve.py:150-153: LSB-first bit i -> byte i >> 3, bit i & 7."""
    for idx in probes(k24, seed, m_bits, k_hashes):
        bits[idx >> 3] |= 1 << (idx & 7)


def bloom_contains(bits, k24: bytes, seed: int, m_bits: int, k_hashes: int) -> bool:
    """sieve.py:155-159."""
    return all(bits[i >> 3] >> (i & 7) & 1 for i in probes(k24, seed, m_bits, k_hashes))


def policy_tag(kind: str, sk_batches: int, sk_first: bool):
    """sieve.py:169-181."""
    if kind == "data-parallel":
        return 0, 0, 0
    if kind == "all-streamk":
        return 6, 0, 0
    return sk_batches, sk_batches, int(sk_first)


def bank_bytes(filters) -> bytes:
    """sieve.py:325-336.  filters: list of (tag, sk_b, sk_f, seed, m_bits, k_hashes, n_ins, bits)."""
    buf = bytearray(b"SKPS") + struct.pack("<HH", 1, len(filters))
    for tag, skb, skf, seed, m_bits, kh, n_ins, bits in filters:
        buf += struct.pack("<BBBBIQIQ", tag, skb, skf, 0, seed, m_bits, kh, n_ins)
        buf += bytes(bits)
    buf += struct.pack("<I", zlib.crc32(bytes(buf)))
    return bytes(buf)


class Bank:
    """A canonical-order bank (SieveBank, sieve.py:200-313) over plain bytearrays."""

    def __init__(self, policies, capacity=10_000, fp=0.01):
        self.policies = list(policies)  # (kind, sk_batches, sk_first)
        self.m_bits, self.k = filter_params(capacity, fp)
        self.seeds = [filter_seed(i) for i in range(len(self.policies))]
        self.bits = [bytearray(self.m_bits // 8) for _ in self.policies]
        self.n_ins = [0] * len(self.policies)

    def insert(self, m, n, k, policy):
        i = self.policies.index(policy)
        bloom_insert(self.bits[i], key(m, n, k), self.seeds[i], self.m_bits, self.k)
        self.n_ins[i] += 1

    def query(self, m, n, k):
        kk = key(m, n, k)
        return [p for i, p in enumerate(self.policies)
                if bloom_contains(self.bits[i], kk, self.seeds[i], self.m_bits, self.k)]

    def to_bytes(self) -> bytes:
        rows = []
        for i, p in enumerate(self.policies):
            rows.append((*policy_tag(*p), self.seeds[i], self.m_bits, self.k, self.n_ins[i], self.bits[i]))
        return bank_bytes(rows)


CANONICAL = [("data-parallel", 0, False)] + [("hybrid", s, True) for s in range(1, 6)] + [("all-streamk", 0, False)]


def sort_key(policy):
    """types.py:147-154: (kind rank, sk_batches, 0 if sk_first else 1)."""
    kind, skb, skf = policy
    rank = {"data-parallel": 0, "hybrid": 1, "all-streamk": 2}[kind]
    return (rank, skb, 0 if skf else 1)


def pick_winner(costs):
    """costmodel.py:141-164 ranking: ascending (cost, sort_key); returns (winner, runner_up, gain)."""
    ranked = sorted(costs, key=lambda pc: (pc[1], sort_key(pc[0])))
    w, r = ranked[0], ranked[1] if len(ranked) > 1 else ranked[0]
    gain = (r[1] - w[1]) / r[1] if r[1] > 0 else 0.0
    return w[0], r[0], gain
