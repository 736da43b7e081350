"""Per-policy Bloom-filter bank: the Stream-K++ selection layer (host side).

Drop-in for ``gemmsched.sieve`` (reference ``sieve.py``), byte-compatible:
identical sizing (sieve.py:63-78), seeds by bank position (81-83), double
hashing probes ``((h1 + i*h2) mod 2^64) mod m_bits`` (86-97), LSB-first bit
packing (107-166), bank-order query answers (283-301), and the versioned
``SKPS`` file with CRC32 trailer and the same validation order and exception
classes (315-402).  Hashing, probing, membership, serialisation and parsing
run in C++ (libskpp.so); this module owns the numpy bit arrays and the
Python object model.
"""

from __future__ import annotations

import ctypes
import math
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .types import KEY_BYTES, Policy, PolicyKind, ProblemSize, canonical_policies, encode_key

MAGIC = b"SKPS"
FORMAT_VERSION = 1
DEFAULT_CAPACITY = 10_000
DEFAULT_FP_TARGET = 0.01
_MAX_HASHES = 32
_KEY = struct.Struct("<QQQ")


class SieveFormatError(ValueError):
    """A serialized bank is malformed."""


class BadMagicError(SieveFormatError):
    pass


class UnsupportedVersionError(SieveFormatError):
    pass


class ChecksumError(SieveFormatError):
    pass


class TruncatedError(SieveFormatError):
    pass


_FORMAT_ERRORS = {
    _lib.ETRUNCATED: TruncatedError,
    _lib.EBADMAGIC: BadMagicError,
    _lib.EVERSION: UnsupportedVersionError,
    _lib.EFORMAT: SieveFormatError,
    _lib.ECHECKSUM: ChecksumError,
}


def filter_params(capacity: int, fp_target: float) -> tuple[int, int]:
    """(m_bits, k_hashes) for a design load and false-positive target."""
    if capacity < 1:
        raise ValueError("capacity must be >= 1")
    if not 0.0 < fp_target < 1.0:
        raise ValueError("fp_target must be in (0, 1)")
    m_bits = ctypes.c_uint64()
    k = ctypes.c_uint32()
    _lib.check(_lib.lib.skpp_filter_params(capacity, float(fp_target), ctypes.byref(m_bits), ctypes.byref(k)))
    return int(m_bits.value), int(k.value)


def filter_seed(index: int) -> int:
    """32-bit seed of the filter at bank position ``index``."""
    return int(_lib.lib.skpp_filter_seed(index))


def hash_probes(key: bytes, seed: int, m_bits: int, k_hashes: int) -> list[int]:
    if len(key) != KEY_BYTES:
        raise ValueError(f"key must be {KEY_BYTES} bytes, got {len(key)}")
    if m_bits < 1 or k_hashes < 1:
        raise ValueError("m_bits and k_hashes must be >= 1")
    out = (ctypes.c_uint64 * k_hashes)()
    _lib.check(_lib.lib.skpp_hash_probes(bytes(key), seed & 0xFFFFFFFF, m_bits, k_hashes, out))
    return [int(v) for v in out]


def predicted_fp_rate(m_bits: int, k_hashes: int, n_inserted: int) -> float:
    """(1 - e^(-k n / m))^k."""
    if n_inserted <= 0:
        return 0.0
    return (1.0 - math.exp(-k_hashes * n_inserted / m_bits)) ** k_hashes


class BloomFilter:
    """m_bits packed LSB-first (bit i in byte i >> 3 at position i & 7), k probes."""

    __slots__ = ("m_bits", "k_hashes", "seed", "n_inserted", "bits")

    def __init__(
        self,
        m_bits: int,
        k_hashes: int,
        seed: int,
        *,
        bits: np.ndarray | None = None,
        n_inserted: int = 0,
    ):
        if m_bits < 64 or m_bits % 64:
            raise ValueError("m_bits must be a positive multiple of 64")
        if not 1 <= k_hashes <= _MAX_HASHES:
            raise ValueError(f"k_hashes must be in [1, {_MAX_HASHES}]")
        if not 0 <= seed <= 0xFFFFFFFF:
            raise ValueError("seed must fit in 32 bits")
        nbytes = m_bits // 8
        if bits is None:
            bits = np.zeros(nbytes, dtype=np.uint8)
        else:
            bits = np.ascontiguousarray(bits, dtype=np.uint8)
            if bits.shape != (nbytes,):
                raise ValueError(f"bit array must have {nbytes} bytes")
        self.m_bits = m_bits
        self.k_hashes = k_hashes
        self.seed = seed
        self.n_inserted = n_inserted
        self.bits = bits

    @classmethod
    def for_capacity(cls, capacity: int, fp_target: float, seed: int) -> "BloomFilter":
        m_bits, k = filter_params(capacity, fp_target)
        return cls(m_bits, k, seed)

    def probes(self, key: bytes) -> list[int]:
        return hash_probes(key, self.seed, self.m_bits, self.k_hashes)

    def _mnk(self, key: bytes) -> tuple[int, int, int]:
        if len(key) != KEY_BYTES:
            raise ValueError(f"key must be {KEY_BYTES} bytes, got {len(key)}")
        return _KEY.unpack(key)

    def insert(self, key: bytes) -> None:
        m, n, k = self._mnk(key)
        if not self.bits.flags.c_contiguous or not self.bits.flags.writeable:
            self.bits = np.array(self.bits, dtype=np.uint8)
        _lib.check(
            _lib.lib.skpp_bloom_insert(self.bits.ctypes.data, self.m_bits, self.k_hashes, self.seed, m, n, k)
        )
        self.n_inserted += 1

    def contains(self, key: bytes) -> bool:
        m, n, k = self._mnk(key)
        bits = np.ascontiguousarray(self.bits)
        return bool(
            _lib.lib.skpp_bloom_contains(bits.ctypes.data, self.m_bits, self.k_hashes, self.seed, m, n, k)
        )

    __contains__ = contains

    def predicted_fp_rate(self, n: int | None = None) -> float:
        return predicted_fp_rate(self.m_bits, self.k_hashes, self.n_inserted if n is None else n)


def _policy_tag(policy: Policy) -> tuple[int, int, int]:
    """(tag, sk_batches, sk_first) header bytes (sieve.py:169-181)."""
    if policy.kind is PolicyKind.DATA_PARALLEL:
        return 0, 0, 0
    if policy.kind is PolicyKind.ALL_STREAM_K:
        return 6, 0, 0
    if policy.sk_batches > 0xFF:
        raise ValueError("sk_batches too large to serialize")
    return policy.sk_batches, policy.sk_batches, int(policy.sk_first)


def _policy_from_header(h: _lib.FilterHeader) -> Policy:
    # The C parser already rejected inconsistent tags (sieve.py:184-197).
    if h.sk_batches == 0:
        return Policy.data_parallel() if h.tag == 0 else Policy.all_stream_k()
    return Policy.hybrid(int(h.sk_batches), sk_first=bool(h.sk_first))


class _Snapshot:
    """Native copy of a bank's bits and seeds for the single-query fast path."""

    __slots__ = ("ptr", "cache")

    def __init__(self, bits2d: np.ndarray, seeds: np.ndarray, m_bits: int, k_hashes: int):
        self.ptr = _lib.lib.skpp_bank_snapshot(
            bits2d.ctypes.data, seeds.ctypes.data, bits2d.shape[0], m_bits, k_hashes
        )
        if not self.ptr:
            raise RuntimeError("skpp_bank_snapshot failed")
        self.cache: dict[int, list[Policy]] = {}

    def __del__(self):
        ptr, self.ptr = getattr(self, "ptr", None), None
        if ptr:
            _lib.lib.skpp_bank_snapshot_free(ptr)


class SieveBank:
    """Ordered (policy, filter) pairs sharing one (m_bits, k_hashes) geometry.

    Any number of concurrent readers may query a bank that is not being
    inserted into; insertion needs exclusive access (sieve.py:200-206).
    """

    def __init__(
        self,
        policies: list[Policy] | None = None,
        capacity: int = DEFAULT_CAPACITY,
        fp_target: float = DEFAULT_FP_TARGET,
        *,
        filters: list[tuple[Policy, BloomFilter]] | None = None,
    ):
        if filters is not None:
            if policies is not None:
                raise ValueError("pass either policies or prebuilt filters")
            self._check_filters(filters)
            self.filters = list(filters)
        else:
            if policies is None:
                policies = canonical_policies()
            if len(set(policies)) != len(policies):
                raise ValueError("policies must be distinct")
            if not policies:
                raise ValueError("bank needs at least one policy")
            m_bits, k = filter_params(capacity, fp_target)
            self.filters = [(p, BloomFilter(m_bits, k, filter_seed(i))) for i, p in enumerate(policies)]
        self.capacity = capacity
        self.fp_target = fp_target
        self._index = {p: f for p, f in self.filters}
        self._fast = None

    @staticmethod
    def _check_filters(filters: list[tuple[Policy, BloomFilter]]) -> None:
        if not filters:
            raise ValueError("bank needs at least one policy")
        pols = [p for p, _ in filters]
        if len(set(pols)) != len(pols):
            raise ValueError("policies must be distinct")
        if len({(f.m_bits, f.k_hashes) for _, f in filters}) != 1:
            raise ValueError("all filters in a bank must share (m_bits, k_hashes)")
        if len({f.seed for _, f in filters}) != len(filters):
            raise ValueError("filter seeds must be distinct")

    @classmethod
    def canonical(cls, capacity: int = DEFAULT_CAPACITY, fp_target: float = DEFAULT_FP_TARGET) -> "SieveBank":
        return cls(canonical_policies(), capacity, fp_target)

    @property
    def policies(self) -> list[Policy]:
        return [p for p, _ in self.filters]

    @property
    def m_bits(self) -> int:
        return self.filters[0][1].m_bits

    @property
    def k_hashes(self) -> int:
        return self.filters[0][1].k_hashes

    def filter_for(self, policy: Policy) -> BloomFilter:
        try:
            return self._index[policy]
        except KeyError:
            raise KeyError(f"policy {policy} not in bank") from None

    def insert(self, size: ProblemSize, policy: Policy) -> None:
        """Record ``policy`` as a candidate for ``size``."""
        self.filter_for(policy).insert(encode_key(size))
        self._fast = None

    def _stacked(self) -> tuple[np.ndarray, np.ndarray]:
        bits2d = np.ascontiguousarray(np.stack([f.bits for _, f in self.filters]))
        seeds = np.array([f.seed for _, f in self.filters], dtype=np.uint32)
        return bits2d, seeds

    def _fast_state(self):
        # Rebuilt lazily after inserts; racing readers build equal snapshots.
        fast = self._fast
        if fast is None:
            if len(self.filters) > 64:
                return None
            bits2d, seeds = self._stacked()
            fast = _Snapshot(bits2d, seeds, self.m_bits, self.k_hashes)
            self._fast = fast
        return fast

    def _policies_of(self, fast: _Snapshot, mask: int) -> list[Policy]:
        hit = fast.cache.get(mask)
        if hit is None:
            hit = [p for f, (p, _) in enumerate(self.filters) if mask >> f & 1]
            fast.cache[mask] = hit
        return hit

    def query(self, size: ProblemSize) -> list[Policy]:
        """Policies whose filter reports ``size``, in bank order (no false negatives)."""
        fast = self._fast_state()
        if fast is None:
            key = encode_key(size)
            return [p for p, f in self.filters if f.contains(key)]
        mask = _lib.lib.skpp_bank_snapshot_query(fast.ptr, size.m, size.n, size.k)
        return self._policies_of(fast, mask).copy()

    def query_masks(self, sizes: list[ProblemSize]) -> np.ndarray:
        """Hit masks of many sizes in one native call (bit f = filter f)."""
        if len(self.filters) > 64:
            raise ValueError("batched query supports at most 64 filters")
        bits2d, seeds = self._stacked()
        arr = np.array([(s.m, s.n, s.k) for s in sizes], dtype=np.uint64).reshape(-1, 3)
        masks = np.zeros(len(sizes), dtype=np.uint64)
        _lib.check(
            _lib.lib.skpp_bank_query_masks(
                bits2d.ctypes.data, seeds.ctypes.data, bits2d.shape[0], self.m_bits, self.k_hashes,
                arr.ctypes.data, len(sizes), masks.ctypes.data,
            )
        )
        return masks

    # -- serialization: "SKPS" | u16 version | u16 count | per filter
    #    <BBBBIQIQ> header + m_bits/8 bytes | u32 crc32 of all preceding bytes

    def to_bytes(self) -> bytes:
        hdrs = (_lib.FilterHeader * len(self.filters))()
        for i, (policy, f) in enumerate(self.filters):
            tag, sk_b, sk_f = _policy_tag(policy)
            hdrs[i] = _lib.FilterHeader(tag, sk_b, sk_f, 0, f.seed, f.m_bits, f.k_hashes, f.n_inserted)
        bits = np.concatenate([np.ascontiguousarray(f.bits, dtype=np.uint8) for _, f in self.filters])
        size = int(_lib.lib.skpp_bank_serialized_bytes(hdrs, len(self.filters)))
        out = np.empty(size, dtype=np.uint8)
        written = ctypes.c_uint64()
        _lib.check(
            _lib.lib.skpp_bank_serialize(
                hdrs, bits.ctypes.data, len(self.filters), out.ctypes.data, size, ctypes.byref(written)
            )
        )
        return out[: written.value].tobytes()

    @classmethod
    def from_bytes(cls, data: bytes) -> "SieveBank":
        data = bytes(data)
        count = ctypes.c_uint32(0)
        cap = 0
        if len(data) >= 8 and data[:4] == MAGIC:
            cap = data[6] | data[7] << 8
        hdrs = (_lib.FilterHeader * max(cap, 1))()
        offsets = (ctypes.c_uint64 * max(cap, 1))()
        rc = _lib.lib.skpp_bank_parse(data, len(data), hdrs, offsets, cap, ctypes.byref(count))
        if rc != _lib.OK:
            err = _FORMAT_ERRORS.get(rc)
            if err is None:
                raise _lib.SkppError(rc, _lib.last_error())
            raise err(_lib.last_error())
        raw = np.frombuffer(data, dtype=np.uint8)
        filters: list[tuple[Policy, BloomFilter]] = []
        for i in range(count.value):
            h = hdrs[i]
            nbytes = h.m_bits // 8
            bits = raw[offsets[i] : offsets[i] + nbytes].copy()
            bf = BloomFilter(int(h.m_bits), int(h.k_hashes), int(h.seed), bits=bits, n_inserted=int(h.n_inserted))
            filters.append((_policy_from_header(h), bf))
        cls._check_filters(filters)
        bank = cls.__new__(cls)
        bank.filters = filters
        bank.capacity = None
        bank.fp_target = None
        bank._index = {p: f for p, f in filters}
        bank._fast = None
        return bank

    def save(self, path: str | Path) -> None:
        Path(path).write_bytes(self.to_bytes())

    @classmethod
    def load(cls, path: str | Path) -> "SieveBank":
        return cls.from_bytes(Path(path).read_bytes())


@dataclass(frozen=True, slots=True)
class EliminationStats:
    """Share of non-baseline evaluations skipped, false negatives, absolute saving."""

    eliminated_fraction: float
    false_negatives: int
    evaluations_saved: int


def elimination_stats(bank: SieveBank, records, baseline: Policy | None = None) -> EliminationStats:
    """Sieve-guided tuning over records: evaluate query(size) plus the baseline (sieve.py:420-448)."""
    if not records:
        raise ValueError("records must be nonempty")
    if baseline is None:
        baseline = Policy.data_parallel()
    if baseline not in bank._index:
        raise KeyError(f"baseline {baseline} not in bank")
    n_pol = len(bank.filters)
    possible = len(records) * (n_pol - 1)
    base_bit = 1 << [p for p, _ in bank.filters].index(baseline)
    pos = {p: i for i, (p, _) in enumerate(bank.filters)}
    if n_pol <= 64:
        masks = [int(v) for v in bank.query_masks([r.size for r in records])]
    else:  # pragma: no cover - banks above 64 policies take the per-filter path
        masks = [sum(1 << pos[p] for p in bank.query(r.size)) for r in records]
    evaluated = 0
    false_neg = 0
    for rec, mask in zip(records, masks):
        cand = mask | base_bit
        evaluated += bin(cand).count("1") - 1
        w = pos.get(rec.winner)
        if w is None or not cand >> w & 1:
            false_neg += 1
    saved = possible - evaluated
    return EliminationStats(saved / possible if possible > 0 else 1.0, false_neg, saved)
