"""MurmurHash3 x64_128 through the native library.

Drop-in for ``gemmsched.hashing`` (reference ``hashing.py``): the portable
``murmur3_x64_128`` (hashing.py:41-91), the 24-byte key specialisation
``hash24`` (hashing.py:129-170, 191-194) and the all-filters membership mask
``query_mask`` (hashing.py:172-189, 196-206).  The reference compiles the
fast path with numba; here it is C++ in libskpp.so (``skpp_hash24``,
``skpp_bank_query_mask``), so ``HAVE_NUMBA`` — which the reference uses to
mean "the fast path is available" — is always True.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

MASK64 = (1 << 64) - 1
HAVE_NUMBA = True  # fast path present (native, not numba)
HAVE_NATIVE = True

_out2 = (ctypes.c_uint64 * 2)


def murmur3_x64_128(data: bytes, seed: int) -> tuple[int, int]:
    """128-bit MurmurHash3 (x64) of ``data``; the seed is taken modulo 2^32."""
    data = bytes(data)
    out = _out2()
    _lib.lib.skpp_murmur3_x64_128(data, len(data), seed & 0xFFFFFFFF, out)
    return int(out[0]), int(out[1])


def hash24(m: int, n: int, k: int, seed: int) -> tuple[int, int]:
    """murmur3_x64_128 of the little-endian (m, n, k) key with a 64-bit seed."""
    out = _out2()
    _lib.lib.skpp_hash24(m, n, k, seed, out)
    return int(out[0]), int(out[1])


def query_mask(
    bits: np.ndarray,
    seeds: np.ndarray,
    m_bits: int,
    k_hashes: int,
    m: int,
    n: int,
    k: int,
) -> int:
    """Bit f of the result is set iff filter f (row f of ``bits``) reports (m, n, k)."""
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    seeds64 = np.asarray(seeds, dtype=np.uint64)
    if seeds64.size and int(seeds64.max()) > 0xFFFFFFFF:
        raise ValueError("filter seeds must fit in 32 bits")
    seeds32 = np.ascontiguousarray(seeds64.astype(np.uint32))
    if bits.ndim != 2 or bits.shape[0] != seeds32.shape[0] or bits.shape[0] > 64:
        raise ValueError("bits must be (n_filters <= 64, m_bits/8) with one seed per filter")
    if bits.shape[1] * 8 != m_bits:
        raise ValueError("bit rows must hold m_bits/8 bytes")
    return int(
        _lib.lib.skpp_bank_query_mask(
            bits.ctypes.data, seeds32.ctypes.data, bits.shape[0], m_bits, k_hashes, m, n, k
        )
    )
