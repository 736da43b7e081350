"""ctypes binding of libskpp.so (the C ABI in include/skpp.h).

There is no Python fallback behind these symbols: if the library cannot be
loaded, importing the package raises, so nothing silently runs on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import _build

LIB_PATH: Path = _build.LIB_PATH

# status codes (include/skpp.h)
OK = 0
EINVAL, ETILE, EALIGN, EARCH, ELAUNCH, EWORKSPACE, EGRID, ECAPACITY = 1, 2, 3, 4, 5, 6, 7, 8
ETRUNCATED, EBADMAGIC, EVERSION, EFORMAT, ECHECKSUM = 20, 21, 22, 23, 24

F32, F16, BF16 = 0, 1, 2
DATA_PARALLEL, HYBRID, ALL_STREAM_K = 0, 1, 2
TRACE_FIELDS = 8  # tile, kb, ke, write_mode, phase, role, tile_m, tile_n


class Problem(C.Structure):
    _fields_ = [("m", C.c_uint64), ("n", C.c_uint64), ("k", C.c_uint64)]


class Tile(C.Structure):
    _fields_ = [("blk_m", C.c_uint32), ("blk_n", C.c_uint32), ("blk_k", C.c_uint32), ("tile_order", C.c_uint32)]


def tile_c(tile) -> Tile:
    """skpp_tile_t of a TileShape (tile order 0, the reference's) or a KernelTile."""
    return Tile(tile.blk_m, tile.blk_n, tile.blk_k, getattr(tile, "band_rows", 0))


class PolicyC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("sk_batches", C.c_int32), ("sk_first", C.c_int32)]


class SchedC(C.Structure):
    _fields_ = [
        ("m_tiles", C.c_uint64),
        ("n_tiles", C.c_uint64),
        ("iters_per_tile", C.c_uint64),
        ("total_tiles", C.c_uint64),
        ("total_iters", C.c_uint64),
        ("dp_tiles", C.c_uint64),
        ("sk_tiles", C.c_uint64),
        ("sk_iters", C.c_uint64),
        ("ipw", C.c_uint64),
        ("g", C.c_uint32),
        ("sk_first", C.c_uint32),
    ]


class Operands(C.Structure):
    _fields_ = [
        ("a", C.c_void_p),
        ("lda", C.c_int64),
        ("b", C.c_void_p),
        ("ldb", C.c_int64),
        ("c", C.c_void_p),
        ("ldc", C.c_int64),
        ("in_dtype", C.c_int32),
        ("out_dtype", C.c_int32),
    ]


class FilterHeader(C.Structure):
    _fields_ = [
        ("tag", C.c_uint8),
        ("sk_batches", C.c_uint8),
        ("sk_first", C.c_uint8),
        ("reserved", C.c_uint8),
        ("seed", C.c_uint32),
        ("m_bits", C.c_uint64),
        ("k_hashes", C.c_uint32),
        ("n_inserted", C.c_uint64),
    ]


_P = C.POINTER
_u8p = _P(C.c_uint8)
_u32p = _P(C.c_uint32)
_u64p = _P(C.c_uint64)
_i64p = _P(C.c_int64)

# name -> (restype, argtypes); every symbol declared in include/skpp.h
SIGNATURES = {
    "skpp_last_error": (C.c_char_p, []),
    "skpp_version": (C.c_char_p, []),
    "skpp_sched_make": (C.c_int, [_P(Problem), _P(Tile), C.c_uint32, _P(PolicyC), _P(SchedC)]),
    "skpp_schedule_trace": (C.c_int, [_P(Problem), _P(Tile), C.c_uint32, _P(PolicyC), C.c_uint32,
                                      C.c_void_p, C.c_void_p]),
    "skpp_sched_count": (C.c_int, [_P(SchedC), _u64p, _u64p]),
    "skpp_sched_items": (C.c_int, [_P(SchedC), _i64p, C.c_uint64, _u64p]),
    "skpp_validate_intervals": (
        C.c_int,
        [_u64p, _u64p, C.c_uint64, C.c_uint64, _u64p, _u64p],
    ),
    "skpp_tile_coords": (C.c_int, [_P(SchedC), C.c_uint32, C.c_uint64, _P(C.c_uint64), _P(C.c_uint64)]),
    "skpp_workspace_bytes": (C.c_uint64, [_P(Problem), _P(Tile), C.c_uint32]),
    "skpp_tile_supported": (C.c_int, [_P(Tile)]),
    "skpp_gemm_launch": (
        C.c_int,
        [
            _P(Problem),
            _P(Tile),
            _P(PolicyC),
            C.c_uint32,
            _P(Operands),
            C.c_void_p,
            C.c_uint64,
            C.c_void_p,
            C.c_uint64,
            C.c_void_p,
            C.c_void_p,
        ],
    ),
    "skpp_plan_create": (
        C.c_int,
        [_P(Problem), _P(Tile), _P(PolicyC), C.c_uint32, _P(Operands), C.c_void_p, C.c_uint64,
         C.c_void_p, _P(C.c_void_p)],
    ),
    "skpp_plan_workspace_bytes": (C.c_uint64, [C.c_void_p]),
    "skpp_plan_launch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "skpp_plan_destroy": (None, [C.c_void_p]),
    "skpp_schedule_trace_device": (
        C.c_int,
        [_P(Problem), _P(Tile), _P(PolicyC), C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p],
    ),
    "skpp_set_device": (C.c_int, [C.c_int]),
    "skpp_stream_is_capturing": (C.c_int, [C.c_void_p]),
    "skpp_debug_timeline": (None, [C.c_void_p]),
    "skpp_set_pdl": (None, [C.c_int]),
    "skpp_set_cooperative": (None, [C.c_int]),
    "skpp_test_hold_sms": (C.c_int, [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    "skpp_set_b3d": (None, [C.c_int]),
    "skpp_set_a3d": (None, [C.c_int]),
    "skpp_set_l2_prefetch": (None, [C.c_int]),
    "skpp_set_l2_hints": (None, [C.c_int]),
    "skpp_set_debug": (None, [C.c_int]),
    "skpp_device_info": (C.c_int, [C.c_int, _P(C.c_int32), _P(C.c_int32), _P(C.c_int32)]),
    "skpp_max_coresident": (C.c_int, [_P(Tile), _P(C.c_int32)]),
    "skpp_murmur3_x64_128": (None, [C.c_char_p, C.c_uint64, C.c_uint32, _u64p]),
    "skpp_hash24": (None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u64p]),
    "skpp_filter_params": (C.c_int, [C.c_uint64, C.c_double, _u64p, _u32p]),
    "skpp_filter_seed": (C.c_uint32, [C.c_uint64]),
    "skpp_hash_probes": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint64, C.c_uint32, _u64p]),
    "skpp_bloom_insert": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64],
    ),
    "skpp_bloom_contains": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64],
    ),
    "skpp_bank_query_mask": (
        C.c_uint64,
        [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64],
    ),
    "skpp_bank_query_masks": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p],
    ),
    "skpp_bank_snapshot": (C.c_void_p, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32]),
    "skpp_bank_snapshot_query": (C.c_uint64, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64]),
    "skpp_bank_snapshot_free": (None, [C.c_void_p]),
    "skpp_crc32": (C.c_uint32, [C.c_char_p, C.c_uint64, C.c_uint32]),
    "skpp_bank_serialized_bytes": (C.c_uint64, [_P(FilterHeader), C.c_uint32]),
    "skpp_bank_serialize": (
        C.c_int,
        [_P(FilterHeader), C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, _u64p],
    ),
    "skpp_bank_parse": (
        C.c_int,
        [C.c_char_p, C.c_uint64, _P(FilterHeader), _u64p, C.c_uint32, _u32p],
    ),
}


def _load() -> C.CDLL:
    # Development hook for same-box A/B runs of two kernel builds (tools/ab_libs.py):
    # SKPP_LIB names another build of libskpp.so; entry points it lacks stay unbound.
    override = os.environ.get("SKPP_LIB")
    if not override and _build.is_stale():
        # In-tree sources are newer than the library (or it is missing): rebuild.
        # On a box without nvcc this raises, which is the intended loud failure.
        _build.build()
    path = override or str(LIB_PATH)
    try:
        lib = C.CDLL(path)
    except OSError as exc:  # pragma: no cover - exercised only on broken installs
        raise ImportError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        if override and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class SkppError(RuntimeError):
    """A libskpp call failed; ``code`` is the SKPP_E* status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def last_error() -> str:
    raw = lib.skpp_last_error()
    return raw.decode("utf-8", "replace") if raw else ""


def check(rc: int) -> None:
    if rc != OK:
        raise SkppError(rc, last_error())
