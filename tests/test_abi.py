"""The C-ABI library loads on a CPU-only machine and exports every symbol include/skpp.h declares."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "skpp.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(skpp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("skpp_gemm_launch", "skpp_workspace_bytes", "skpp_schedule_trace_device",
                 "skpp_murmur3_x64_128", "skpp_bank_query_mask", "skpp_bank_parse", "skpp_sched_items",
                 "skpp_validate_intervals", "skpp_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2408_11417_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers the same set
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_host_entry_points_work_without_gpu():
    from paper_2408_11417_b200 import _lib

    out = (ctypes.c_uint64 * 2)()
    _lib.lib.skpp_murmur3_x64_128(b"foo", 3, 0, out)
    assert (out[0], out[1]) == (16316970633193145697, 9128664383759220103)
    assert _lib.lib.skpp_tile_supported(_lib.Tile(128, 128, 64)) == 1
    assert _lib.lib.skpp_tile_supported(_lib.Tile(64, 64, 32)) == 0
    assert _lib.lib.skpp_workspace_bytes(_lib.Problem(512, 512, 16384), _lib.Tile(128, 128, 64), 148) > 0
    assert b"sm_100a" in _lib.lib.skpp_version()


def test_gemm_launch_validates_before_touching_the_device():
    from paper_2408_11417_b200 import _lib

    ops = _lib.Operands(None, 64, None, 64, None, 64, _lib.BF16, _lib.F32)
    rc = _lib.lib.skpp_gemm_launch(_lib.Problem(64, 64, 64), _lib.Tile(64, 64, 64), _lib.PolicyC(0, 0, 0), 148,
                                   ops, None, 0, None, 0, None, None)
    assert rc == _lib.ETILE
    assert "not implemented" in _lib.last_error()
    rc = _lib.lib.skpp_gemm_launch(_lib.Problem(64, 64, 64), _lib.Tile(128, 128, 64), _lib.PolicyC(0, 0, 0), 148,
                                   ops, None, 0, None, 0, None, None)
    assert rc == _lib.EINVAL  # null operands


def test_product_refuses_to_run_without_cuda():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import numpy as np

    import paper_2408_11417_b200 as sk

    size, tile = sk.ProblemSize(128, 128, 64), sk.TileShape(128, 128, 64)
    sched = sk.build_schedule(size, tile, sk.HardwareModel(148, 1), sk.Policy.data_parallel())
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sk.execute_schedule(np.zeros((128, 64)), np.zeros((64, 128)), sched, tile, size)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2408_11417_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in text and "import oracle" not in text, f
