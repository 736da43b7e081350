"""Build libskpp.so in-tree with nvcc for sm_100a (B200).

The library holds both halves of the C ABI declared in ``include/skpp.h``:
the CUDA kernels (``csrc/skpp_gemm.cu``) and the host selection layer
(``csrc/skpp_host.cpp``).  It is written next to this file so that it travels
with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libskpp.so"
SOURCES = [CSRC / "skpp_gemm.cu", CSRC / "skpp_host.cpp"]
HEADERS = [CSRC / "skpp_sched.h", REPO_DIR / "include" / "skpp.h"]

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-shared",
    "-Xcompiler",
    "-fPIC",
    "-O3",
    "-std=c++17",
    "-lineinfo",
    *ARCH_FLAGS,
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: cannot build libskpp.so")
    return cand


HASH_PATH = LIB_PATH.with_name(LIB_PATH.name + ".srchash")


def source_hash() -> str:
    """Content hash of every source and header plus the compile flags."""
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for p in SOURCES + HEADERS:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def is_stale() -> bool:
    """True when the library is missing or was built from different sources.

    Content hashes (not mtimes) so that a copied checkout, e.g. the snapshot
    shipped to a GPU box, does not trigger a rebuild.
    """
    if not LIB_PATH.exists() or not HASH_PATH.exists():
        return True
    return HASH_PATH.read_text().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile libskpp.so if it is missing or older than its sources."""
    if not force and not is_stale():
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(f".so.tmp{os.getpid()}")
    cmd = [_nvcc(), *NVCC_FLAGS, *map(str, SOURCES), "-o", str(tmp)]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        tmp.unlink(missing_ok=True)
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB_PATH)
    HASH_PATH.write_text(source_hash() + "\n")
    return LIB_PATH


if __name__ == "__main__":  # pragma: no cover
    print(build(force=True, verbose=True))
