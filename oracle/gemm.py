"""Oracle restatement of the reference executor (gemmsched executor.py).

float64 numpy: every work item adds ``a[r0:r1, k0:k1] @ b[k0:k1, c0:c1]``
into C (executor.py:93-112).  Used as the parity checker for integer inputs
and as the timed CPU baseline (``bench.py --impl reference``).
"""

from __future__ import annotations

import numpy as np


def reference_gemm(a, b):
    """executor.py:31-41."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2:
        raise ValueError("reference_gemm expects 2-D matrices")
    if a.shape[1] != b.shape[0]:
        raise ValueError("inner dimensions disagree")
    return a @ b


def random_int_matrix(rows, cols, rng, lo=-8, hi=8):
    """executor.py:44-48: integers in [lo, hi] as float64 (A drawn before B by callers)."""
    return rng.integers(lo, hi + 1, size=(rows, cols)).astype(np.float64)


def execute_schedule(a, b, schedule, m, n, k, bm, bn, bk, n_tiles):
    """executor.py:51-112 (sequential order): run each item's MAC block and accumulate."""
    c = np.zeros((m, n), dtype=np.float64)
    for wg in schedule:
        for t, kb, ke, _wm, _ph in wg:
            tm, tn = divmod(t, n_tiles)
            r0, c0 = tm * bm, tn * bn
            r1, c1 = min(r0 + bm, m), min(c0 + bn, n)
            k0, k1 = kb * bk, min(ke * bk, k)
            c[r0:r1, c0:c1] += a[r0:r1, k0:k1] @ b[k0:k1, c0:c1]
    return c
