"""Liveness of Stream-K grids that share the GPU (run on a B200 via gpurun).

Phase-2 reducers spin on peer flags, so a Stream-K grid must never be partially resident.
Stream-K grids launch cooperatively (skpp_set_cooperative, default on): gang-scheduled,
all CTAs or none.  These tests drive concurrent Stream-K grids on streams of different
priorities in one process, and two such processes on one GPU at once; each must finish
(bounded by a timeout far below the kernel's 17 s flag watchdog x rounds) with bitwise
results.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "_liveness_worker.py")


def _run_workers(n_proc, rounds, streams):
    procs = [subprocess.Popen([sys.executable, WORKER, str(rounds), str(streams), str(11 + i), ROOT],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, cwd=ROOT)
             for i in range(n_proc)]
    outs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=300)
            outs.append((p.returncode, out))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    return outs


def test_concurrent_streamk_grids_on_prioritised_streams():
    (rc, out), = _run_workers(1, 200, 4)
    assert rc == 0 and out.strip().endswith("ok"), out[-2000:]


def test_two_processes_share_one_gpu():
    outs = _run_workers(2, 200, 3)
    for rc, out in outs:
        assert rc == 0 and out.strip().endswith("ok"), out[-2000:]
