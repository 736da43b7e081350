"""GEMM entry point: run a Stream-K++ schedule on the B200.

Drop-in for ``gemmsched.executor`` (reference ``executor.py``).  The
reference executes each ``WorkItem`` on the host as
``c[r0:r1,c0:c1] += a[r0:r1,k0:k1] @ b[k0:k1,c0:c1]`` in float64
(executor.py:51-124).  Here :func:`execute_schedule` hands the whole schedule
to one persistent sm_100a kernel through ``skpp_gemm_launch``: fp16/bf16
operands, fp32 tensor-core accumulation, and a deterministic fixed-order
partial-tile fixup instead of atomic adds.  There is no CPU fallback — on a
machine without a B200 these functions raise.

* ``execute_schedule(a, b, sched, tile, size, *, order, rng, workers)`` keeps
  the reference signature and error messages.  numpy inputs are copied to
  the GPU as ``in_dtype`` (default bf16) and the result comes back as float64
  numpy; CUDA tensors stay on the device and return a CUDA tensor of
  ``out_dtype`` (default fp32).  ``order``/``rng``/``workers`` are validated
  as in the reference and otherwise have no effect: the device result does
  not depend on completion order (the fixup order is fixed).
* ``reference_gemm`` / ``random_int_matrix`` / ``run_equivalence`` mirror
  executor.py:31-48, 127-145; ``reference_gemm`` is the reference's plain
  float64 ``A @ B`` oracle used only for the equivalence report.
* :func:`gemm` is the tensor-level API (policy instead of a materialised
  schedule) used by the sweep and the benchmark.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .scheduler import Schedule, build_schedule, closed_form, grid_info
from .types import HardwareModel, Policy, ProblemSize, TileShape, tile_grid

try:
    import torch
except ImportError as exc:  # pragma: no cover - torch is part of the image
    raise ImportError("paper_2408_11417_b200.executor needs torch for device memory") from exc

DEFAULT_GEMM_TILE = TileShape(128, 128, 64)

_IN_DTYPES = {torch.float16: _lib.F16, torch.bfloat16: _lib.BF16}
_OUT_DTYPES = {torch.float32: _lib.F32, torch.float16: _lib.F16, torch.bfloat16: _lib.BF16}
_NAMED = {
    "fp16": torch.float16,
    "float16": torch.float16,
    "bf16": torch.bfloat16,
    "bfloat16": torch.bfloat16,
    "fp32": torch.float32,
    "float32": torch.float32,
}


def _as_dtype(d, default):
    if d is None:
        return default
    if isinstance(d, str):
        return _NAMED[d.lower()]
    return d


@dataclass(frozen=True, slots=True)
class EquivalenceReport:
    exact_match: bool
    max_abs_diff: float


def reference_gemm(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """float64 ``A @ B`` oracle (executor.py:31-41)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2:
        raise ValueError("reference_gemm expects 2-D matrices")
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"inner dimensions disagree: A is {a.shape}, B is {b.shape}")
    return a @ b


def random_int_matrix(
    rows: int, cols: int, rng: np.random.Generator, lo: int = -8, hi: int = 8
) -> np.ndarray:
    """Integer-valued float64 matrix, exact under any summation order (executor.py:44-48)."""
    return rng.integers(lo, hi + 1, size=(rows, cols)).astype(np.float64)


# -- device plumbing ----------------------------------------------------------

_tls = threading.local()
_ws_lock = threading.Lock()
_workspaces: dict[tuple[int, int], torch.Tensor] = {}
_sm_counts: dict[int, int] = {}


def _require_cuda() -> int:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "the Stream-K++ GEMM runs only on a CUDA device (sm_100a B200); "
            "there is no CPU fallback"
        )
    dev = torch.cuda.current_device()
    if getattr(_tls, "device", None) != dev:
        _lib.check(_lib.lib.skpp_set_device(dev))
        _tls.device = dev
    return dev


def sm_count(device: int | None = None) -> int:
    """Streaming multiprocessors of the device (148 on a B200)."""
    dev = _require_cuda() if device is None else device
    if dev not in _sm_counts:
        n = ctypes.c_int32()
        _lib.check(_lib.lib.skpp_device_info(dev, ctypes.byref(n), None, None))
        _sm_counts[dev] = int(n.value)
    return _sm_counts[dev]


def max_coresident(tile: TileShape) -> int:
    _require_cuda()
    n = ctypes.c_int32()
    _lib.check(
        _lib.lib.skpp_max_coresident(_lib.tile_c(tile), ctypes.byref(n))
    )
    return int(n.value)


def default_g(tile: TileShape, device: int | None = None) -> int:
    """Persistent workgroups of one launch: the tile's declared grid (``KernelTile.grid``),
    else one CTA per SM, or one CTA pair per two SMs for 256-row (cta_group::2) tiles."""
    return tile_grid(tile) or sm_count(device) // (2 if tile.blk_m == 256 else 1)


def tile_supported(tile: TileShape) -> bool:
    return bool(_lib.lib.skpp_tile_supported(_lib.tile_c(tile)))




def _new_workspace(nbytes: int, device: int, stream_handle: int) -> torch.Tensor:
    """Allocate a fixup workspace on the launch stream and zero it there.

    The kernel needs the control block (epoch header, slot flags, band states) zeroed
    (skpp.h: "zero-filled the first time it is used"); the whole buffer is zeroed, once per
    allocation, so no partial slot ever holds recycled memory.  Allocating and zeroing on the
    stream the kernel runs on (not torch's current stream) orders the memset before the
    first launch and ties the block's lifetime to that stream.

    Outside a graph capture the device is then synchronised once, so the fill has landed
    before the first launch can start.  Stream order alone was not enough: in about 1 of 125
    fresh processes the first Stream-K launch (programmatic dependent launch, right behind the
    fill) ran concurrently with the fill, which zeroed the epoch header and the early slots
    under it (`profiles/round2/session5/`).  The cost is one host sync per new workspace.
    """
    size = max(nbytes, 1 << 20)
    with torch.cuda.stream(torch.cuda.ExternalStream(stream_handle, device=f"cuda:{device}")):
        buf = torch.zeros(size, dtype=torch.uint8, device=f"cuda:{device}")
    if not _is_capturing(stream_handle):
        torch.cuda.synchronize(device)
    return buf


def workspace_for(nbytes: int, device: int, stream_handle: int) -> torch.Tensor:
    """Fixup workspace for eager launches, cached per (device, stream).

    The kernel keeps the workspace consistent itself (flags are tagged with
    an epoch stored in the workspace header and advanced by the last CTA of
    each launch), so a cached buffer serves every later launch on the same
    stream: launches on one stream are ordered, so they never use it at once.
    Plans hold a reference to the buffer they were bound to, so growing the
    cache never frees memory in use.  Graph-captured launches do not use this
    cache: each plan gets its own workspace (:meth:`GemmPlan.prepare_for_capture`).
    """
    key = (device, stream_handle)
    with _ws_lock:
        buf = _workspaces.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = _new_workspace(nbytes, device, stream_handle)
            _workspaces[key] = buf
        return buf


def _is_capturing(handle: int) -> bool:
    rc = _lib.lib.skpp_stream_is_capturing(handle)
    if rc < 0:
        raise _lib.SkppError(rc, _lib.last_error())
    return rc == 1


class GemmPlan:
    """A prepared launch: C = A @ B under one policy, reusable and graph-capturable.

    The schedule scalars, kernel choice and TMA descriptors are built once in
    C++ (``skpp_plan_create``); :meth:`launch` binds the per-stream workspace
    and makes a single ``skpp_plan_launch`` call on the current stream.
    """

    def __init__(
        self,
        a: torch.Tensor,
        b: torch.Tensor,
        c: torch.Tensor,
        policy: Policy,
        tile: TileShape = DEFAULT_GEMM_TILE,
        g: int | None = None,
        trace_cap: int = 0,
    ):
        dev = _require_cuda()
        if a.dim() != 2 or b.dim() != 2 or c.dim() != 2:
            raise ValueError("gemm expects 2-D matrices")
        if a.shape[1] != b.shape[0]:
            raise ValueError(f"inner dimensions disagree: A is {tuple(a.shape)}, B is {tuple(b.shape)}")
        if tuple(c.shape) != (a.shape[0], b.shape[1]):
            raise ValueError("output shape does not match (m, n)")
        if a.dtype not in _IN_DTYPES or b.dtype != a.dtype:
            raise ValueError("A and B must both be float16 or both bfloat16")
        if c.dtype not in _OUT_DTYPES:
            raise ValueError("output must be float32, float16 or bfloat16")
        for name, t in (("A", a), ("B", b), ("C", c)):
            if not t.is_cuda:
                raise ValueError(f"{name} must be a CUDA tensor")
            if t.stride(1) != 1:
                raise ValueError(f"{name} must be row-major (unit column stride)")
        if not tile_supported(tile):
            raise ValueError(
                f"tile {tile.blk_m}x{tile.blk_n}x{tile.blk_k} is not implemented by the sm_100a "
                "kernel (blk_m=128: blk_n in {64,128,256}, blk_k in {16,32,64,128}; "
                "blk_m=256 CTA pair: blk_n in {128,256}, blk_k in {32,64,128})"
            )
        m, k = a.shape
        n = b.shape[1]
        self.size = ProblemSize(int(m), int(n), int(k))
        self.tile = tile
        self.policy = policy
        self.g = default_g(tile, dev) if g is None else int(g)
        self.a, self.b, self.c = a, b, c  # keep the operands alive as long as the plan
        self.device = dev
        self.sched_c = closed_form(self.size, tile, self.g, policy)
        from .scheduler import policy_to_c

        self.trace_cap = int(trace_cap)
        if self.trace_cap:
            self.trace = torch.full(
                (self.g, self.trace_cap, _lib.TRACE_FIELDS), -1, dtype=torch.int64, device=a.device
            )
            self.trace_counts = torch.zeros(self.g, dtype=torch.int64, device=a.device)
        else:
            self.trace = self.trace_counts = None
        ops = _lib.Operands(
            a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0),
            _IN_DTYPES[a.dtype], _OUT_DTYPES[c.dtype],
        )
        handle = ctypes.c_void_p()
        rc = _lib.lib.skpp_plan_create(
            _lib.Problem(m, n, k), _lib.tile_c(tile), policy_to_c(policy),
            self.g, ops,
            self.trace.data_ptr() if self.trace is not None else None, self.trace_cap,
            self.trace_counts.data_ptr() if self.trace_counts is not None else None,
            ctypes.byref(handle),
        )
        if rc != _lib.OK:
            msg = _lib.last_error()
            if rc in (_lib.ETILE, _lib.EALIGN, _lib.EINVAL, _lib.EGRID):
                raise ValueError(msg)
            raise _lib.SkppError(rc, msg)
        self._handle = handle.value
        self.ws_bytes = int(_lib.lib.skpp_plan_workspace_bytes(self._handle))
        self._launch = _lib.lib.skpp_plan_launch
        self._ws_cache: dict[int, tuple] = {}
        self._private_ws: torch.Tensor | None = None

    def __del__(self):
        h, self._handle = getattr(self, "_handle", None), None
        if h:
            _lib.lib.skpp_plan_destroy(h)

    @property
    def uses_fixup(self) -> bool:
        return self.sched_c.sk_tiles > 0

    def prepare_for_capture(self, stream: torch.cuda.Stream | None = None) -> None:
        """Give this plan its own workspace before its launches are captured into a CUDA graph.

        Captured launches never share the per-stream eager workspace: graphs captured on
        one stream could otherwise be replayed concurrently on different streams and race
        on one flags/partials area.  Without this call, the first captured launch allocates
        the private workspace inside the capture (its header memset then becomes a graph
        node, re-run before the GEMM on every replay); calling this first is the recommended
        path, since it also settles the zero-fill before any launch (see ``_new_workspace``).  One workspace must never serve two executions at once: a graph (like any
        launch of this plan) must not be replayed concurrently with itself.
        """
        if self.ws_bytes and self._private_ws is None:
            handle = stream.cuda_stream if stream is not None else torch._C._cuda_getCurrentRawStream(self.device)
            self._private_ws = _new_workspace(self.ws_bytes, self.device, handle)

    def share_workspace_of(self, other: "GemmPlan") -> None:
        """Capture this plan's launches on ``other``'s private workspace.  Only for launches
        that run strictly one after another (e.g. a rotation of plans inside one graph)."""
        if not self.ws_bytes:
            return
        other.prepare_for_capture()
        if other._private_ws is None or other._private_ws.numel() < self.ws_bytes:
            raise ValueError("the other plan's workspace is too small for this plan")
        self._private_ws = other._private_ws

    def launch(self, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        handle = stream.cuda_stream if stream is not None else torch._C._cuda_getCurrentRawStream(self.device)
        if self.ws_bytes and _is_capturing(handle):
            if self._private_ws is None:
                self._private_ws = _new_workspace(self.ws_bytes, self.device, handle)
            buf = self._private_ws
            ws = (buf.data_ptr(), buf.numel(), buf)
        else:
            ws = self._ws_cache.get(handle)
            if ws is None:
                if self.ws_bytes:
                    buf = workspace_for(self.ws_bytes, self.device, handle)
                    ws = (buf.data_ptr(), buf.numel(), buf)
                else:
                    ws = (None, 0, None)
                self._ws_cache[handle] = ws
        rc = self._launch(self._handle, ws[0], ws[1], handle)
        if rc != _lib.OK:
            raise _lib.SkppError(rc, _lib.last_error())
        return self.c

    def trace_items(self) -> list[list[tuple[int, int, int, int, int, int]]]:
        """Per-CTA items recorded by the last traced launch (device -> host)."""
        if self.trace is None:
            raise ValueError("plan was built without trace_cap")
        counts = self.trace_counts.cpu().tolist()
        rows = self.trace.cpu().numpy()
        out = []
        for x in range(self.g):
            cnt = int(counts[x])
            if cnt > self.trace_cap:
                raise ValueError(f"CTA {x} recorded {cnt} items > trace_cap {self.trace_cap}")
            out.append([tuple(int(v) for v in r) for r in rows[x, :cnt]])
        return out


def gemm(
    a: torch.Tensor,
    b: torch.Tensor,
    policy: Policy,
    *,
    tile: TileShape = DEFAULT_GEMM_TILE,
    g: int | None = None,
    out: torch.Tensor | None = None,
    out_dtype: torch.dtype = torch.float32,
) -> torch.Tensor:
    """C = A @ B on the current CUDA stream under a Stream-K++ policy."""
    if out is None:
        out = torch.empty((a.shape[0], b.shape[1]), dtype=out_dtype, device=a.device)
    return GemmPlan(a, b, out, policy, tile, g).launch()


def _pad_cols(t: torch.Tensor, mult: int = 8) -> torch.Tensor:
    """Zero-pad the column count to a multiple of `mult` (TMA needs 16-byte row strides)."""
    cols = t.shape[1]
    if cols % mult == 0 and t.stride(1) == 1 and t.stride(0) % mult == 0:
        return t
    padded = torch.zeros((t.shape[0], (cols + mult - 1) // mult * mult), dtype=t.dtype, device=t.device)
    padded[:, :cols] = t
    return padded


def _check_closed_form(sched: Schedule, size: ProblemSize, tile: TileShape) -> None:
    mark = getattr(sched, "_skpp_closed_form", None)
    if mark is not None and mark[0] == size and mark[1] == tile and mark[2] is sched.assignments:
        return
    expected = build_schedule(size, tile, HardwareModel(sched.g, 1), sched.policy)
    if expected.assignments != sched.assignments:
        raise ValueError(
            "schedule differs from the closed form of its policy; the device kernel "
            "executes policy schedules (build_schedule output) only"
        )


# Plans of execute_schedule calls, keyed by everything the native plan bakes in (device,
# operand addresses, row strides, dtypes, problem, tile, policy, g).  Repeated calls of one
# shape get the same device addresses back from torch's caching allocator, so they skip the
# plan build (three cuTensorMapEncodeTiled calls and the schedule closed form, ~14 us,
# profiles/round2/e2e_overhead.jsonl).  A cached plan holds no tensor references (the caller's
# tensors own the memory); it is launched only when live tensors match its key exactly.
_PLAN_CACHE: "dict[tuple, GemmPlan]" = {}
_PLAN_CACHE_MAX = 64
_plan_cache_stats = {"hits": 0, "misses": 0}


def _cached_plan(a, b, c, policy, tile, g):
    key = (a.device.index, a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0),
           tuple(a.shape), tuple(b.shape), a.dtype, c.dtype, tile, policy, g)
    with _ws_lock:
        plan = _PLAN_CACHE.get(key)
        if plan is not None:
            _plan_cache_stats["hits"] += 1
            _PLAN_CACHE[key] = _PLAN_CACHE.pop(key)  # most recently used last
            return plan
    plan = GemmPlan(a, b, c, policy, tile, g)
    plan.a = plan.b = plan.c = None  # the key's tensors own the memory, not the plan
    with _ws_lock:
        _plan_cache_stats["misses"] += 1
        _PLAN_CACHE[key] = plan
        while len(_PLAN_CACHE) > _PLAN_CACHE_MAX:
            _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
    return plan


def execute_schedule(
    a,
    b,
    sched: Schedule,
    tile: TileShape,
    size: ProblemSize,
    *,
    order: str = "scheduled",
    rng: np.random.Generator | None = None,
    workers: int = 1,
    in_dtype=None,
    out_dtype=None,
):
    """Run every work item of ``sched`` on the GPU and return C = A @ B."""
    is_torch = isinstance(a, torch.Tensor)
    if is_torch:
        a_shape, b_shape = tuple(a.shape), tuple(b.shape)
    else:
        a = np.asarray(a, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        a_shape, b_shape = a.shape, b.shape
    if a_shape != (size.m, size.k) or b_shape != (size.k, size.n):
        raise ValueError(
            f"matrix shapes {a_shape} x {b_shape} do not match "
            f"problem size ({size.m}, {size.n}, {size.k})"
        )
    if sched.grid != grid_info(size, tile):
        raise ValueError("schedule was built for a different problem/tile")
    if order == "shuffled":
        if rng is None:
            raise ValueError('order="shuffled" requires an rng')
    elif order != "scheduled":
        raise ValueError(f"unknown order {order!r}")
    _check_closed_form(sched, size, tile)

    dev = _require_cuda()
    host_result = False
    if is_torch:
        if not a.is_cuda:
            # Host tensors (ideally pinned): copy in, and hand the result back on the host.
            host_result = True
            a = a.to(f"cuda:{dev}", non_blocking=True)
            b = b.to(f"cuda:{dev}", non_blocking=True)
        op_dtype = a.dtype if a.dtype in _IN_DTYPES else _as_dtype(in_dtype, torch.bfloat16)
        res_dtype = _as_dtype(out_dtype, torch.float32)
        ad = a.to(op_dtype)
        bd = b.to(op_dtype)
    else:
        op_dtype = _as_dtype(in_dtype, torch.bfloat16)
        res_dtype = _as_dtype(out_dtype, torch.float32)
        ad = torch.from_numpy(a).to(op_dtype).pin_memory().to(f"cuda:{dev}", non_blocking=True)
        bd = torch.from_numpy(b).to(op_dtype).pin_memory().to(f"cuda:{dev}", non_blocking=True)
    ad = _pad_cols(ad)
    bd = _pad_cols(bd)
    if ad.shape[1] != size.k:
        # K was padded for A's row stride: pad B's rows to the same K with zeros.
        bk = torch.zeros((ad.shape[1], bd.shape[1]), dtype=bd.dtype, device=bd.device)
        bk[: size.k] = bd
        bd = bk
    c = torch.empty((size.m, bd.shape[1]), dtype=res_dtype, device=ad.device)
    # Padding K or N up to a multiple of 8 never changes ceil(K/blk_k) or
    # ceil(N/blk_n) (the implemented blk_n/blk_k are multiples of 8), so the
    # launched schedule is the caller's; padded K only adds zero products.
    _cached_plan(ad, bd, c, sched.policy, tile, sched.g).launch()
    out = c[:, : size.n]
    if is_torch:
        if not host_result:
            return out
        # pinned staging (torch's caching host allocator): ~4x faster D2H than pageable
        host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        host.copy_(out, non_blocking=True)
        torch.cuda.current_stream(ad.device).synchronize()
        return host
    return out.to(torch.float64).cpu().numpy()


def run_equivalence(
    size: ProblemSize,
    tile: TileShape,
    hw: HardwareModel,
    policy: Policy,
    rng_seed: int,
    *,
    in_dtype="bf16",
) -> EquivalenceReport:
    """Build, execute on the GPU and compare one instance (executor.py:127-145)."""
    rng = np.random.default_rng(rng_seed)
    a = random_int_matrix(size.m, size.k, rng)
    b = random_int_matrix(size.k, size.n, rng)
    sched = build_schedule(size, tile, hw, policy)
    got = execute_schedule(a, b, sched, tile, size, in_dtype=in_dtype)
    want = reference_gemm(a, b)
    diff = np.abs(got - want)
    return EquivalenceReport(
        exact_match=bool(np.array_equal(got, want)),
        max_abs_diff=float(diff.max()) if diff.size else 0.0,
    )
