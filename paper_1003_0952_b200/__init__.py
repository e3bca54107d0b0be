"""B200-native CSRC sparse matrix-vector product (arXiv 1003.0952 hot path).

Host mirror of the reference's C++ interface (/root/reference/proj/include/csrc)
over the C-ABI library ``libcsrc_b200.so`` (include/csrc_gpu.h):

=====================================  =============================================
reference (file:line)                  here
=====================================  =============================================
``csrc::CsrcMatrix`` csrc_matrix.hpp:14  :class:`CsrcMatrix`
``spmv_csrc`` kernels.hpp:25-43          :func:`spmv_csrc` (GPU, plan-free one-shot stream)
``spmv_csrc_transpose`` kernels.hpp:47   :func:`spmv_csrc_transpose`
``Strategy`` parallel.hpp:19-23          :class:`Strategy`
``ParallelSpmv`` parallel.hpp:151-446    :class:`GpuSpmv` (``ParallelSpmv`` alias)
``spmv_parallel`` parallel.hpp:449-454   :func:`spmv_parallel`
``allocation_stats`` parallel.hpp:35-38  :func:`allocation_stats`
``partition_by_nnz`` partition.hpp:55    :func:`partition_by_nnz`
``effective_ranges`` partition.hpp:104   :func:`effective_ranges`
``build_interval_plan`` partition.hpp:113 :func:`build_interval_plan`
``color_rows`` coloring.hpp:119-164      :func:`color_rows`
``validate_coloring`` coloring.hpp:175   :func:`validate_coloring`
``ColorfulPlan`` parallel.hpp:54-94      :class:`ColorfulPlan`
``LocalBuffersPlan`` parallel.hpp:40-52  :class:`LocalBuffersPlan`
``working_set_kb`` working_set.hpp:17    :func:`working_set_kb`
``count_ops`` cost_model.hpp:20-42       :func:`model_flops`
``build_csr`` csr.hpp:55-92              :func:`build_csr` (device, construct.py)
``csr_to_csrc`` csrc_matrix.hpp:44-91    :func:`csr_to_csrc`, :func:`build_csrc`
``decompose_rect`` csrc_matrix.hpp:113   :func:`decompose_rect`
``spmv_csrc_rect`` kernels.hpp:69-91     :func:`spmv_csrc_rect`; ``GpuSpmv(CsrcRectMatrix, s)``
``spmv_csr`` kernels.hpp:7-22            :func:`spmv_csr`; ``GpuSpmv(CsrMatrix, s)``
=====================================  =============================================

Errors raise :class:`Error` (``csrc::Error``, common.hpp:15-18) with the
reference's wording.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _lib as L

__all__ = [
    "Error", "CsrcMatrix", "StrategyKind", "AccumMethod", "ConflictMode", "ColorOrder",
    "DType", "Strategy", "PhaseTimings", "GpuSpmv", "ParallelSpmv", "spmv_csrc",
    "spmv_csrc_transpose", "spmv_parallel", "allocation_stats", "partition_by_nnz",
    "effective_ranges", "build_interval_plan", "RowPartition", "EffectiveRange",
    "IntervalPlan", "Coloring", "ColoringValidity", "color_rows", "validate_coloring",
    "conflict_edge_counts", "ColorfulPlan", "LocalBuffersPlan", "working_set_kb",
    "model_bytes", "model_flops", "Mesh", "generate_fixture", "CONFIGS", "config_matrix",
    "fixture_u01", "TripletMatrix", "CsrMatrix", "CsrcRectMatrix", "build_csr", "build_csrc",
    "csr_to_csrc", "decompose_rect", "csrc_to_triplets", "spmv_csrc_rect", "spmv_csr",
]


class Error(RuntimeError):
    """csrc::Error (common.hpp:15-18)."""


def _check(rc: int) -> None:
    if rc != 0:
        raise Error(L.last_error().decode(errors="replace"))


# --------------------------------------------------------------------- types
class StrategyKind(enum.IntEnum):
    """csrc::StrategyKind (parallel.hpp:16) plus the GPU-only kernels."""

    sequential = 0
    local_buffers = 1
    colorful = 2
    atomic = 3
    windowed = 4
    gather = 5


class AccumMethod(enum.IntEnum):
    """csrc::AccumMethod (parallel.hpp:17)."""

    all_in_one = 0
    per_buffer = 1
    effective = 2
    interval = 3


class ConflictMode(enum.IntEnum):
    """csrc::ConflictMode (coloring.hpp:15-18)."""

    neighborhood = 0
    exact = 1


class ColorOrder(enum.IntEnum):
    """csrc::ColorOrder (coloring.hpp:35)."""

    natural = 0
    largest_first = 1
    smallest_last = 2


class DType(enum.IntEnum):
    f64 = 0
    f32 = 1


@dataclass
class Strategy:
    """csrc::Strategy {kind, accum, p} (parallel.hpp:19-23) + device options."""

    kind: StrategyKind = StrategyKind.sequential
    accum: AccumMethod = AccumMethod.effective
    p: int = 1
    dtype: DType = DType.f64
    conflict_mode: ConflictMode = ConflictMode.neighborhood
    color_order: ColorOrder = ColorOrder.natural
    device: int = 0
    bands: int = 0  # device bands (CTAs); 0 = auto

    def _c(self) -> L.GpuStrategy:
        return L.GpuStrategy(int(self.kind), int(self.accum), int(self.p), int(self.dtype),
                             int(self.conflict_mode), int(self.color_order), int(self.device),
                             int(self.bands))


@dataclass
class PhaseTimings:
    """csrc::PhaseTimings (parallel.hpp:26-30); seconds, from CUDA events."""

    init_max: float = 0.0
    compute_max: float = 0.0
    accumulate_max: float = 0.0
    halo: float = 0.0


def _as(arr, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(arr), dtype=dtype)


@dataclass
class CsrcMatrix:
    """csrc::CsrcMatrix (csrc_matrix.hpp:14-30): ad[n], ia[n+1], ja[k] (< row),
    al[k] = a_ij, au[k] = a_ji (empty iff value_symmetric)."""

    n: int
    ad: np.ndarray
    ia: np.ndarray
    ja: np.ndarray
    al: np.ndarray
    au: np.ndarray = field(default_factory=lambda: np.zeros(0))
    value_symmetric: bool = False

    def __post_init__(self):
        self.n = int(self.n)
        self.ad = _as(self.ad, np.float64)
        self.ia = _as(self.ia, np.int32)
        self.ja = _as(self.ja, np.int32)
        self.al = _as(self.al, np.float64)
        self.au = _as(self.au, np.float64)
        self._keep = None

    def k_off(self) -> int:
        return int(self.ja.size)

    def nnz_full(self) -> int:
        return self.n + 2 * self.k_off()

    def nnz_stored(self) -> int:
        return self.n + (1 if self.value_symmetric else 2) * self.k_off()

    def upper(self) -> np.ndarray:
        return self.al if self.value_symmetric else self.au

    def _c(self) -> L.HostMatrix:
        if self.ia.size != self.n + 1 and not (self.n == 0 and self.ia.size in (0, 1)):
            raise Error(f"ia has length {self.ia.size}, expected {self.n + 1}")
        ia = self.ia if self.ia.size else np.zeros(1, np.int32)
        k = int(ia[self.n]) if self.n > 0 else 0
        if self.ja.size != k or self.al.size != k:
            raise Error(f"ja/al have lengths {self.ja.size}/{self.al.size}, expected ia[n] = {k}")
        if not self.value_symmetric and self.au.size != k:
            raise Error(f"au has length {self.au.size}, expected {k}")
        self._keep = ia
        ptr = lambda a, t: a.ctypes.data_as(C.POINTER(t)) if a.size else None  # noqa: E731
        return L.HostMatrix(
            self.n, k, ptr(self.ad, C.c_double), ia.ctypes.data_as(L.P_i32),
            ptr(self.ja, C.c_int32), ptr(self.al, C.c_double),
            None if self.value_symmetric else ptr(self.au, C.c_double),
            1 if self.value_symmetric else 0,
        )


def working_set_kb(n: int, nnz_stored: int, value_symmetric: bool) -> float:
    """working_set_kb (working_set.hpp:17-25)."""
    if n < 1:
        raise Error("working_set_kb: n must be >= 1")
    return L.model_bytes(n, nnz_stored, 1 if value_symmetric else 0, 0) / 1024.0


def model_bytes(a: CsrcMatrix, dtype: DType = DType.f64) -> int:
    """Algorithmic bytes of one product (working_set.hpp:11-23; fp32: 6nnz+10n+4)."""
    nnz = a.nnz_stored()
    return int(L.model_bytes(a.n, nnz, 1 if a.value_symmetric else 0, int(dtype)))


def model_flops(a: CsrcMatrix) -> int:
    """count_ops flops for csrc (cost_model.hpp:20-42, Format::csrc at :33): 2*nnz_full - n."""
    return int(L.model_flops(a.n, a.nnz_full()))


# ------------------------------------------------------------------ plans
@dataclass
class RowPartition:
    """csrc::RowPartition (partition.hpp:13-20)."""

    p: int
    block_start: List[int]
    block_nnz: List[int]

    def begin(self, t: int) -> int:
        return self.block_start[t]

    def end(self, t: int) -> int:
        return self.block_start[t + 1]


@dataclass
class EffectiveRange:
    """csrc::EffectiveRange (partition.hpp:24-29), inclusive [lo, hi]."""

    lo: int
    hi: int

    def covers(self, q: int) -> bool:
        return self.lo <= q <= self.hi


@dataclass
class IntervalPlan:
    """csrc::IntervalPlan (partition.hpp:33-41)."""

    boundaries: List[int]
    intervals: List[Tuple[int, int, List[int]]]  # (begin, end, contributors)


def partition_by_nnz(a: CsrcMatrix, p: int) -> RowPartition:
    bs = np.zeros(max(p, 0) + 1, np.int32)
    bn = np.zeros(max(p, 1), np.int64)
    _check(L.partition_by_nnz(C.byref(a._c()), p, bs.ctypes.data_as(L.P_i32),
                              bn.ctypes.data_as(L.P_i64)))
    return RowPartition(p, bs.tolist(), bn[:p].tolist())


def effective_ranges(a: CsrcMatrix, part: RowPartition) -> List[EffectiveRange]:
    bs = np.asarray(part.block_start, np.int32)
    lo = np.zeros(part.p, np.int32)
    hi = np.zeros(part.p, np.int32)
    _check(L.effective_ranges(C.byref(a._c()), part.p, bs.ctypes.data_as(L.P_i32),
                              lo.ctypes.data_as(L.P_i32), hi.ctypes.data_as(L.P_i32)))
    return [EffectiveRange(int(l), int(h)) for l, h in zip(lo, hi)]


def build_interval_plan(ranges: List[EffectiveRange]) -> IntervalPlan:
    p = len(ranges)
    lo = np.asarray([r.lo for r in ranges], np.int32)
    hi = np.asarray([r.hi for r in ranges], np.int32)
    ni, nc, nb = C.c_int32(), C.c_int32(), C.c_int32()
    P = L.P_i32
    lp, hp = lo.ctypes.data_as(P), hi.ctypes.data_as(P)
    _check(L.interval_plan(p, lp, hp, C.byref(ni), C.byref(nc), C.byref(nb),
                           None, None, None, None, None))
    ib = np.zeros(ni.value + 1, np.int32)
    ie = np.zeros(ni.value + 1, np.int32)
    cp = np.zeros(ni.value + 1, np.int32)
    cc = np.zeros(nc.value + 1, np.int32)
    bd = np.zeros(nb.value + 1, np.int32)
    _check(L.interval_plan(p, lp, hp, C.byref(ni), C.byref(nc), C.byref(nb),
                           ib.ctypes.data_as(P), ie.ctypes.data_as(P), cp.ctypes.data_as(P),
                           cc.ctypes.data_as(P), bd.ctypes.data_as(P)))
    ivs = [(int(ib[i]), int(ie[i]), cc[cp[i]:cp[i + 1]].tolist()) for i in range(ni.value)]
    return IntervalPlan(bd[: nb.value].tolist(), ivs)


@dataclass
class Coloring:
    """csrc::Coloring (coloring.hpp:29-33)."""

    color: np.ndarray
    n_colors: int

    @property
    def classes(self) -> List[np.ndarray]:
        return [np.flatnonzero(self.color == c).astype(np.int32) for c in range(self.n_colors)]


@dataclass
class ColoringValidity:
    """csrc::ColoringValidity (coloring.hpp:167-171)."""

    valid: bool
    row_a: int = -1
    row_b: int = -1
    position: int = -1


def color_rows(a: CsrcMatrix, mode: ConflictMode = ConflictMode.neighborhood,
               order: ColorOrder = ColorOrder.natural) -> Coloring:
    """color_rows(build_conflict_graph(a, mode), order) (coloring.hpp:93-164)."""
    color = np.zeros(max(a.n, 1), np.int32)
    nc = C.c_int32()
    _check(L.color_rows(C.byref(a._c()), int(mode), int(order), color.ctypes.data_as(L.P_i32),
                        C.byref(nc)))
    return Coloring(color[: a.n].copy(), nc.value)


def conflict_edge_counts(a: CsrcMatrix, mode: ConflictMode) -> Tuple[int, int]:
    d, i = C.c_int64(), C.c_int64()
    _check(L.conflict_edge_counts(C.byref(a._c()), int(mode), C.byref(d), C.byref(i)))
    return d.value, i.value


def validate_coloring(a: CsrcMatrix, c: Coloring) -> ColoringValidity:
    color = _as(c.color, np.int32)
    v, ra, rb, q = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    _check(L.validate_coloring(C.byref(a._c()), color.ctypes.data_as(L.P_i32), c.n_colors,
                               C.byref(v), C.byref(ra), C.byref(rb), C.byref(q)))
    return ColoringValidity(bool(v.value), ra.value, rb.value, q.value)


@dataclass
class ColorfulPlan:
    """csrc::ColorfulPlan (parallel.hpp:54-94)."""

    coloring: Coloring
    class_slices: Optional[np.ndarray] = None  # [n_colors, p, 2]

    @staticmethod
    def build(a: CsrcMatrix, p: int, mode: ConflictMode = ConflictMode.neighborhood,
              order: ColorOrder = ColorOrder.natural) -> "ColorfulPlan":
        plan = ColorfulPlan(color_rows(a, mode, order))
        plan.slice(a, p)
        return plan

    def slice(self, a: CsrcMatrix, p: int) -> None:
        out = np.zeros((max(self.coloring.n_colors, 1), p, 2), np.int64)
        color = _as(self.coloring.color, np.int32)
        _check(L.colorful_slices(C.byref(a._c()), color.ctypes.data_as(L.P_i32),
                                 self.coloring.n_colors, p, out.ctypes.data_as(L.P_i64)))
        self.class_slices = out[: self.coloring.n_colors]


@dataclass
class LocalBuffersPlan:
    """csrc::LocalBuffersPlan (parallel.hpp:40-52)."""

    partition: RowPartition
    ranges: List[EffectiveRange]
    intervals: IntervalPlan

    @staticmethod
    def build(a: CsrcMatrix, p: int) -> "LocalBuffersPlan":
        part = partition_by_nnz(a, p)
        ranges = effective_ranges(a, part)
        return LocalBuffersPlan(part, ranges, build_interval_plan(ranges))


def allocation_stats(s: Strategy) -> int:
    """allocation_stats (parallel.hpp:35-38)."""
    if s.kind == StrategyKind.local_buffers and s.p >= 2:
        return s.p
    return 0


# ---------------------------------------------------------------- executor
class GpuSpmv:
    """GPU counterpart of csrc::ParallelSpmv (parallel.hpp:151-446).

    ``GpuSpmv(a, strategy)`` builds the device plan (matrix copied to HBM);
    ``apply(x)`` / ``apply(x, y)`` run the product with host vectors (H2D of x,
    kernels, D2H of y); ``apply_device`` takes device pointers (torch tensors or
    raw ints) and enqueues asynchronously on a CUDA stream.
    """

    def __init__(self, a, strategy: Strategy = Strategy(), plan=None,
                 band: Optional[Tuple[int, int]] = None):
        if isinstance(a, CsrMatrix):
            # spmv_csr (kernels.hpp:7-22): a plan over a general CSR matrix
            if plan is not None or band is not None:
                raise Error("CSR plans take no explicit plan or band")
            self._a_n = int(a.n_rows)
            self._strategy = strategy
            self._plan_in = None
            self._h = C.c_void_p()
            rp = _as(a.row_ptr, np.int32)
            ci = _as(a.col_idx, np.int32)
            va = _as(a.values, np.float64)
            s = strategy._c()
            _check(L.plan_create_csr(int(a.n_rows), int(a.n_cols), rp.ctypes.data_as(L.P_i32),
                                     ci.ctypes.data_as(L.P_i32) if ci.size else None,
                                     va.ctypes.data_as(L.P_f64) if va.size else None, C.byref(s), C.byref(self._h)))
            self._timings = PhaseTimings()
            return
        rect = a if isinstance(a, CsrcRectMatrix) else None
        if rect is not None:
            a = rect.square
        self._a_n = a.n
        self._a_ref = a  # buffers_plan / colorful_plan are built from it on request
        self._strategy = strategy
        self._plan_in = plan
        self._h = C.c_void_p()
        cm = a._c()
        s = strategy._c()
        if rect is not None:
            # ParallelSpmv(const CsrcRectMatrix&, Strategy[, plan]) (parallel.hpp:168-181)
            if band is not None:
                raise Error("rectangular plans take no band")
            trp = _as(rect.rect.row_ptr, np.int32)
            tci = _as(rect.rect.col_idx, np.int32)
            tva = _as(rect.rect.values, np.float64)
            self._keep_rect = (trp, tci, tva)
            tp = (trp.ctypes.data_as(L.P_i32), tci.ctypes.data_as(L.P_i32) if tci.size else None,
                  tva.ctypes.data_as(L.P_f64) if tva.size else None)
            if plan is None:
                rc = L.plan_create_rect(C.byref(cm), C.byref(s), int(rect.m), *tp, C.byref(self._h))
            elif isinstance(plan, ColorfulPlan):
                color = _as(plan.coloring.color, np.int32)
                rc = L.plan_create_rect_plan(C.byref(cm), C.byref(s), int(rect.m), *tp,
                                             color.ctypes.data_as(L.P_i32), plan.coloring.n_colors, None, 0,
                                             C.byref(self._h))
            elif isinstance(plan, LocalBuffersPlan):
                bs = np.asarray(plan.partition.block_start, np.int32)
                rc = L.plan_create_rect_plan(C.byref(cm), C.byref(s), int(rect.m), *tp, None, 0,
                                             bs.ctypes.data_as(L.P_i32), plan.partition.p, C.byref(self._h))
            else:
                raise Error("plan must be a ColorfulPlan or LocalBuffersPlan")
        elif isinstance(plan, ColorfulPlan):
            color = _as(plan.coloring.color, np.int32)
            rc = L.plan_create_colored(C.byref(cm), C.byref(s), color.ctypes.data_as(L.P_i32),
                                       plan.coloring.n_colors, C.byref(self._h))
        elif isinstance(plan, LocalBuffersPlan):
            bs = np.asarray(plan.partition.block_start, np.int32)
            rc = L.plan_create_partitioned(C.byref(cm), C.byref(s), bs.ctypes.data_as(L.P_i32),
                                           plan.partition.p, C.byref(self._h))
        elif band is not None:
            rc = L.plan_create_band(C.byref(cm), C.byref(s), int(band[0]), int(band[1]),
                                    C.byref(self._h))
        elif plan is None:
            rc = L.plan_create(C.byref(cm), C.byref(s), C.byref(self._h))
        else:
            raise Error("plan must be a ColorfulPlan or LocalBuffersPlan")
        _check(rc)
        self._timings = PhaseTimings()

    def close(self) -> None:
        if self._h:
            L.plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> int:
        return self._h.value or 0

    def info(self) -> L.PlanInfo:
        inf = L.PlanInfo()
        _check(L.plan_get_info(self._h, C.byref(inf)))
        return inf

    def buffers_allocated(self) -> int:
        """ParallelSpmv::buffers_allocated (parallel.hpp:223)."""
        return self.info().buffers_allocated

    def strategy(self) -> Strategy:
        """ParallelSpmv::strategy (parallel.hpp:224)."""
        return self._strategy

    def _active(self) -> bool:
        s = self._strategy
        return s.kind in (StrategyKind.local_buffers, StrategyKind.colorful) and s.p >= 2

    def buffers_plan(self) -> Optional["LocalBuffersPlan"]:
        """ParallelSpmv::buffers_plan (parallel.hpp:225): the caller's plan, or the
        one build_default_plan (parallel.hpp:236-242) makes; None when inactive."""
        if isinstance(self._plan_in, LocalBuffersPlan):
            return self._plan_in
        if self._strategy.kind != StrategyKind.local_buffers or not self._active():
            return None
        if not hasattr(self, "_bp"):
            self._bp = LocalBuffersPlan.build(self._a_ref, self._strategy.p)
        return self._bp

    def colorful_plan(self) -> Optional["ColorfulPlan"]:
        """ParallelSpmv::colorful_plan (parallel.hpp:226): the colouring the plan runs,
        sliced for p workers (ColorfulPlan::slice, parallel.hpp:69-93)."""
        if isinstance(self._plan_in, ColorfulPlan):
            return self._plan_in
        if self._strategy.kind != StrategyKind.colorful or not self._active():
            return None
        if not hasattr(self, "_cp"):
            nc = C.c_int32()
            _check(L.plan_get_coloring(self._h, None, C.byref(nc)))
            color = np.zeros(max(self._a_n, 1), np.int32)
            _check(L.plan_get_coloring(self._h, color.ctypes.data_as(L.P_i32), C.byref(nc)))
            self._cp = ColorfulPlan(Coloring(color[: self._a_n], nc.value))
            self._cp.slice(self._a_ref, self._strategy.p)
        return self._cp

    def set_timing(self, on: bool = True) -> None:
        _check(L.set_timing(self._h, 1 if on else 0))

    def last_timings(self) -> PhaseTimings:
        """ParallelSpmv::last_timings (parallel.hpp:222), seconds."""
        t = L.Timings()
        _check(L.last_timings(self._h, C.byref(t)))
        return PhaseTimings(t.init_ms / 1e3, t.compute_ms / 1e3, t.accumulate_ms / 1e3,
                            t.halo_ms / 1e3)

    def apply(self, x, y: Optional[np.ndarray] = None, transpose: bool = False) -> np.ndarray:
        """ParallelSpmv::apply (parallel.hpp:183-220)."""
        xv = _as(x, np.float64)
        if y is None or y.dtype != np.float64 or not y.flags.c_contiguous:
            out = np.empty(self._a_n, np.float64)
        else:
            if y.size != self._a_n:
                y.resize(self._a_n, refcheck=False)
            out = y
        fn = L.spmv_transpose if transpose else L.spmv
        _check(fn(self._h, xv.ctypes.data_as(L.P_f64), xv.size, out.ctypes.data_as(L.P_f64)))
        if y is not None and out is not y:
            y[...] = out
            return y
        return out

    @staticmethod
    def _ptr(t) -> int:
        if t is None:
            return 0
        if isinstance(t, int):
            return t
        return int(t.data_ptr())

    @staticmethod
    def _stream(stream, t=None):
        """The cudaStream_t a device call enqueues on. An int is a raw handle
        (0 = the plan's own stream, as in the C ABI). None with torch tensors
        = torch's current stream on the tensor's device, like any torch op;
        None with raw pointers = the plan's stream. Torch's default stream is
        the legacy NULL stream: it is passed as cudaStreamLegacy (handle 1),
        because a NULL handle means the plan's (non-blocking) stream."""
        if isinstance(stream, int):
            return stream or None
        if stream is None:
            if t is None or isinstance(t, int):
                return None
            import torch
            stream = torch.cuda.current_stream(t.device)
        return int(stream.cuda_stream) or 1

    def apply_device(self, x, y, stream=None, transpose: bool = False) -> None:
        """y = A x on device tensors (or raw pointers), enqueued on `stream`
        (default: torch's current stream, see _stream)."""
        _check(L.spmv_device(self._h, self._ptr(x), self._ptr(y), self._stream(stream, x),
                             1 if transpose else 0))

    def apply_device_graph(self, x, y, stream=None) -> None:
        """apply_device replayed from a CUDA graph. stream None = the plan's
        own stream (a graph cannot be captured on the legacy NULL stream)."""
        st = stream if isinstance(stream, int) else (stream.cuda_stream if stream else 0)
        _check(L.spmv_device_graph(self._h, self._ptr(x), self._ptr(y), st or None))

    def apply_device_part(self, x, y, part: int, stream=None) -> None:
        _check(L.spmv_device_part(self._h, self._ptr(x), self._ptr(y), self._stream(stream, x), part))

    def halo_accumulate(self, y, dst_off: int, recv, length: int, stream=None) -> None:
        _check(L.halo_accumulate(self._h, self._ptr(y), dst_off, self._ptr(recv), length,
                                 self._stream(stream, y)))

    def gather_interior(self) -> Tuple[int, int]:
        """Rows (plan-relative) that read x only on the plan's own rows."""
        a, b = C.c_int32(), C.c_int32()
        _check(L.gather_interior(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def apply_device_rows(self, x, y, rows_begin: int, rows_end: int, stream=None,
                          transpose: bool = False) -> None:
        """Gather plans: the product on rows [rows_begin, rows_end) only."""
        _check(L.spmv_device_rows(self._h, self._ptr(x), self._ptr(y), self._stream(stream, x),
                                  1 if transpose else 0,
                                  int(rows_begin), int(rows_end)))

    def band_split(self) -> int:
        v = C.c_int32()
        _check(L.band_split(self._h, C.byref(v)))
        return v.value

    def time_products(self, x, y, reps: int, flush_bytes: int = 0):
        tot = np.zeros(reps, np.float64)
        ker = np.zeros(reps, np.float64)
        _check(L.time_products(self._h, self._ptr(x), self._ptr(y), reps, flush_bytes,
                               tot.ctypes.data_as(L.P_f64), ker.ctypes.data_as(L.P_f64)))
        return tot, ker


ParallelSpmv = GpuSpmv


def spmv_parallel(a: CsrcMatrix, x, s: Strategy) -> Tuple[np.ndarray, PhaseTimings]:
    """spmv_parallel (parallel.hpp:449-454)."""
    ex = GpuSpmv(a, s)
    try:
        ex.set_timing(True)
        y = ex.apply(x)
        return y, ex.last_timings()
    finally:
        ex.close()


def _oneshot(a: CsrcMatrix, xv: np.ndarray, transpose: bool, device: int) -> np.ndarray:
    y = np.empty(a.n, np.float64)
    _check(L.spmv_oneshot(C.byref(a._c()), xv.ctypes.data_as(L.P_f64), xv.size, y.ctypes.data_as(L.P_f64),
                          1 if transpose else 0, device))
    return y


def spmv_csrc(a: CsrcMatrix, x, dtype: DType = DType.f64, device: int = 0) -> np.ndarray:
    """spmv_csrc (kernels.hpp:25-43) on the GPU, one shot: fp64 streams the CSRC
    arrays as stored through the plan-free path (csrc_gpu_spmv_oneshot); fp32
    builds a plan (the one-shot path is fp64, the reference's type)."""
    xv = _as(x, np.float64)
    if xv.size != a.n:
        raise Error(f"spmv_csrc: x has length {xv.size}, expected {a.n}")
    if dtype == DType.f64:
        return _oneshot(a, xv, False, device)
    ex = GpuSpmv(a, Strategy(StrategyKind.sequential, dtype=dtype, device=device))
    try:
        return ex.apply(xv)
    finally:
        ex.close()


def spmv_csr(a, x, dtype: DType = DType.f64) -> np.ndarray:
    """spmv_csr (kernels.hpp:7-22) on the GPU: a general CSR matrix (CsrMatrix)."""
    xv = _as(x, np.float64)
    if xv.size != a.n_cols:
        raise Error(f"spmv_csr: x has length {xv.size}, expected {a.n_cols}")
    ex = GpuSpmv(a, Strategy(StrategyKind.sequential, dtype=dtype))
    try:
        return ex.apply(xv)
    finally:
        ex.close()


def spmv_csrc_rect(a, x, dtype: DType = DType.f64) -> np.ndarray:
    """spmv_csrc_rect (kernels.hpp:69-91): CSRC square part + CSR tail; x has m entries."""
    xv = _as(x, np.float64)
    if xv.size != a.m:
        raise Error(f"spmv_csrc_rect: x has length {xv.size}, expected {a.m}")
    ex = GpuSpmv(a, Strategy(StrategyKind.sequential, dtype=dtype))
    try:
        return ex.apply(xv)
    finally:
        ex.close()


def spmv_csrc_transpose(a: CsrcMatrix, x, dtype: DType = DType.f64) -> np.ndarray:
    """spmv_csrc_transpose (kernels.hpp:47-65): al/au swapped, zero-copy."""
    xv = _as(x, np.float64)
    if xv.size != a.n:
        raise Error(f"spmv_csrc_transpose: x has length {xv.size}, expected {a.n}")
    if dtype == DType.f64:
        return _oneshot(a, xv, True, 0)
    ex = GpuSpmv(a, Strategy(StrategyKind.sequential, dtype=dtype))
    try:
        return ex.apply(xv, transpose=True)
    finally:
        ex.close()


# ---------------------------------------------------------------- fixtures
class Mesh(enum.IntEnum):
    grid2d_q1 = 0
    grid3d_27 = 1
    elasticity = 2
    grid3d_27_rcm = 3


def fixture_u01(seed: int, a: int, b: int) -> float:
    return float(L.fixture_u01(seed, a, b))


def generate_fixture(mesh: Mesh, nx: int, ny: int, nz: int, seed: int, diag_base: float,
                     threads: int = 0):
    """Synthetic FE matrix in CSRC form + x.

    Returns (CsrcMatrix, x, order) where order[u] is the final index of
    natural node/dof u.
    """
    spec = L.FixtureSpec(int(mesh), nx, ny, nz, seed, diag_base, threads)
    h = C.c_void_p()
    _check(L.fixture_generate(C.byref(spec), C.byref(h)))
    try:
        m = L.HostMatrix()
        _check(L.fixture_matrix(h, C.byref(m)))
        n, k = m.n, m.k
        cp = lambda p, cnt, dt: np.ctypeslib.as_array(p, shape=(cnt,)).astype(dt, copy=True)  # noqa: E731
        a = CsrcMatrix(
            n,
            cp(m.ad, n, np.float64),
            cp(m.ia, n + 1, np.int32),
            cp(m.ja, k, np.int32) if k else np.zeros(0, np.int32),
            cp(m.al, k, np.float64) if k else np.zeros(0),
            cp(m.au, k, np.float64) if k else np.zeros(0),
            False,
        )
        x = cp(L.fixture_x(h), n, np.float64)
        order = cp(L.fixture_order(h), n, np.int32)
    finally:
        L.fixture_free(h)
    return a, x, order


# BASELINE.json configs: mesh, nx, ny, nz, seed, diag_base
CONFIGS = {
    "c1": dict(mesh=Mesh.grid2d_q1, nx=256, ny=256, nz=1, seed=42, diag_base=10.0,
               desc="2D Q1 256x256, 9-point, seed 42"),
    "c2": dict(mesh=Mesh.grid3d_27, nx=64, ny=64, nz=64, seed=7, diag_base=30.0,
               desc="3D 64^3, 27-point, seed 7"),
    "c3": dict(mesh=Mesh.grid3d_27_rcm, nx=160, ny=160, nz=160, seed=11, diag_base=30.0,
               desc="3D 160^3, 27-point, permuted (seed 11) + RCM"),
    "c4": dict(mesh=Mesh.elasticity, nx=96, ny=96, nz=96, seed=3, diag_base=100.0,
               desc="elasticity 96^3 x 3 dof, 81-entry rows, seed 3"),
    "c5": dict(mesh=Mesh.grid3d_27, nx=256, ny=256, nz=256, seed=99, diag_base=30.0,
               desc="3D 256^3, 27-point, seed 99"),
}


def config_matrix(name: str, threads: int = 0):
    c = CONFIGS[name]
    return generate_fixture(c["mesh"], c["nx"], c["ny"], c["nz"], c["seed"], c["diag_base"],
                            threads)


from .construct import (  # noqa: E402  (needs Error / CsrcMatrix defined above)
    CsrMatrix, CsrcRectMatrix, TripletMatrix, build_csr, build_csrc, csr_to_csrc, csrc_to_triplets,
    decompose_rect,
)
