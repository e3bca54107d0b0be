"""Multi-GPU CSRC product: one process per GPU, row bands.

Two band forms:

* gather (default): rank g runs the gather kernel on its rows
  [block_start[g], block_start[g+1]); a row reads x below the band (its lower
  pairs) and above it (the rows that name it as a column), so x is replicated
  over [lo_g, x_hi_g) and the rank writes exactly its own y rows: no y
  exchange at all (weak-scaling shards, no data-path collective).
  For repeated products (an iterative solver feeding y back as x) each rank
  owns only x on its rows; ``apply_device(..., refresh_x=True)`` then
  exchanges the x halo [lo_g, row_begin) ∪ [row_end, x_hi_g) with grouped
  NCCL send/recv on a communication stream while the band's interior rows
  (``csrc_gpu_gather_interior``: rows reading only own x) run, and finishes
  the boundary rows once the halo has landed (``csrc_gpu_spmv_device_rows``).
* windowed (scatter): the y-halo reduce below.

Rank g owns rows [block_start[g], block_start[g+1]) of
``partition_by_nnz(a, world)`` (partition.hpp:55-90, bit-exact) and computes
its band with a band plan of the windowed kernel. Because ja[t] < row(t)
(csrc_matrix.hpp:18), a band only scatters *downward*, into
[lo_g, block_start[g]) where lo_g is its effective_range lo
(partition.hpp:94-102): that halo partial is shipped to the owning lower
ranks and added there. This is the reference's `effective` accumulation
(parallel.hpp:371-382) at GPU granularity.

Per product (``apply_device``):
  1. boundary rows (those whose scatters reach below block_start[g]) run
     first on the compute stream; an event marks the halo complete;
  2. the communication stream waits on that event and posts the grouped
     ncclSend/ncclRecv of the halo slices (torch.distributed P2P over NCCL,
     NVLink/NVSwitch on the B200 box);
  3. the interior rows run concurrently on the compute stream;
  4. the received partials are reduced into the owned rows with a red.global
     kernel (csrc_gpu_halo_accumulate) once the receives complete.

x is replicated over each rank's [lo_g, end_g).

Host mode (``band_compute`` given, CPU tensors, gloo) runs the same exchange
plan with an injected band product; tests/test_dist.py uses it to check the
halo logic on CPU with world size 2.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import numpy as np

from . import CsrcMatrix, GpuSpmv, Strategy, StrategyKind, effective_ranges, partition_by_nnz


@dataclass
class HaloPlan:
    rank: int
    world: int
    row_begin: int
    row_end: int
    lo: int
    # (peer, q0, q1): global positions [q0, q1) of my halo owned by peer
    sends: List[Tuple[int, int, int]]
    # (peer, q0, q1): global positions [q0, q1) of my rows in peer's halo
    recvs: List[Tuple[int, int, int]]
    # device vectors: x_local covers [x_lo, x_hi), y_local covers [y_lo, row_end)
    x_hi: int = -1
    y_lo: int = -1
    mode: str = "windowed"
    # gather form, x-halo refresh: (peer, q0, q1) global x positions I send
    # (my rows in peer's x range) / receive (peer's rows in my x range)
    x_sends: List[Tuple[int, int, int]] = dataclasses.field(default_factory=list)
    x_recvs: List[Tuple[int, int, int]] = dataclasses.field(default_factory=list)

    def __post_init__(self):
        if self.x_hi < 0:
            self.x_hi = self.row_end
        if self.y_lo < 0:
            self.y_lo = self.lo

    @property
    def x_lo(self) -> int:
        return self.lo

    @property
    def vec_len(self) -> int:
        return self.row_end - self.lo

    def halo_bytes(self, elem: int = 8) -> Tuple[int, int]:
        s = sum(q1 - q0 for _, q0, q1 in self.sends) * elem
        r = sum(q1 - q0 for _, q0, q1 in self.recvs) * elem
        return s, r


def band_x_hi(a: CsrcMatrix, r0: int, r1: int) -> int:
    """End of the x range rows [r0, r1) read in the gather form: one past the
    last row r whose stored pairs name a column in [r0, r1)."""
    rows = np.repeat(np.arange(a.n, dtype=np.int64), np.diff(a.ia))
    m = (a.ja >= r0) & (a.ja < r1)
    return int(max(r1, rows[m].max() + 1)) if m.any() else int(r1)


def bands_x_hi(a: CsrcMatrix, block_start: List[int]) -> List[int]:
    """band_x_hi for every band of a partition (csrc_bands_x_hi: one threaded
    pass over the rows in the product library)."""
    import ctypes as C
    from . import _check
    from . import _lib as L
    p = len(block_start) - 1
    bs = np.asarray(block_start, np.int32)
    out = np.zeros(max(p, 1), np.int32)
    _check(L.bands_x_hi(C.byref(a._c()), p, bs.ctypes.data_as(L.P_i32), out.ctypes.data_as(L.P_i32)))
    return [int(v) for v in out[:p]]


def gather_plan(a: CsrcMatrix, world: int, rank: int, x_hi: Optional[int] = None,
                all_x_hi: Optional[List[int]] = None) -> HaloPlan:
    """Gather-form band of rank `rank`: x over [lo, x_hi), own y rows only.
    The x-halo lists say which x rows move between ranks when only the owned
    rows of x are current (refresh_x)."""
    part = partition_by_nnz(a, world)
    ranges = effective_ranges(a, part)
    bs = [part.begin(b) for b in range(world)] + [a.n]
    his = all_x_hi if all_x_hi is not None else bands_x_hi(a, bs)
    r0, r1 = bs[rank], bs[rank + 1]
    hi = his[rank] if x_hi is None else x_hi
    lo = ranges[rank].lo
    x_sends, x_recvs = [], []
    for b in range(world):
        if b == rank:
            continue
        q0, q1 = max(lo, bs[b]), min(hi, bs[b + 1])  # peer b's rows inside my x range
        if q0 < q1:
            x_recvs.append((b, q0, q1))
        q0, q1 = max(ranges[b].lo, r0), min(his[b], r1)  # my rows inside peer b's x range
        if q0 < q1:
            x_sends.append((b, q0, q1))
    return HaloPlan(rank, world, r0, r1, lo, [], [], x_hi=hi, y_lo=r0, mode="gather",
                    x_sends=x_sends, x_recvs=x_recvs)


def halo_plan(a: CsrcMatrix, world: int, rank: int) -> HaloPlan:
    """Exchange plan of rank `rank` (identical inputs on every rank)."""
    part = partition_by_nnz(a, world)
    ranges = effective_ranges(a, part)
    r0, r1 = part.begin(rank), part.end(rank)
    lo = ranges[rank].lo
    sends, recvs = [], []
    for b in range(rank):  # owners of my halo [lo, r0)
        q0, q1 = max(lo, part.begin(b)), min(r0, part.end(b))
        if q0 < q1:
            sends.append((b, q0, q1))
    for c in range(rank + 1, world):  # higher ranks whose halo covers my rows
        q0, q1 = max(ranges[c].lo, r0), min(part.begin(c), r1)
        if q0 < q1:
            recvs.append((c, q0, q1))
    return HaloPlan(rank, world, r0, r1, lo, sends, recvs)


class DistSpmv:
    """Band-decomposed product on the current process group.

    Device mode: x_local covers global positions [plan.x_lo, plan.x_hi),
    y_local [plan.y_lo, plan.row_end) (CUDA tensors); after ``apply_device``
    the owned rows y_local[row_begin - y_lo:] hold the final product rows.
    Gather form: y_lo = row_begin, x_hi above the band; windowed form:
    x_lo = y_lo = lo, x_hi = row_end.
    """

    def __init__(self, a: CsrcMatrix, strategy: Optional[Strategy] = None, group=None,
                 band_compute: Optional[Callable] = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        s = strategy or Strategy(StrategyKind.gather)
        if s.kind in (StrategyKind.sequential, StrategyKind.local_buffers, StrategyKind.colorful):
            s = dataclasses.replace(s, kind=StrategyKind.gather)  # band forms: gather or scatter
        self.mode = "gather" if s.kind == StrategyKind.gather else "windowed"
        self.band_compute = band_compute
        self.ex = None
        if self.mode == "gather":
            part = partition_by_nnz(a, self.world)
            r0, r1 = part.begin(self.rank), part.end(self.rank)
            x_hi = None
            if band_compute is None:
                self.ex = GpuSpmv(a, s, band=(r0, r1))
                x_hi = int(self.ex.info().x_hi)
            self.plan = gather_plan(a, self.world, self.rank, x_hi)
            assert self.plan.x_hi == (x_hi if x_hi is not None else self.plan.x_hi)
        else:
            self.plan = halo_plan(a, self.world, self.rank)
            if band_compute is None:
                self.ex = GpuSpmv(a, s, band=(self.plan.row_begin, self.plan.row_end))
        if self.ex is not None:
            assert self.ex.info().lo == self.plan.lo
        self._bufs = None
        self._streams = None

    def close(self):
        if self.ex is not None:
            self.ex.close()
            self.ex = None

    # -------------------------------------------------------------- exchange
    def _staged(self) -> bool:
        """gloo moves CPU tensors only: device slices are staged through host
        copies (the one-GPU functional check of the N > 1 path; NCCL moves the
        device slices directly)."""
        if not hasattr(self, "_gloo"):
            self._gloo = self.dist.get_backend(self.group) == "gloo"
        return self._gloo

    def _batch(self, sends, recvs):
        """Grouped P2P: sends / recvs are (peer, tensor) lists. Returns works whose
        wait() also lands staged receives in their device slices."""
        dist = self.dist
        if not self._staged() or not any(t.is_cuda for _, t in sends + recvs):
            ops = [dist.P2POp(dist.isend, t, peer, self.group) for peer, t in sends]
            ops += [dist.P2POp(dist.irecv, t, peer, self.group) for peer, t in recvs]
            return dist.batch_isend_irecv(ops) if ops else []
        hs = [(peer, t.cpu()) for peer, t in sends]
        hr = [(peer, t, t.new_empty(t.shape, device="cpu")) for peer, t in recvs]
        ops = [dist.P2POp(dist.isend, h, peer, self.group) for peer, h in hs]
        ops += [dist.P2POp(dist.irecv, h, peer, self.group) for peer, _, h in hr]
        works = dist.batch_isend_irecv(ops) if ops else []

        class Landed:
            def wait(_self):
                for w in works:
                    w.wait()
                for _, dev_t, h in hr:
                    dev_t.copy_(h)
        return [Landed()]

    def _post_x(self, x_local):
        """Grouped P2P of the x halo (gather form): my rows to the peers whose
        x range covers them, the peers' rows into my halo slices."""
        p = self.plan
        return self._batch([(peer, x_local[q0 - p.x_lo:q1 - p.x_lo]) for peer, q0, q1 in p.x_sends],
                           [(peer, x_local[q0 - p.x_lo:q1 - p.x_lo]) for peer, q0, q1 in p.x_recvs])

    def exchange_x(self, x_local):
        """Blocking x-halo refresh: afterwards x_local holds current x on
        [x_lo, x_hi) given current values on the owned rows."""
        for w in self._post_x(x_local):
            w.wait()
        return x_local

    def _post(self, y_local, recv_bufs):
        p = self.plan
        return self._batch([(peer, y_local[q0 - p.lo:q1 - p.lo]) for peer, q0, q1 in p.sends],
                           [(peer, buf) for (peer, q0, q1), buf in zip(p.recvs, recv_bufs)])

    def apply_host(self, x_local, y_local, refresh_x: bool = False):
        """Host mode (gloo): band product via the injected callable."""
        import torch

        p = self.plan
        if refresh_x and self.mode == "gather":
            self.exchange_x(x_local)
        y_local.copy_(torch.as_tensor(self.band_compute(p, x_local.numpy())))
        if self.mode == "gather":
            return y_local  # own rows only, nothing to exchange
        recv_bufs = [torch.empty(q1 - q0, dtype=y_local.dtype) for _, q0, q1 in p.recvs]
        for w in self._post(y_local, recv_bufs):
            w.wait()
        for (peer, q0, q1), buf in zip(p.recvs, recv_bufs):
            y_local[q0 - p.lo:q1 - p.lo] += buf
        return y_local

    def apply_device(self, x_local, y_local, overlap: bool = True, refresh_x: bool = False):
        import torch

        p = self.plan
        if self.mode == "gather":
            if not refresh_x or (not p.x_sends and not p.x_recvs):
                self.ex.apply_device(x_local, y_local)
                return y_local
            if self._streams is None:
                self._streams = (torch.cuda.current_stream(), torch.cuda.Stream())
                self._ev_halo = torch.cuda.Event()
                self._ev_recv = torch.cuda.Event()
                self._interior = self.ex.gather_interior()
            comp, comm = self._streams
            g0, g1 = self._interior
            n_rows = p.row_end - p.row_begin
            self._ev_halo.record(comp)  # owned x rows are current on the compute stream
            comm.wait_event(self._ev_halo)
            with torch.cuda.stream(comm):
                for w in self._post_x(x_local):
                    w.wait()
                self._ev_recv.record(comm)
            if overlap and g0 < g1:
                self.ex.apply_device_rows(x_local, y_local, g0, g1, comp)  # interior: own x only
                comp.wait_event(self._ev_recv)
                self.ex.apply_device_rows(x_local, y_local, 0, g0, comp)
                self.ex.apply_device_rows(x_local, y_local, g1, n_rows, comp)
            else:
                comp.wait_event(self._ev_recv)
                self.ex.apply_device(x_local, y_local, comp)
            return y_local
        if self._streams is None:
            self._streams = (torch.cuda.current_stream(), torch.cuda.Stream())
            self._bufs = [torch.empty(q1 - q0, dtype=y_local.dtype, device=y_local.device)
                          for _, q0, q1 in p.recvs]
            self._ev_halo = torch.cuda.Event()
            self._ev_recv = torch.cuda.Event()
        comp, comm = self._streams
        if not overlap or (not p.sends and not p.recvs):
            self.ex.apply_device(x_local, y_local, comp)
            comm.wait_stream(comp)
            with torch.cuda.stream(comm):
                works = self._post(y_local, self._bufs)
                for w in works:
                    w.wait()
                self._ev_recv.record(comm)
        else:
            self.ex.apply_device_part(x_local, y_local, 0, comp)  # zero y + boundary rows
            self._ev_halo.record(comp)
            comm.wait_event(self._ev_halo)
            with torch.cuda.stream(comm):
                works = self._post(y_local, self._bufs)
                for w in works:
                    w.wait()
                self._ev_recv.record(comm)
            self.ex.apply_device_part(x_local, y_local, 1, comp)  # interior, overlaps the halo
        comp.wait_event(self._ev_recv)
        for (peer, q0, q1), buf in zip(p.recvs, self._bufs):
            self.ex.halo_accumulate(y_local, q0 - p.lo, buf, q1 - q0, comp)
        return y_local


def gather_product(plan: HaloPlan, y_local, world_y: Optional[np.ndarray] = None):
    """Owned rows of y_local as numpy (rows [row_begin, row_end))."""
    arr = y_local.detach().cpu().numpy() if hasattr(y_local, "detach") else np.asarray(y_local)
    own = arr[plan.row_begin - plan.y_lo:]
    if world_y is not None:
        world_y[plan.row_begin:plan.row_end] = own
    return own


# ------------------------------------------------------------- C-ABI executor
FORMS = {"windowed": 0, "gather": 1}


def band_lists(a: CsrcMatrix, world: int, rank: int, form: str):
    """The C-ABI executor's exchange lists (csrc_gpu_band_lists_get): (info,
    sends [(peer, q0, q1)], recvs [(peer, q0, q1)])."""
    import ctypes as C
    from . import _check
    from . import _lib as L
    info = L.BandLists()
    _check(L.band_lists_get(C.byref(a._c()), world, rank, FORMS[form], C.byref(info), None, None, None, None,
                            None, None))
    arr = [np.zeros(max(info.n_sends if i < 3 else info.n_recvs, 1), np.int32) for i in range(6)]
    _check(L.band_lists_get(C.byref(a._c()), world, rank, FORMS[form], C.byref(info),
                            *[x.ctypes.data_as(L.P_i32) for x in arr]))
    sends = [(int(p), int(q0), int(q1)) for p, q0, q1 in zip(arr[0][:info.n_sends], arr[1], arr[2])]
    recvs = [(int(p), int(q0), int(q1)) for p, q0, q1 in zip(arr[3][:info.n_recvs], arr[4], arr[5])]
    return info, sends, recvs


class NcclBandSpmv:
    """The C-ABI band executor (csrc_gpu_band_exec_*, paper_1003_0952_b200/csrc/
    bandexec.cpp): the band plan, the exchange lists and an NCCL communicator
    owned by the product library. The NCCL unique id is created on rank 0 and
    broadcast over the caller's torch.distributed group (any channel works)."""

    def __init__(self, a: CsrcMatrix, strategy: Optional[Strategy] = None, form: str = "windowed", group=None):
        import ctypes as C
        import torch
        import torch.distributed as dist
        from . import _check
        from . import _lib as L
        self._L, self._check = L, _check
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        idb = (C.c_uint8 * 128)()
        if rank == 0:
            _check(L.nccl_get_unique_id(idb))
        t = torch.tensor(list(bytes(idb)), dtype=torch.uint8)
        if world > 1:
            dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
            t = t.to(dev)
            dist.broadcast(t, 0, group)
            t = t.cpu()
        idb = (C.c_uint8 * 128)(*t.tolist())
        s = strategy or Strategy(StrategyKind[form])
        self._h = C.c_void_p()
        _check(L.band_exec_create(C.byref(a._c()), C.byref(s._c()), world, rank, FORMS[form], idb,
                                  C.byref(self._h)))
        info = L.BandLists()
        _check(L.band_exec_get_info(self._h, C.byref(info)))
        self.lists = info
        self.form = form

    def apply_device(self, x_local, y_local, refresh_x: bool = False, stream=None):
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(x_local.device)
        self._check(self._L.band_exec_apply(self._h, x_local.data_ptr(), y_local.data_ptr(),
                                            int(st.cuda_stream) or None, 1 if refresh_x else 0))

    def check(self):
        self._check(self._L.band_exec_check(self._h))

    def close(self):
        if self._h:
            self._L.band_exec_destroy(self._h)
            self._h = None
