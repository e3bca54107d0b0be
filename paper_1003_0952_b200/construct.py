"""CSRC construction on the GPU: host mirror of the reference's ingestion
types and functions over the C-ABI (include/csrc_gpu.h, csrc/assemble.cu).

=========================================  ======================================
reference (file:line)                      here
=========================================  ======================================
``csrc::TripletMatrix`` csr.hpp:13-24        :class:`TripletMatrix`
``csrc::CsrMatrix`` csr.hpp:28-51            :class:`CsrMatrix`
``build_csr`` csr.hpp:55-92                  :func:`build_csr` (device sort + reduce)
``csr_to_csrc`` csrc_matrix.hpp:44-91        :func:`csr_to_csrc`, :func:`build_csrc`
``CsrcRectMatrix`` csrc_matrix.hpp:35-39     :class:`CsrcRectMatrix`
``decompose_rect`` csrc_matrix.hpp:113-142   :func:`decompose_rect`
``csrc_to_csr`` csrc_matrix.hpp:95-108       :func:`csrc_to_triplets` (its triplet order)
=========================================  ======================================

All of these run on ``device`` (default 0) and fail with :class:`Error` when
no GPU is present; there is no host fallback. Results are zero-copy numpy
views of the library's host arrays; the handle is freed with the last view.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

from . import _lib as L


def _err():
    from . import Error  # late import: __init__ imports this module
    return Error


def _check(rc: int) -> None:
    if rc != 0:
        raise _err()(L.last_error().decode(errors="replace"))


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t)) if a.size else None


class _Owner:
    """Keeps a csrc_built_t alive while numpy views of its host arrays exist."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            L.built_free(self.h)
        except Exception:
            pass


def _view(p, count: int, ctype, dt, owner: _Owner) -> np.ndarray:
    """Zero-copy numpy view of `count` elements at `p`, owned by the handle."""
    if count == 0:
        return np.zeros(0, dt)
    buf = (ctype * count).from_address(C.cast(p, C.c_void_p).value)
    buf._owner = owner  # the array's base keeps the handle alive
    return np.frombuffer(buf, dtype=dt)


@dataclass
class TripletMatrix:
    """csrc::TripletMatrix (csr.hpp:13-24): coordinate entries, duplicates
    summed by :func:`build_csr`."""

    n_rows: int = 0
    n_cols: int = 0
    rows: List[int] = field(default_factory=list)
    cols: List[int] = field(default_factory=list)
    values: List[float] = field(default_factory=list)

    def add(self, row: int, col: int, value: float) -> None:
        self.rows.append(int(row))
        self.cols.append(int(col))
        self.values.append(float(value))

    def arrays(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        return (np.ascontiguousarray(self.rows, np.int32), np.ascontiguousarray(self.cols, np.int32),
                np.ascontiguousarray(self.values, np.float64))


@dataclass
class CsrMatrix:
    """csrc::CsrMatrix (csr.hpp:28-51), canonical: columns strictly increasing."""

    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return int(self.values.size)

    def has_entry(self, row: int, col: int) -> bool:
        b, e = int(self.row_ptr[row]), int(self.row_ptr[row + 1])
        q = b + int(np.searchsorted(self.col_idx[b:e], col))
        return q < e and int(self.col_idx[q]) == col

    def at(self, row: int, col: int) -> float:
        b, e = int(self.row_ptr[row]), int(self.row_ptr[row + 1])
        q = b + int(np.searchsorted(self.col_idx[b:e], col))
        return float(self.values[q]) if q < e and int(self.col_idx[q]) == col else 0.0


@dataclass
class CsrcRectMatrix:
    """csrc::CsrcRectMatrix (csrc_matrix.hpp:35-39): CSRC square part + CSR
    tail over columns n..m-1 with local column indices."""

    square: object
    rect: CsrMatrix
    m: int


def _triplet_args(t, n_rows=None, n_cols=None):
    if isinstance(t, TripletMatrix):
        r, c, v = t.arrays()
        return t.n_rows, t.n_cols, r, c, v
    n_rows, n_cols, r, c, v = t
    return (int(n_rows), int(n_cols), np.ascontiguousarray(r, np.int32),
            np.ascontiguousarray(c, np.int32), np.ascontiguousarray(v, np.float64))


def _csrc_from_handle(h, owner: _Owner):
    from . import CsrcMatrix
    m = L.HostMatrix()
    _check(L.built_matrix(h, C.byref(m)))
    n, k = m.n, m.k
    sym = bool(m.value_symmetric)
    f, i = C.c_double, C.c_int32
    return CsrcMatrix(n, _view(m.ad, n, f, np.float64, owner), _view(m.ia, n + 1, i, np.int32, owner),
                      _view(m.ja, k, i, np.int32, owner), _view(m.al, k, f, np.float64, owner),
                      np.zeros(0) if sym else _view(m.au, k, f, np.float64, owner), sym)


def _timings(h) -> dict:
    ms = (C.c_double * 4)()
    _check(L.built_timings(h, ms))
    return dict(h2d_ms=ms[0], sort_ms=ms[1], convert_ms=ms[2], d2h_ms=ms[3])


def build_csr(t, device: int = 0) -> CsrMatrix:
    """build_csr (csr.hpp:55-92): canonical CSR, duplicates summed (device
    radix sort + run reduction). ``t`` is a :class:`TripletMatrix` or a tuple
    (n_rows, n_cols, rows, cols, values)."""
    nr, nc, r, c, v = _triplet_args(t)
    h = C.c_void_p()
    _check(L.build_csr(nr, nc, r.size, _ptr(r, C.c_int32), _ptr(c, C.c_int32), _ptr(v, C.c_double),
                       device, C.byref(h)))
    owner = _Owner(h)
    n_rows, n_cols, nnz = C.c_int32(), C.c_int32(), C.c_int64()
    rp, ci, va = L.P_i32(), L.P_i32(), L.P_f64()
    _check(L.built_csr(h, C.byref(n_rows), C.byref(n_cols), C.byref(nnz), C.byref(rp), C.byref(ci),
                       C.byref(va)))
    return CsrMatrix(n_rows.value, n_cols.value, _view(rp, n_rows.value + 1, C.c_int32, np.int32, owner),
                     _view(ci, nnz.value, C.c_int32, np.int32, owner),
                     _view(va, nnz.value, C.c_double, np.float64, owner))


def build_csrc(t, device: int = 0, timings: dict = None):
    """csr_to_csrc(build_csr(t)) fused on the device (no CSR round trip)."""
    nr, nc, r, c, v = _triplet_args(t)
    if nr != nc:
        raise _err()("csr_to_csrc: matrix is not square")
    h = C.c_void_p()
    _check(L.build_csrc(nr, r.size, _ptr(r, C.c_int32), _ptr(c, C.c_int32), _ptr(v, C.c_double), device,
                        C.byref(h)))
    owner = _Owner(h)
    if timings is not None:
        timings.update(_timings(h))
    return _csrc_from_handle(h, owner)


def csr_to_csrc(a: CsrMatrix, device: int = 0):
    """csr_to_csrc (csrc_matrix.hpp:44-91) of a canonical CSR."""
    rp = np.ascontiguousarray(a.row_ptr, np.int32)
    ci = np.ascontiguousarray(a.col_idx, np.int32)
    va = np.ascontiguousarray(a.values, np.float64)
    h = C.c_void_p()
    _check(L.csr_to_csrc(int(a.n_rows), int(a.n_cols), rp.ctypes.data_as(L.P_i32), _ptr(ci, C.c_int32),
                         _ptr(va, C.c_double), device, C.byref(h)))
    return _csrc_from_handle(h, _Owner(h))


def decompose_rect(a: CsrMatrix, device: int = 0) -> CsrcRectMatrix:
    """decompose_rect (csrc_matrix.hpp:113-142, symmetrize = false)."""
    rp = np.ascontiguousarray(a.row_ptr, np.int32)
    ci = np.ascontiguousarray(a.col_idx, np.int32)
    va = np.ascontiguousarray(a.values, np.float64)
    h = C.c_void_p()
    _check(L.decompose_rect(int(a.n_rows), int(a.n_cols), rp.ctypes.data_as(L.P_i32), _ptr(ci, C.c_int32),
                            _ptr(va, C.c_double), device, C.byref(h)))
    owner = _Owner(h)
    sq = _csrc_from_handle(h, owner)
    m, nnz = C.c_int32(), C.c_int64()
    trp, tci, tva = L.P_i32(), L.P_i32(), L.P_f64()
    _check(L.built_rect_tail(h, C.byref(m), C.byref(nnz), C.byref(trp), C.byref(tci), C.byref(tva)))
    tail = CsrMatrix(sq.n, m.value - sq.n, _view(trp, sq.n + 1, C.c_int32, np.int32, owner),
                     _view(tci, nnz.value, C.c_int32, np.int32, owner),
                     _view(tva, nnz.value, C.c_double, np.float64, owner))
    return CsrcRectMatrix(sq, tail, m.value)


def csrc_to_triplets(a) -> Tuple[int, int, np.ndarray, np.ndarray, np.ndarray]:
    """The triplets csrc_to_csr (csrc_matrix.hpp:95-108) feeds build_csr, in
    its order: per row i, (i, i, ad), then per stored pair (i, j, al), (j, i, au)."""
    n = a.n
    cnt = np.diff(a.ia.astype(np.int64))
    rows_of = np.repeat(np.arange(n, dtype=np.int32), cnt)
    per_row = 1 + 2 * cnt
    start = np.concatenate([[0], np.cumsum(per_row)[:-1]]).astype(np.int64)
    m = int(per_row.sum())
    r = np.empty(m, np.int32)
    c = np.empty(m, np.int32)
    v = np.empty(m, np.float64)
    r[start] = np.arange(n, dtype=np.int32)
    c[start] = np.arange(n, dtype=np.int32)
    v[start] = a.ad
    k = a.ja.size
    if k:
        t = np.arange(k, dtype=np.int64)
        base = start[rows_of] + 1 + 2 * (t - a.ia[rows_of].astype(np.int64))
        r[base], c[base], v[base] = rows_of, a.ja, a.al
        r[base + 1], c[base + 1], v[base + 1] = a.ja, rows_of, a.upper()
    return n, n, r, c, v
