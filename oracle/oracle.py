"""ORACLE — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker (or the timed
CPU baseline). The product (paper_1003_0952_b200/) never imports it.

Two checkers:
  * ``Oracle``  — the plain-C restatement in oracle/csrc_oracle.c (always
    available once ``make -C oracle`` ran), each function citing the reference
    file:line it restates;
  * ``Ref``     — the reference itself, compiled from /root/reference headers
    into oracle/_ref/libcsrc_ref.so (available where it was built).

plus a numpy restatement of the fixture definitions (``mesh_triplets``) that
builds the BASELINE meshes entry by entry, so the reference's own
build_csr -> csr_to_csrc pipeline can pin the product's direct CSRC assembly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libcsrc_oracle.so")
FIXTURES_SO = os.path.join(HERE, "_build", "libcsrc_fixtures.so")


def host_isa_level() -> int:
    """x86-64 micro-architecture level (2, 3 or 4) of the CPU this process runs
    on, from /proc/cpuinfo flags. Stands in for -march=native: the reference is
    compiled here once per level (oracle/Makefile) and loaded at the host's."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    fl = set(line.split(":", 1)[1].split())
                    break
            else:
                return 2
    except OSError:
        return 2
    v3 = {"avx", "avx2", "bmi1", "bmi2", "f16c", "fma", "movbe", "abm", "xsave"}
    v4 = {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"}
    if v3 <= fl:
        return 4 if v4 <= fl else 3
    return 2


def _ref_so() -> str:
    lvl = host_isa_level()
    for l in range(lvl, 1, -1):
        p = os.path.join(HERE, "_ref", "libcsrc_ref.so" if l == 2 else f"libcsrc_ref_v{l}.so")
        if os.path.exists(p):
            return p
    return os.path.join(HERE, "_ref", "libcsrc_ref.so")


# The checker is the x86-64-v2 build: no FMA contraction, so its arithmetic is the
# plain-C oracle's bit for bit (tests/test_oracle.py). The ISA-level builds are the
# timed CPU baseline only (bench.py); with FMA their y differs in the last bits.
REF_SO = os.path.join(HERE, "_ref", "libcsrc_ref.so")
REF_SO_FAST = _ref_so()


def host_cores() -> dict:
    """Logical CPUs this process may run on and the physical cores behind them
    (sysfs topology: distinct (package, core) pairs of the allowed CPUs)."""
    cpus = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count() or 1))
    phys = set()
    for c in cpus:
        base = f"/sys/devices/system/cpu/cpu{c}/topology/"
        try:
            with open(base + "physical_package_id") as f:
                pk = f.read().strip()
            with open(base + "core_id") as f:
                co = f.read().strip()
            phys.add((pk, co))
        except OSError:
            phys.add(("?", str(c)))
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return dict(logical=len(cpus), physical=len(phys), model=model, isa_level=host_isa_level())

P_i32 = C.POINTER(C.c_int32)
P_i64 = C.POINTER(C.c_int64)
P_f64 = C.POINTER(C.c_double)
P_int = C.POINTER(C.c_int)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None and a.size else None


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class Oracle:
    """ctypes wrapper of oracle/csrc_oracle.c."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        self.lib = C.CDLL(ORACLE_SO)
        L = self.lib
        L.oracle_working_set_bytes.restype = C.c_int64
        L.oracle_working_set_bytes.argtypes = [C.c_int64, C.c_int64, C.c_int]
        L.oracle_color_rows.restype = C.c_int

    def spmv_csrc(self, a, x, transpose=False):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(a.n, np.float64)
        au = None if a.value_symmetric else a.au
        fn = self.lib.oracle_spmv_csrc_transpose if transpose else self.lib.oracle_spmv_csrc
        fn(C.c_int32(a.n), _p(a.ad, C.c_double), _p(a.ia, C.c_int32), _p(a.ja, C.c_int32),
           _p(a.al, C.c_double), _p(au, C.c_double), _p(x, C.c_double), _p(y, C.c_double))
        return y

    def spmv_csrc_rect(self, r, x):
        """spmv_csrc_rect (kernels.hpp:69-91); r has .square, .rect, .m."""
        a, t = r.square, r.rect
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(a.n, np.float64)
        au = None if a.value_symmetric else a.au
        self.lib.oracle_spmv_csrc_rect(
            C.c_int32(a.n), _p(a.ad, C.c_double), _p(a.ia, C.c_int32), _p(a.ja, C.c_int32),
            _p(a.al, C.c_double), _p(au, C.c_double), _p(np.ascontiguousarray(t.row_ptr, np.int32), C.c_int32),
            _p(np.ascontiguousarray(t.col_idx, np.int32), C.c_int32),
            _p(np.ascontiguousarray(t.values, np.float64), C.c_double), _p(x, C.c_double), _p(y, C.c_double))
        return y

    def spmv_local_buffers(self, a, x, block_start):
        x = np.ascontiguousarray(x, np.float64)
        p = len(block_start) - 1
        bs = np.asarray(block_start, np.int32)
        y = np.zeros(a.n, np.float64)
        scratch = np.zeros(p * a.n, np.float64)
        au = None if a.value_symmetric else a.au
        self.lib.oracle_spmv_local_buffers(
            C.c_int32(a.n), _p(a.ad, C.c_double), _p(a.ia, C.c_int32), _p(a.ja, C.c_int32),
            _p(a.al, C.c_double), _p(au, C.c_double), _p(x, C.c_double), C.c_int(p),
            _p(bs, C.c_int32), _p(y, C.c_double), _p(scratch, C.c_double))
        return y

    def build_csrc(self, n, rows, cols, vals):
        """build_csr -> csr_to_csrc. Returns a CsrcMatrix-like dict or raises."""
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = np.ascontiguousarray(vals, np.float64)
        m = rows.size
        rp = np.zeros(n + 1, np.int32)
        ci = np.zeros(max(m, 1), np.int32)
        vv = np.zeros(max(m, 1), np.float64)
        nnz = C.c_int64()
        bad = C.c_int64()
        rc = self.lib.oracle_build_csr(C.c_int32(n), C.c_int32(n), C.c_int64(m), _p(rows, C.c_int32),
                                       _p(cols, C.c_int32), _p(vals, C.c_double),
                                       _p(rp, C.c_int32), _p(ci, C.c_int32), _p(vv, C.c_double),
                                       C.byref(nnz), C.byref(bad))
        if rc:
            e = bad.value
            raise ValueError(f"build_csr: entry ({rows[e]}, {cols[e]}) outside {n}x{n} bounds")
        ad = np.zeros(n, np.float64)
        ia = np.zeros(n + 1, np.int32)
        ja = np.zeros(max(nnz.value, 1), np.int32)
        al = np.zeros(max(nnz.value, 1), np.float64)
        au = np.zeros(max(nnz.value, 1), np.float64)
        k = C.c_int64()
        vs = C.c_int()
        ei, ej = C.c_int32(), C.c_int32()
        rc = self.lib.oracle_csr_to_csrc(C.c_int32(n), _p(rp, C.c_int32), _p(ci, C.c_int32),
                                         _p(vv, C.c_double), _p(ad, C.c_double), _p(ia, C.c_int32),
                                         _p(ja, C.c_int32), _p(al, C.c_double), _p(au, C.c_double),
                                         C.byref(k), C.byref(vs), C.byref(ei), C.byref(ej))
        if rc == 2:
            i, j = ei.value, ej.value
            raise ValueError(f"csr_to_csrc: entry ({i}, {j}) has no transpose ({j}, {i})")
        if rc == 3:
            raise ValueError(f"csr_to_csrc: row {ei.value} has no diagonal entry")
        kk = k.value
        return dict(n=n, ad=ad, ia=ia, ja=ja[:kk].copy(), al=al[:kk].copy(),
                    au=np.zeros(0) if vs.value else au[:kk].copy(), value_symmetric=bool(vs.value))

    def partition_by_nnz(self, a, p):
        bs = np.zeros(p + 1, np.int32)
        bn = np.zeros(max(p, 1), np.int64)
        rc = self.lib.oracle_partition_by_nnz(C.c_int32(a.n), _p(a.ia, C.c_int32),
                                              C.c_int(int(a.value_symmetric)), C.c_int(p),
                                              _p(bs, C.c_int32), _p(bn, C.c_int64))
        if rc:
            raise ValueError(f"partition_by_nnz: need 1 <= p <= n, got p={p}, n={a.n}")
        return bs.tolist(), bn[:p].tolist()

    def effective_ranges(self, a, block_start):
        p = len(block_start) - 1
        bs = np.asarray(block_start, np.int32)
        lo = np.zeros(p, np.int32)
        hi = np.zeros(p, np.int32)
        self.lib.oracle_effective_ranges(_p(a.ia, C.c_int32), _p(a.ja, C.c_int32), C.c_int(p),
                                         _p(bs, C.c_int32), _p(lo, C.c_int32), _p(hi, C.c_int32))
        return lo.tolist(), hi.tolist()

    def interval_plan(self, lo, hi):
        p = len(lo)
        lo = np.asarray(lo, np.int32)
        hi = np.asarray(hi, np.int32)
        bd = np.zeros(2 * p + 1, np.int32)
        ib = np.zeros(2 * p + 1, np.int32)
        ie = np.zeros(2 * p + 1, np.int32)
        cp = np.zeros(2 * p + 2, np.int32)
        cc = np.zeros(2 * p * p + 1, np.int32)
        nb, ni = C.c_int(), C.c_int()
        self.lib.oracle_interval_plan(C.c_int(p), _p(lo, C.c_int32), _p(hi, C.c_int32),
                                      _p(bd, C.c_int32), C.byref(nb), _p(ib, C.c_int32),
                                      _p(ie, C.c_int32), _p(cp, C.c_int32), _p(cc, C.c_int32),
                                      C.byref(ni))
        ivs = [(int(ib[i]), int(ie[i]), cc[cp[i]:cp[i + 1]].tolist()) for i in range(ni.value)]
        return bd[: nb.value].tolist(), ivs

    def color_rows(self, a, mode=0, order=0):
        color = np.zeros(max(a.n, 1), np.int32)
        nc = self.lib.oracle_color_rows(C.c_int32(a.n), _p(a.ia, C.c_int32), _p(a.ja, C.c_int32),
                                        C.c_int(mode), C.c_int(order), _p(color, C.c_int32))
        return color[: a.n].copy(), nc

    def conflict_edge_counts(self, a, mode=0):
        d, i = C.c_int64(), C.c_int64()
        self.lib.oracle_conflict_edge_counts(C.c_int32(a.n), _p(a.ia, C.c_int32),
                                             _p(a.ja, C.c_int32), C.c_int(mode), C.byref(d),
                                             C.byref(i))
        return d.value, i.value

    def validate_coloring(self, a, color, n_colors):
        color = np.ascontiguousarray(color, np.int32)
        ra, rb, q = C.c_int32(), C.c_int32(), C.c_int32()
        ok = self.lib.oracle_validate_coloring(C.c_int32(a.n), _p(a.ia, C.c_int32),
                                               _p(a.ja, C.c_int32), _p(color, C.c_int32),
                                               C.c_int(n_colors), C.byref(ra), C.byref(rb),
                                               C.byref(q))
        return bool(ok), ra.value, rb.value, q.value

    def working_set_bytes(self, n, nnz, vs):
        return int(self.lib.oracle_working_set_bytes(n, nnz, int(vs)))

    def count_ops(self, fmt, n, nnz_full):
        f, l = C.c_int64(), C.c_int64()
        self.lib.oracle_count_ops(C.c_int(fmt), C.c_int64(n), C.c_int64(nnz_full), C.byref(f),
                                  C.byref(l))
        return f.value, l.value

    def bench_source_vector(self, n):
        x = np.zeros(n, np.float64)
        self.lib.oracle_bench_source_vector(C.c_int64(n), _p(x, C.c_double))
        return x


class Ref:
    """ctypes wrapper of the reference itself (oracle/_ref/libcsrc_ref.so)."""

    def __init__(self, fast=False):
        so = REF_SO_FAST if fast else REF_SO
        if not os.path.exists(so):
            raise FileNotFoundError(so)
        self.so = so
        self.lib = C.CDLL(so)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_trip_size.restype = C.c_int64
        L.ref_exec_create.restype = C.c_void_p
        L.ref_exec_create.argtypes = [C.c_int32, C.c_int64, P_f64, P_i32, P_i32, P_f64, P_f64,
                                      C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.ref_exec_run.restype = C.c_double
        L.ref_exec_run.argtypes = [C.c_void_p, P_f64, P_f64, C.c_int32, P_f64]
        L.ref_exec_destroy.argtypes = [C.c_void_p]
        L.ref_exec_buffers.argtypes = [C.c_void_p]
        L.ref_working_set_kb.restype = C.c_double
        L.ref_working_set_kb.argtypes = [C.c_int64, C.c_int64, C.c_int32]
        L.ref_gen_random_sym.argtypes = [C.c_int32, C.c_double, C.c_uint64, C.c_int32]

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def _chk(self, rc):
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())

    def _trip(self):
        m = self.lib.ref_trip_size()
        r = np.zeros(m, np.int32)
        c = np.zeros(m, np.int32)
        v = np.zeros(m, np.float64)
        self.lib.ref_trip_copy(_p(r, C.c_int32), _p(c, C.c_int32), _p(v, C.c_double))
        return r, c, v

    def gen_random_sym(self, n, density, seed, vs=False):
        self._chk(self.lib.ref_gen_random_sym(n, density, seed, int(vs)))
        return self._trip()

    def gen_band(self, n, h, vs=False):
        self._chk(self.lib.ref_gen_band(C.c_int32(n), C.c_int32(h), C.c_int32(int(vs))))
        return self._trip()

    def gen_dense(self, n):
        self._chk(self.lib.ref_gen_dense(C.c_int32(n)))
        return self._trip()

    def build_csrc(self, n, rows, cols, vals):
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = np.ascontiguousarray(vals, np.float64)
        self._chk(self.lib.ref_build_csrc(C.c_int32(n), C.c_int64(rows.size), _p(rows, C.c_int32),
                                          _p(cols, C.c_int32), _p(vals, C.c_double)))
        nn, k, vs = C.c_int32(), C.c_int64(), C.c_int32()
        self.lib.ref_built_sizes(C.byref(nn), C.byref(k), C.byref(vs))
        kk = k.value
        ad = np.zeros(n, np.float64)
        ia = np.zeros(n + 1, np.int32)
        ja = np.zeros(max(kk, 1), np.int32)
        al = np.zeros(max(kk, 1), np.float64)
        au = np.zeros(max(kk, 1), np.float64)
        self.lib.ref_built_copy(_p(ad, C.c_double), _p(ia, C.c_int32), _p(ja, C.c_int32),
                                _p(al, C.c_double), _p(au, C.c_double))
        return dict(n=n, ad=ad, ia=ia, ja=ja[:kk].copy(), al=al[:kk].copy(),
                    au=np.zeros(0) if vs.value else au[:kk].copy(), value_symmetric=bool(vs.value))

    def build_csr(self, n_rows, n_cols, rows, cols, vals):
        """build_csr (csr.hpp:55-92) -> (row_ptr, col_idx, values)."""
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = np.ascontiguousarray(vals, np.float64)
        self._chk(self.lib.ref_build_csr(C.c_int32(n_rows), C.c_int32(n_cols), C.c_int64(rows.size),
                                         _p(rows, C.c_int32), _p(cols, C.c_int32), _p(vals, C.c_double)))
        return self._csr_out()

    def _csr_out(self):
        nr, nc, nnz = C.c_int32(), C.c_int32(), C.c_int64()
        self.lib.ref_csr_sizes(C.byref(nr), C.byref(nc), C.byref(nnz))
        rp = np.zeros(nr.value + 1, np.int32)
        ci = np.zeros(max(nnz.value, 1), np.int32)
        va = np.zeros(max(nnz.value, 1), np.float64)
        self.lib.ref_csr_copy(_p(rp, C.c_int32), _p(ci, C.c_int32), _p(va, C.c_double))
        return rp, ci[: nnz.value].copy(), va[: nnz.value].copy()

    def _built_out(self):
        nn, k, vs = C.c_int32(), C.c_int64(), C.c_int32()
        self.lib.ref_built_sizes(C.byref(nn), C.byref(k), C.byref(vs))
        n, kk = nn.value, k.value
        ad = np.zeros(max(n, 1), np.float64)
        ia = np.zeros(n + 1, np.int32)
        ja = np.zeros(max(kk, 1), np.int32)
        al = np.zeros(max(kk, 1), np.float64)
        au = np.zeros(max(kk, 1), np.float64)
        self.lib.ref_built_copy(_p(ad, C.c_double), _p(ia, C.c_int32), _p(ja, C.c_int32),
                                _p(al, C.c_double), _p(au, C.c_double))
        return dict(n=n, ad=ad[:n].copy(), ia=ia, ja=ja[:kk].copy(), al=al[:kk].copy(),
                    au=np.zeros(0) if vs.value else au[:kk].copy(), value_symmetric=bool(vs.value))

    def decompose_rect(self, n_rows, n_cols, rp, ci, va):
        """decompose_rect (csrc_matrix.hpp:113-142) -> (square dict, (trp, tci, tva))."""
        rp = np.ascontiguousarray(rp, np.int32)
        ci = np.ascontiguousarray(ci, np.int32)
        va = np.ascontiguousarray(va, np.float64)
        self._chk(self.lib.ref_decompose_rect(C.c_int32(n_rows), C.c_int32(n_cols), _p(rp, C.c_int32),
                                              _p(ci, C.c_int32), _p(va, C.c_double)))
        return self._built_out(), self._csr_out()

    def spmv_csr(self, n_rows, n_cols, rp, ci, va, x):
        """spmv_csr (kernels.hpp:7-22) of the reference itself."""
        rp = np.ascontiguousarray(rp, np.int32)
        ci = np.ascontiguousarray(ci, np.int32)
        va = np.ascontiguousarray(va, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(max(n_rows, 1), np.float64)
        self._chk(self.lib.ref_spmv_csr(C.c_int32(n_rows), C.c_int32(n_cols), _p(rp, C.c_int32), _p(ci, C.c_int32),
                                        _p(va, C.c_double), _p(x, C.c_double), _p(y, C.c_double)))
        return y[:n_rows]

    def spmv_csrc_rect(self, r, x):
        """spmv_csrc_rect (kernels.hpp:69-91) of the reference itself."""
        a, t = r.square, r.rect
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(a.n, np.float64)
        au = None if a.value_symmetric else a.au
        trp = np.ascontiguousarray(t.row_ptr, np.int32)
        tci = np.ascontiguousarray(t.col_idx, np.int32)
        tva = np.ascontiguousarray(t.values, np.float64)
        self._chk(self.lib.ref_spmv_csrc_rect(
            C.c_int32(a.n), C.c_int64(a.ja.size), _p(a.ad, C.c_double), _p(a.ia, C.c_int32),
            _p(a.ja, C.c_int32), _p(a.al, C.c_double), _p(au, C.c_double),
            C.c_int32(int(a.value_symmetric)), C.c_int32(r.m), _p(trp, C.c_int32), _p(tci, C.c_int32),
            _p(tva, C.c_double), _p(x, C.c_double), C.c_int64(x.size), _p(y, C.c_double)))
        return y

    def spmv_csrc(self, a, x, transpose=False):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(a.n, np.float64)
        au = None if a.value_symmetric else a.au
        self._chk(self.lib.ref_spmv_csrc(
            C.c_int32(a.n), C.c_int64(a.ja.size), _p(a.ad, C.c_double), _p(a.ia, C.c_int32),
            _p(a.ja, C.c_int32), _p(a.al, C.c_double), _p(au, C.c_double),
            C.c_int32(int(a.value_symmetric)), _p(x, C.c_double), _p(y, C.c_double),
            C.c_int32(int(transpose))))
        return y

    def partition_by_nnz(self, a, p):
        bs = np.zeros(p + 1, np.int32)
        bn = np.zeros(max(p, 1), np.int64)
        self._chk(self.lib.ref_partition_by_nnz(C.c_int32(a.n), C.c_int64(a.ja.size),
                                                _p(a.ia, C.c_int32), C.c_int32(int(a.value_symmetric)),
                                                C.c_int32(p), _p(bs, C.c_int32), _p(bn, C.c_int64)))
        return bs.tolist(), bn[:p].tolist()

    def effective_ranges(self, a, block_start):
        p = len(block_start) - 1
        bs = np.asarray(block_start, np.int32)
        lo = np.zeros(p, np.int32)
        hi = np.zeros(p, np.int32)
        self._chk(self.lib.ref_effective_ranges(C.c_int32(a.n), C.c_int64(a.ja.size),
                                                _p(a.ia, C.c_int32), _p(a.ja, C.c_int32),
                                                C.c_int32(p), _p(bs, C.c_int32), _p(lo, C.c_int32),
                                                _p(hi, C.c_int32)))
        return lo.tolist(), hi.tolist()

    def interval_plan(self, lo, hi):
        p = len(lo)
        lo = np.asarray(lo, np.int32)
        hi = np.asarray(hi, np.int32)
        ni, nb = C.c_int32(), C.c_int32()
        ib = np.zeros(2 * p + 1, np.int32)
        ie = np.zeros(2 * p + 1, np.int32)
        cp = np.zeros(2 * p + 2, np.int32)
        cc = np.zeros(2 * p * p + 1, np.int32)
        bd = np.zeros(2 * p + 1, np.int32)
        self._chk(self.lib.ref_interval_plan(C.c_int32(p), _p(lo, C.c_int32), _p(hi, C.c_int32),
                                             C.byref(ni), _p(ib, C.c_int32), _p(ie, C.c_int32),
                                             _p(cp, C.c_int32), _p(cc, C.c_int32), C.byref(nb),
                                             _p(bd, C.c_int32)))
        ivs = [(int(ib[i]), int(ie[i]), cc[cp[i]:cp[i + 1]].tolist()) for i in range(ni.value)]
        return bd[: nb.value].tolist(), ivs

    def color_rows(self, a, mode=0, order=0):
        color = np.zeros(max(a.n, 1), np.int32)
        nc = C.c_int32()
        nd, ni = C.c_int64(), C.c_int64()
        self._chk(self.lib.ref_color_rows(C.c_int32(a.n), C.c_int64(a.ja.size), _p(a.ia, C.c_int32),
                                          _p(a.ja, C.c_int32), C.c_int32(mode), C.c_int32(order),
                                          _p(color, C.c_int32), C.byref(nc), C.byref(nd),
                                          C.byref(ni)))
        return color[: a.n].copy(), nc.value, (nd.value, ni.value)

    def validate_coloring(self, a, color, n_colors):
        color = np.ascontiguousarray(color, np.int32)
        out = np.zeros(4, np.int32)
        self._chk(self.lib.ref_validate_coloring(C.c_int32(a.n), C.c_int64(a.ja.size),
                                                 _p(a.ia, C.c_int32), _p(a.ja, C.c_int32),
                                                 _p(color, C.c_int32), C.c_int32(n_colors),
                                                 _p(out, C.c_int32)))
        return bool(out[0]), int(out[1]), int(out[2]), int(out[3])

    def colorful_slices(self, a, color, n_colors, p):
        color = np.ascontiguousarray(color, np.int32)
        out = np.zeros(max(n_colors, 1) * p * 2, np.int64)
        self._chk(self.lib.ref_colorful_slices(C.c_int32(a.n), C.c_int64(a.ja.size),
                                               _p(a.ia, C.c_int32), C.c_int32(int(a.value_symmetric)),
                                               _p(color, C.c_int32), C.c_int32(n_colors),
                                               C.c_int32(p), _p(out, C.c_int64)))
        return out[: n_colors * p * 2].reshape(n_colors, p, 2)

    def exec_create(self, a, kind, accum, p):
        au = None if a.value_symmetric else a.au
        h = self.lib.ref_exec_create(a.n, a.ja.size, _p(a.ad, C.c_double), _p(a.ia, C.c_int32),
                                     _p(a.ja, C.c_int32), _p(a.al, C.c_double), _p(au, C.c_double),
                                     int(a.value_symmetric), kind, accum, p)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return h

    def exec_run(self, h, x, reps, n):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(n, np.float64)
        ph = np.zeros(3, np.float64)
        dt = self.lib.ref_exec_run(h, _p(x, C.c_double), _p(y, C.c_double), reps, _p(ph, C.c_double))
        return dt, y, ph

    def exec_buffers(self, h):
        return int(self.lib.ref_exec_buffers(h))

    def exec_destroy(self, h):
        self.lib.ref_exec_destroy(h)

    def working_set_kb(self, n, nnz, vs):
        return float(self.lib.ref_working_set_kb(n, nnz, int(vs)))


# ------------------------------------------------- fixtures without the product
class CpuCsrc:
    """Plain CSRC arrays (the csrc::CsrcMatrix fields) for the oracle side."""

    def __init__(self, n, ad, ia, ja, al, au, value_symmetric=False):
        self.n, self.ad, self.ia, self.ja, self.al, self.au = int(n), ad, ia, ja, al, au
        self.value_symmetric = bool(value_symmetric)

    def k_off(self):
        return int(self.ja.size)

    def nnz_full(self):
        return self.n + 2 * self.k_off()

    def nnz_stored(self):
        return self.n + (1 if self.value_symmetric else 2) * self.k_off()


# BASELINE.json configs (the same definitions as paper_1003_0952_b200.CONFIGS,
# checked equal in tests/test_oracle.py): mesh, nx, ny, nz, seed, diag_base
ORACLE_CONFIGS = {
    "c1": (0, 256, 256, 1, 42, 10.0),
    "c2": (1, 64, 64, 64, 7, 30.0),
    "c3": (3, 160, 160, 160, 11, 30.0),
    "c4": (2, 96, 96, 96, 3, 100.0),
    "c5": (1, 256, 256, 256, 99, 30.0),
}


class _FixtureSpec(C.Structure):
    _fields_ = [("mesh", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("seed", C.c_uint64), ("diag_base", C.c_double), ("threads", C.c_int32)]


class _HostMatrix(C.Structure):
    _fields_ = [("n", C.c_int32), ("k", C.c_int64), ("ad", P_f64), ("ia", P_i32), ("ja", P_i32),
                ("al", P_f64), ("au", P_f64), ("value_symmetric", C.c_int32)]


def fixture(mesh, nx, ny, nz, seed, diag_base, threads=0):
    """The seeded fixture from the standalone generator
    oracle/_build/libcsrc_fixtures.so (fixtures/csrc_fixtures.cpp) -- the
    reference arm and oracle-side code never map the product library.
    Returns (CpuCsrc, x)."""
    if not os.path.exists(FIXTURES_SO):
        build_oracle()
    lib = C.CDLL(FIXTURES_SO)
    lib.csrc_fixture_generate.argtypes = [C.POINTER(_FixtureSpec), C.POINTER(C.c_void_p)]
    lib.csrc_fixture_matrix.argtypes = [C.c_void_p, C.POINTER(_HostMatrix)]
    lib.csrc_fixture_x.restype = P_f64
    lib.csrc_fixture_x.argtypes = [C.c_void_p]
    lib.csrc_fixture_free.argtypes = [C.c_void_p]
    lib.csrc_fixture_last_error.restype = C.c_char_p
    spec = _FixtureSpec(int(mesh), nx, ny, nz, seed, diag_base, threads)
    h = C.c_void_p()
    if lib.csrc_fixture_generate(C.byref(spec), C.byref(h)):
        raise ValueError(lib.csrc_fixture_last_error().decode())
    try:
        m = _HostMatrix()
        lib.csrc_fixture_matrix(h, C.byref(m))
        n, k = m.n, m.k
        cp = lambda q, cnt: np.ctypeslib.as_array(q, shape=(cnt,)).copy() if cnt else np.zeros(0, q._type_)  # noqa
        a = CpuCsrc(n, cp(m.ad, n), cp(m.ia, n + 1), cp(m.ja, k), cp(m.al, k), cp(m.au, k), False)
        x = cp(lib.csrc_fixture_x(h), n)
    finally:
        lib.csrc_fixture_free(h)
    return a, x


def config_fixture(name, threads=0):
    return fixture(*ORACLE_CONFIGS[name], threads=threads)


def working_set_bytes(n, nnz_stored, value_symmetric=False, f32=False):
    """working_set_kb (working_set.hpp:17-25) in bytes: 8(ad+al+au+x+y) + 4(ia+ja)
    for f64 values; f32 values: 4 per value."""
    k = (nnz_stored - n) // (1 if value_symmetric else 2)
    vb = 4 if f32 else 8
    vals = n + (1 if value_symmetric else 2) * k
    return vb * (vals + 2 * n) + 4 * (n + 1 + k)


# ------------------------------------------------- fixture restatement (numpy)
# U01(seed, a, b) = (h >> 11) * 2^-53 with
# h = mix(mix(mix(seed*G + C0) ^ a*K1) ^ b*K2), mix = splitmix64 finaliser.
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def u01(seed, a, b):
    with np.errstate(over="ignore"):
        s = np.uint64(seed)
        h = _mix(s * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x632BE59BD9B4E019))
        h = _mix(h ^ (np.asarray(a, np.uint64) * np.uint64(0xD6E8FEB86659FD93)))
        h = _mix(h ^ (np.asarray(b, np.uint64) * np.uint64(0xCA5A826395121157)))
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


X_STREAM = 1 << 32
PERM_STREAM = 1 << 33


def _grid_pairs(nx, ny, nz):
    """All (u, v) node pairs with v in the 27/9-point neighbourhood of u, u != v."""
    x, y, z = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    u = ((z * ny + y) * nx + x).ravel()
    x, y, z = x.ravel(), y.ravel(), z.ravel()
    us, vs = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if dx == dy == dz == 0:
                    continue
                xx, yy, zz = x + dx, y + dy, z + dz
                ok = (xx >= 0) & (xx < nx) & (yy >= 0) & (yy < ny) & (zz >= 0) & (zz < nz)
                us.append(u[ok])
                vs.append(((zz * ny + yy) * nx + xx)[ok])
    return np.concatenate(us), np.concatenate(vs)


def rcm_reference(n, adj):
    """Pure-Python deterministic RCM, adj = list of sorted lists."""
    deg = [len(a) for a in adj]
    key = lambda v: (deg[v], v)  # noqa: E731
    placed = [False] * n
    order = []

    def bfs(r):
        level = {r: 0}
        q = [r]
        h = 0
        while h < len(q):
            v = q[h]
            h += 1
            for w in adj[v]:
                if not placed[w] and w not in level:
                    level[w] = level[v] + 1
                    q.append(w)
        ecc = max(level.values())
        return ecc, [v for v in q if level[v] == ecc]

    while len(order) < n:
        r = min((v for v in range(n) if not placed[v]), key=key)
        ecc, last = bfs(r)
        while True:
            c = min(last, key=key)
            ecc_c, last_c = bfs(c)
            if ecc_c <= ecc:
                break
            r, ecc, last = c, ecc_c, last_c
        head = len(order)
        order.append(r)
        placed[r] = True
        while head < len(order):
            v = order[head]
            head += 1
            nb = sorted((w for w in adj[v] if not placed[w]), key=key)
            for w in nb:
                placed[w] = True
                order.append(w)
    order.reverse()
    return order  # order[new] = label


def mesh_triplets(mesh, nx, ny, nz, seed, diag_base):
    """Entry-by-entry restatement of a fixture: (n, rows, cols, vals, x, order).

    mesh: 0 grid2d_q1, 1 grid3d_27, 2 elasticity (3 dof), 3 grid3d_27_rcm.
    Values attach to natural ids; for RCM meshes the final matrix is P A P^T.
    """
    dof = 3 if mesh == 2 else 1
    nodes = nx * ny * nz
    n = nodes * dof
    u, v = _grid_pairs(nx, ny, nz)
    f = np.arange(nodes, dtype=np.int64)
    if mesh == 3:
        p = np.arange(nodes, dtype=np.int64)
        for i in range(nodes - 1, 0, -1):
            j = int(u01(seed, i, PERM_STREAM) * (i + 1))
            j = min(j, i)
            p[i], p[j] = p[j], p[i]
        pinv = np.empty_like(p)
        pinv[p] = np.arange(nodes)
        adj = [[] for _ in range(nodes)]
        for a_, b_ in zip(p[u].tolist(), p[v].tolist()):
            adj[a_].append(b_)
        adj = [sorted(a_) for a_ in adj]
        cm = rcm_reference(nodes, adj)
        f = np.empty(nodes, np.int64)
        for new, lab in enumerate(cm):
            f[pinv[lab]] = new
    # dof-level entries in natural ids
    if dof == 1:
        ni, nj = u, v
    else:
        ni = (u[:, None, None] * 3 + np.arange(3)[None, :, None]).repeat(3, axis=2).ravel()
        nj = (v[:, None, None] * 3 + np.arange(3)[None, None, :]).repeat(3, axis=1).ravel()
        # intra-node off-diagonal couplings
        base = np.arange(nodes)[:, None, None] * 3
        ai = (base + np.arange(3)[None, :, None]).repeat(3, axis=2).ravel()
        bj = (base + np.arange(3)[None, None, :]).repeat(3, axis=1).ravel()
        keep = ai != bj
        ni = np.concatenate([ni, ai[keep]])
        nj = np.concatenate([nj, bj[keep]])
    vals = 2.0 * u01(seed, ni, nj) - 1.0
    diag_nat = np.arange(n, dtype=np.int64)
    dvals = diag_base + u01(seed, diag_nat, diag_nat)
    # final ids
    fd = (f[diag_nat // dof] * dof + diag_nat % dof)
    rows = np.concatenate([fd, f[ni // dof] * dof + ni % dof]).astype(np.int32)
    cols = np.concatenate([fd, f[nj // dof] * dof + nj % dof]).astype(np.int32)
    allv = np.concatenate([dvals, vals])
    x = 2.0 * u01(seed, np.arange(n), X_STREAM) - 1.0
    order = (f[np.arange(n) // dof] * dof + np.arange(n) % dof).astype(np.int32)
    return n, rows, cols, allv, x, order


def rel_l2(y, ref):
    ref = np.asarray(ref, np.float64)
    d = np.linalg.norm(np.asarray(y, np.float64) - ref)
    nrm = np.linalg.norm(ref)
    return d / nrm if nrm > 0 else d


def rel_inf(y, ref):
    """relative_error (bench.hpp:93-100): inf-norm, 0 denominator -> absolute."""
    ref = np.asarray(ref, np.float64)
    num = np.max(np.abs(np.asarray(y, np.float64) - ref)) if ref.size else 0.0
    den = np.max(np.abs(ref)) if ref.size else 0.0
    return num if den == 0.0 else num / den
