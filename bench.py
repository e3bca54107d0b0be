"""Benchmark: CSRC SpMV GFLOP/s and effective HBM GB/s (% of roofline) on B200.

One step = one product y = A x over the workload (default: BASELINE.json
config 5, the 3D 256^3 27-point FE matrix in fp64, n = 16.8M, nnz = 449M,
4.80 GB per product by the reference's working-set model).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--dtype f64]
  python bench.py --impl reference ...     reference CPU implementation

N > 1 runs under torchrun, one rank per GPU: rank g owns a partition_by_nnz row
band and the halo partials travel over NCCL (paper_1003_0952_b200/dist.py).
Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CSRC SpMV GFLOP/s and effective HBM GB/s (% of roofline) at 1/2/4/8 B200"


def load_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(workload):
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(workload)
    return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append(dict(sm=float(f[1]), smax=float(f[2]), power=float(f[3]),
                                 hw=f[5], hwt=f[6], swt=f[7], pcap=f[8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = set()
        for r in rows:
            if r["hw"] == "Active":
                reasons.add("hw_slowdown")
            if r["hwt"] == "Active":
                reasons.add("hw_thermal_slowdown")
            if r["swt"] == "Active":
                reasons.add("sw_thermal_slowdown")
            if r["pcap"] == "Active":
                reasons.add("sw_power_cap")
        return {"sm_mhz": statistics.median(r["sm"] for r in rows),
                "sm_max_mhz": max(r["smax"] for r in rows), "samples": len(rows),
                "reasons": sorted(reasons)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


REF_METHODS = [("sequential", 0, 0), ("all_in_one", 1, 0), ("per_buffer", 1, 1), ("effective", 1, 2),
               ("interval", 1, 3)]


def cpu_reference_suite(a, x, seconds, ref_threads=None):
    """The reference's own CPU path timed on this host:
    sequential spmv_csrc (kernels.hpp:25-43, via ParallelSpmv p=1, parallel.hpp:197-202)
    and ParallelSpmv local buffers x {all_in_one, per_buffer, effective, interval}
    (parallel.hpp:309-397) at p = the physical cores this process may use, from
    oracle/_ref (compiled from /root/reference for the host's x86-64 ISA level).
    Colorful is not timed: the reference's std::set conflict graph does not fit at
    C3-C5 (34 GB / 371 s exact, > 62 GB neighbourhood at C5).
    Falls back to the plain-C oracle port (1 thread) where oracle/_ref is absent.
    Each method: one warm product, then a bounded sample of products (median of 3
    runs, bench.hpp:125-128). Returns a dict; `best` names the fastest method."""
    from oracle.oracle import Oracle, Ref, host_cores
    flops = 2 * a.nnz_full()
    hc = host_cores()
    p = ref_threads or max(1, hc["physical"])
    methods = {}
    if Ref.available():
        R = Ref(fast=True)  # the host's ISA-level build (timed baseline)
        per = seconds / len(REF_METHODS)
        for name, kind, accum in REF_METHODS:
            h = R.exec_create(a, kind, accum, 1 if kind == 0 else p)
            try:
                dt1, y, _ = R.exec_run(h, x, 1, a.n)  # warm (first touch of the buffers)
                reps = max(1, min(1000, int(per / 3 / max(dt1, 1e-6))))
                runs = []
                for _ in range(3 if dt1 * reps * 3 <= per * 1.5 else 1):
                    dt, y, ph = R.exec_run(h, x, reps, a.n)
                    runs.append((dt / reps, ph / reps))
                runs.sort(key=lambda r: r[0])
                t, ph = runs[len(runs) // 2]
            finally:
                R.exec_destroy(h)
            methods[name] = dict(ms=t * 1e3, gflops=flops / t / 1e9, p=1 if kind == 0 else p, reps=reps,
                                 runs=len(runs), init_ms=ph[0] * 1e3, compute_ms=ph[1] * 1e3,
                                 accumulate_ms=ph[2] * 1e3)
        kind_s, lib = "reference", os.path.relpath(R.so, ROOT)
    else:
        O = Oracle()
        t0 = time.perf_counter()
        O.spmv_csrc(a, x)
        dt1 = time.perf_counter() - t0
        reps = max(1, min(200, int(seconds / max(dt1, 1e-6))))
        t0 = time.perf_counter()
        for _ in range(reps):
            O.spmv_csrc(a, x)
        t = (time.perf_counter() - t0) / reps
        methods["sequential"] = dict(ms=t * 1e3, gflops=flops / t / 1e9, p=1, reps=reps, runs=1)
        kind_s, lib, p = "port", "oracle/_build/libcsrc_oracle.so", 1
    best = max(methods, key=lambda m: methods[m]["gflops"])
    return dict(value=methods[best]["gflops"], best=best, methods=methods, kind=kind_s, lib=lib,
                cores=methods[best]["p"], host=hc,
                seq_gflops=methods.get("sequential", {}).get("gflops"))


def oracle_side_fixture(args):
    """The workload from the standalone fixture generator (oracle/_build/
    libcsrc_fixtures.so): the reference arm never maps the product library."""
    from oracle.oracle import config_fixture, working_set_bytes
    a, x = config_fixture(args.config)
    if args.dtype == "f32":  # the reference is fp64-only (common.hpp:20): fp32-rounded inputs
        for f in ("ad", "al", "au"):
            setattr(a, f, getattr(a, f).astype(np.float32).astype(np.float64))
        x = x.astype(np.float32).astype(np.float64)
    mb = working_set_bytes(a.n, a.nnz_stored(), a.value_symmetric, f32=args.dtype == "f32")
    return a, x, mb


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref, compiled from /root/reference) on this host's cores, same
    workload, metric and unit. Rank 0 only under torchrun."""
    if world > 1 and rank != 0:
        return 0
    from oracle.oracle import Ref, Oracle, host_cores
    a, x, mb = oracle_side_fixture(args)
    flops = 2 * a.nnz_full()
    hc = host_cores()
    p = max(1, hc["physical"])
    per_step = []
    suite = None
    if Ref.available():
        R = Ref(fast=True)  # the host's ISA-level build (timed baseline)
        # pick the reference's fastest method on this host (one product each), then time it
        probe = {}
        for name, kind, accum in REF_METHODS:
            h = R.exec_create(a, kind, accum, 1 if kind == 0 else p)
            try:
                R.exec_run(h, x, 1, a.n)
                dt, _, _ = R.exec_run(h, x, 1, a.n)
            finally:
                R.exec_destroy(h)
            probe[name] = dict(ms=dt * 1e3, gflops=flops / dt / 1e9)
        best = min(probe, key=lambda m: probe[m]["ms"])
        kind, accum = [(k, ac) for n, k, ac in REF_METHODS if n == best][0]
        p_best = 1 if kind == 0 else p
        h = R.exec_create(a, kind, accum, p_best)
        dt1, _, _ = R.exec_run(h, x, 1, a.n)
        reps = max(1, int(args.ref_seconds / max(args.steps, 1) / max(dt1, 1e-6)))
        for i in range(args.warmup + args.steps):
            dt, _, _ = R.exec_run(h, x, reps if i >= args.warmup else 1, a.n)
            if i >= args.warmup:
                per_step.append(dt / reps)
        R.exec_destroy(h)
        what = "sequential spmv_csrc" if kind == 0 else f"ParallelSpmv(local_buffers/{best}, p={p} physical cores)"
        res = dict(kind="reference", cores=p_best, lib=os.path.relpath(R.so, ROOT),
                   sample=f"each step = {reps} products of the full workload through the reference's {what}, "
                          f"the fastest of its sequential path and four accumulations on this host "
                          f"(one-product probe: methods); {os.path.relpath(R.so, ROOT)} compiled from "
                          f"/root/reference")
        suite = probe
    else:
        O = Oracle()
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            O.spmv_csrc(a, x)
            if i >= args.warmup:
                per_step.append(time.perf_counter() - t0)
        res = dict(kind="port", cores=1, lib="oracle/_build/libcsrc_oracle.so",
                   sample="each step = 1 product, plain-C oracle port of spmv_csrc (1 thread)")
    ms = 1e3 * statistics.median(per_step)
    value = flops / (ms / 1e3) / 1e9
    line = dict(
        metric=METRIC, value=value, unit="GFLOP/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
        ms_per_step=ms, higher_is_better=True, scaling=bench_scaling(args),
        vs_baseline=None, dtype=args.dtype, data="synthetic",
        config=workload_config_plain(args, a, mb, world), impl="reference",
        effective_gbs=mb / (ms / 1e3) / 1e9,
        cpu_baseline=dict(value=value, unit="GFLOP/s", cores=res["cores"], kind=res["kind"],
                          sample=res["sample"], host=hc, methods=suite, lib=res["lib"]),
        e2e=dict(value=value, unit="GFLOP/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
    )
    print(json.dumps(line), flush=True)
    return 0


CONFIG_DESC = {
    "c1": "2D Q1 256x256, 9-point, seed 42",
    "c2": "3D 64^3, 27-point, seed 7",
    "c3": "3D 160^3, 27-point, permuted (seed 11) + RCM",
    "c4": "elasticity 96^3 x 3 dof, 81-entry rows, seed 3",
    "c5": "3D 256^3, 27-point, seed 99",
}


def bench_scaling(args):
    # N > 1: the same matrix split into N row bands (total work fixed as N grows)
    return "strong"


def workload_config_plain(args, a, mb, world):
    return {"workload": f"{args.config}: {CONFIG_DESC[args.config]}, {args.dtype}", "n": a.n,
            "nnz": a.nnz_full(), "pairs": a.k_off(), "kind": args.kind,
            "parallelism": f"row bands x{world}" if world > 1 else "1 GPU",
            "l2": "working set > 126 MB L2 (no flush needed)" if mb > 400e6
            else f"L2 flushed between steps ({args.flush_mb} MB write)"}


def workload_config(args, a, world):
    import paper_1003_0952_b200 as P
    return workload_config_plain(args, a, P.model_bytes(a), world)


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


KERNEL_NAMES = {1: "k_gather_rows", 2: "k_gather_staged", 3: "k_gather_sell"}


def kernel_name(info, kind):
    if kind == "gather":
        return KERNEL_NAMES.get(int(info.gather_form), "k_gather")
    return {"windowed": "k_windowed", "atomic": "k_atomic", "colorful": "k_colored_ring",
            "local_buffers": "k_windowed (+ spill init / accumulate)"}[kind]


def time_plan(P, a, strat, xd, yd, steps, flush, warm=3, env=None):
    """Device-resident products of one plan: mean step / kernel ms (CUDA events on
    the plan's stream), the plan info."""
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        ex = P.GpuSpmv(a, strat)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for _ in range(warm):
        ex.apply_device(xd, yd)
    tot, ker = ex.time_products(xd, yd, steps, flush)
    info = ex.info()
    ex.close()
    return float(np.mean(tot)), float(np.mean(ker)), info


def run_single(args, P, torch, local):
    dtype = P.DType.f32 if args.dtype == "f32" else P.DType.f64
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    a, x, _ = P.config_matrix(args.config)
    mb = P.model_bytes(a, dtype)
    flops = 2 * a.nnz_full()
    strat = P.Strategy(P.StrategyKind[args.kind], P.AccumMethod.interval, p=8, dtype=dtype, device=local)
    flush = 0 if mb > 400e6 else args.flush_mb << 20
    peak, peak_src = load_peaks()

    ex = P.GpuSpmv(a, strat)
    xd = torch.from_numpy(x).to(device="cuda", dtype=tdt)
    yd = torch.zeros_like(xd)
    for _ in range(args.warmup):
        ex.apply_device(xd, yd)
    torch.cuda.synchronize()
    with ClockSampler(local) as cs:
        tot, ker = ex.time_products(xd, yd, args.steps, flush)
        torch.cuda.synchronize()
    clocks = cs.summary()
    ms, kms = float(np.mean(tot)), float(np.mean(ker))
    info = ex.info()
    layout_bytes, row_patterns = int(info.stream_bytes), int(info.row_patterns)
    kname = kernel_name(info, args.kind)
    # our kernels per product (driver memsets not counted)
    launches_per_step = {"gather": 1, "windowed": 1, "atomic": 1, "colorful": 1}.get(args.kind, 3)

    # end to end through the public host API (GpuSpmv.apply -> csrc_gpu_spmv): x in, y out every step
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    ex.apply(xh.numpy(), yh.numpy())
    e2e_steps = max(3, min(args.steps, 50))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ex.apply(xh.numpy(), yh.numpy())
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    # the reference API's own call shape: pageable std::vector-like numpy x and y (y reused, as
    # run_benchmark's apply(x, y) loop does, bench.hpp:225-255)
    xp = np.array(x)
    yp = np.empty_like(xp)
    ex.apply(xp, yp)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ex.apply(xp, yp)
    e2e_pageable_s = (time.perf_counter() - t0) / e2e_steps
    ex.close()

    # the other kernels on the same workload
    others = {}
    specs = {
        "gather_explicit": (P.Strategy(P.StrategyKind.gather, dtype=dtype, device=local), {"CSRC_GPU_GPATTERN": "0"}),
        "windowed": (P.Strategy(P.StrategyKind.windowed, dtype=dtype, device=local), None),
        "atomic": (P.Strategy(P.StrategyKind.atomic, dtype=dtype, device=local), None),
        "colorful": (P.Strategy(P.StrategyKind.colorful, p=8, dtype=dtype, device=local), None),
        "local_buffers": (P.Strategy(P.StrategyKind.local_buffers, P.AccumMethod.interval, p=8, dtype=dtype,
                                     device=local), None),
    }
    for name in [k for k in args.compare.split(",") if k and k != args.kind]:
        st, env = specs[name]
        oms, okms, oinf = time_plan(P, a, st, xd, yd, min(args.steps, 50), flush, env=env)
        others[name] = dict(ms_per_step=oms, gflops=flops / (oms / 1e3) / 1e9, kernel_ms=okms,
                            effective_gbs=mb / (okms / 1e3) / 1e9, frac_of_model_roofline=mb / (okms / 1e3) / 1e9 / peak,
                            stream_bytes=int(oinf.stream_bytes),
                            reads_csrc_as_stored=name in ("windowed", "atomic", "local_buffers"),
                            layout=("CSRC arrays as stored" if name in ("windowed", "atomic", "local_buffers") else
                                    "CSRC pairs class-major (colour classes), renumbered" if name == "colorful" else
                                    "per-row entry streams (CSR re-layout at plan time)"))
    wall = others.get("windowed")
    achieved = layout_bytes / (kms / 1e3) / 1e9
    roofline = dict(
        bound="hbm", achieved=achieved, peak=peak, unit="GB/s", frac=achieved / peak,
        traffic=load_traffic(f"{args.config}-{args.dtype}-{args.kind}"), peak_source=peak_src, kernel=kname,
        kernel_ms=kms, algorithmic_bytes_per_launch=layout_bytes,
        bytes_basis=("the bytes this plan's kernel streams per product (info.stream_bytes): "
                     + ("the CSRC pairs re-laid out at plan time as per-row entry streams with "
                        f"{'27 row patterns instead of column indices' if row_patterns else 'explicit columns'}"
                        if args.kind == "gather" else "the CSRC working-set model (working_set.hpp:11-23)")),
        csrc_model=dict(bytes=mb, effective_gbs=mb / (kms / 1e3) / 1e9,
                        note="reference working-set bytes (10 nnz + 18 n + 4) / kernel time; an effective "
                             "bandwidth, above the peak when the layout moves fewer bytes than the model"),
        row_patterns=row_patterns)
    if wall:
        roofline["csrc_as_stored"] = dict(
            kernel="k_windowed", kernel_ms=wall["kernel_ms"], bytes=mb,
            achieved=mb / (wall["kernel_ms"] / 1e3) / 1e9, frac=mb / (wall["kernel_ms"] / 1e3) / 1e9 / peak,
            note="the CSRC roofline: the kernel that streams ja/al/au/ad/ia as stored (TMA tiles, red.global "
                 "scatter), model bytes / its kernel time")
    line = dict(
        metric=METRIC, value=flops / (ms / 1e3) / 1e9, unit="GFLOP/s", n_gpus=1, steps=args.steps,
        warmup=args.warmup, ms_per_step=ms, higher_is_better=True, scaling=bench_scaling(args),
        vs_baseline=None, dtype=args.dtype, data="synthetic (BASELINE config, seeded fixture, DESIGN.md Fixtures)",
        config=workload_config(args, a, 1), effective_gbs=mb / (ms / 1e3) / 1e9,
        gflops_true=(flops - a.n) / (ms / 1e3) / 1e9, roofline=roofline,
        e2e=dict(value=flops / e2e_s / 1e9, unit="GFLOP/s", h2d_bytes_per_step=a.n * 8, d2h_bytes_per_step=a.n * 8,
                 wall_ms_per_step=e2e_s * 1e3, api="GpuSpmv.apply (csrc_gpu_spmv), pinned host x / y",
                 pageable=dict(value=flops / e2e_pageable_s / 1e9, wall_ms_per_step=e2e_pageable_s * 1e3,
                               api="GpuSpmv.apply with pageable numpy x / y (std::vector shape), y reused")),
        gpu_launches=launches_per_step * args.steps, clocks=clocks)
    if others:
        line["kernels"] = others
    if not args.no_cpu_baseline:
        a_c, x_c, _ = oracle_side_fixture(args)
        res = cpu_reference_suite(a_c, x_c, args.cpu_seconds)
        del a_c, x_c
        line["cpu_baseline"] = dict(
            value=res["value"], unit="GFLOP/s", cores=res["cores"], kind=res["kind"],
            sample=(f"the full workload, median of up to 3 runs of a bounded product count per method "
                    f"({args.cpu_seconds:.0f} s total); value = the fastest method ({res['best']}, "
                    f"p = {res['cores']} of {res['host']['physical']} physical cores / "
                    f"{res['host']['logical']} logical CPUs); {res['lib']}"),
            methods=res["methods"], sequential_gflops=res["seq_gflops"], host=res["host"])
    return line


def run_multi(args, P, torch, world, rank, local, share):
    """N > 1: the matrix in N partition_by_nnz row bands, one per rank; every timed
    step includes the exchange of the band form:
      gather   -- x-halo refresh (grouped NCCL send/recv of the rows other bands read,
                  overlapped with the interior rows), then the boundary rows;
      windowed -- boundary rows, y-halo partials shipped to their owners with grouped
                  NCCL send/recv while the interior rows run, then the halo reduce.
    The primary form is --kind (gather or windowed); the other is timed too ("forms")."""
    import torch.distributed as dist
    from paper_1003_0952_b200.dist import DistSpmv
    dtype = P.DType.f32 if args.dtype == "f32" else P.DType.f64
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    a, x, _ = P.config_matrix(args.config)
    mb = P.model_bytes(a, dtype)
    flops = 2 * a.nnz_full()
    coll_dev = "cpu" if share else "cuda"
    primary = "windowed" if args.kind == "windowed" else "gather"
    forms = {}
    clocks = None
    use_abi = args.exec == "abi" and not share  # NCCL refuses two ranks on one GPU
    for form in [primary] + [f for f in ("gather", "windowed") if f != primary]:
        abi_err = None
        if use_abi:
            # the C-ABI executor: band plan + exchange lists + NCCL communicator in the library
            from paper_1003_0952_b200.dist import NcclBandSpmv, gather_plan, halo_plan
            try:
                ds = NcclBandSpmv(a, P.Strategy(P.StrategyKind[form], dtype=dtype, device=local), form=form)
                p = gather_plan(a, world, rank) if form == "gather" else halo_plan(a, world, rank)
                L = ds.lists
                assert (L.x_lo, L.x_hi, L.y_lo) == (p.x_lo, p.x_hi, p.y_lo)
            except Exception as e:  # noqa: BLE001 -- reported in the JSON line, torch executor instead
                abi_err = str(e)
                ds = DistSpmv(a, P.Strategy(P.StrategyKind[form], dtype=dtype, device=local))
                p = ds.plan
        else:
            ds = DistSpmv(a, P.Strategy(P.StrategyKind[form], dtype=dtype, device=local))
            p = ds.plan
        xd = torch.from_numpy(x[p.x_lo:p.x_hi].copy()).to(device="cuda", dtype=tdt)
        yd = torch.zeros(p.row_end - p.y_lo, device="cuda", dtype=tdt)
        refresh = form == "gather"
        dist.barrier()
        for _ in range(args.warmup):
            ds.apply_device(xd, yd, refresh_x=refresh)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as cs:
            e0.record()
            for _ in range(args.steps):
                ds.apply_device(xd, yd, refresh_x=refresh)
            e1.record()
            torch.cuda.synchronize()
        dist.barrier()
        if clocks is None:
            clocks = cs.summary()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        # e2e: this rank's x slice in (pinned), its owned y rows out, every step
        xh = torch.from_numpy(x[p.x_lo:p.x_hi].copy()).pin_memory()
        yh = torch.empty(p.row_end - p.row_begin, dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        dist.barrier()
        e2e_steps = max(3, min(args.steps, 50))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            xd.copy_(xh.to(tdt), non_blocking=True)
            ds.apply_device(xd, yd, refresh_x=refresh)
            yh.copy_(yd[p.row_begin - p.y_lo:].to(torch.float64), non_blocking=True)
            torch.cuda.synchronize()
        te = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device=coll_dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        hb = torch.tensor([(p.x_hi - p.x_lo) * 8, (p.row_end - p.row_begin) * 8], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(hb)
        halo = (sum(q1 - q0 for _, q0, q1 in p.x_sends) + sum(q1 - q0 for _, q0, q1 in p.x_recvs) if refresh else
                sum(q1 - q0 for _, q0, q1 in p.sends) + sum(q1 - q0 for _, q0, q1 in p.recvs))
        forms[form] = dict(executor="C-ABI csrc_gpu_band_exec (NCCL in the library)" if use_abi and not abi_err
                           else "paper_1003_0952_b200.dist.DistSpmv (torch.distributed)", abi_error=abi_err,
                           ms_per_step=ms, gflops=flops / (ms / 1e3) / 1e9, effective_gbs=mb / (ms / 1e3) / 1e9,
                           e2e_ms=float(te.item()) * 1e3, e2e_gflops=flops / float(te.item()) / 1e9,
                           h2d_bytes_per_step=int(hb[0].item()), d2h_bytes_per_step=int(hb[1].item()),
                           exchange=("x halo (grouped NCCL send/recv), interior rows overlapped" if refresh else
                                     "y halo partials to their owners (grouped NCCL send/recv), interior "
                                     "rows overlapped, then the red.global halo reduce"),
                           rank0_halo_elems=int(halo))
        ds.close()
        del xd, yd
    f0 = forms[primary]
    peak, peak_src = load_peaks()
    return dict(
        metric=METRIC, value=f0["gflops"], unit="GFLOP/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
        ms_per_step=f0["ms_per_step"], higher_is_better=True, scaling=bench_scaling(args), vs_baseline=None,
        dtype=args.dtype, data="synthetic (BASELINE config, seeded fixture, DESIGN.md Fixtures)",
        config=workload_config(args, a, world), effective_gbs=f0["effective_gbs"],
        roofline=dict(bound="hbm", achieved=f0["effective_gbs"] / world, peak=peak, unit="GB/s",
                      frac=f0["effective_gbs"] / world / peak, traffic=None, peak_source=peak_src,
                      kernel="k_gather_staged" if primary == "gather" else "k_windowed",
                      note="per-GPU share of the CSRC model bytes / the max-over-ranks step (exchange included)"),
        e2e=dict(value=f0["e2e_gflops"], unit="GFLOP/s", h2d_bytes_per_step=f0["h2d_bytes_per_step"],
                 d2h_bytes_per_step=f0["d2h_bytes_per_step"], wall_ms_per_step=f0["e2e_ms"]),
        gpu_launches=(4 if primary == "gather" else 4) * args.steps, forms=forms, clocks=clocks,
        shared_gpu=share or None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--kind", default="gather", choices=["gather", "windowed", "atomic", "colorful", "local_buffers"])
    ap.add_argument("--compare", default="gather_explicit,windowed,atomic,colorful,local_buffers",
                    help="other kernels timed on the same workload (reported under 'kernels'); '' = none")
    ap.add_argument("--flush-mb", type=int, default=256)
    ap.add_argument("--ref-seconds", type=float, default=20.0, help="CPU-reference sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="cpu_baseline sample budget")
    ap.add_argument("--exec", default="abi", choices=["abi", "torch"],
                    help="N > 1: the C-ABI band executor (NCCL owned by the library) or the torch.distributed one")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N launches its own N ranks (torchrun on 127.0.0.1), one per GPU
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if world != args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N ranks "
                                                     f"for --gpus N (or omit WORLD_SIZE to self-launch)"}), flush=True)
        return 2
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)

    import torch
    import paper_1003_0952_b200 as P

    # CSRC_BENCH_SHARE_GPU=1: a functional check of the N > 1 path on a box with fewer GPUs than ranks
    # (ranks share the visible GPUs; collectives over gloo). Its numbers are not measurements.
    share = os.environ.get("CSRC_BENCH_SHARE_GPU") == "1"
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world == 1:
        line = run_single(args, P, torch, local)
    else:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        line = run_multi(args, P, torch, world, rank, local, share)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
