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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--kind", default="gather", choices=["gather", "windowed", "atomic", "colorful", "local_buffers"])
    ap.add_argument("--compare", default="gather_explicit,windowed,atomic",
                    help="other kernels timed on the same workload (reported under 'kernels'); '' = none")
    ap.add_argument("--flush-mb", type=int, default=256)
    ap.add_argument("--ref-seconds", type=float, default=20.0, help="CPU-reference sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="cpu_baseline sample budget")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)

    import torch
    import paper_1003_0952_b200 as P

    # CSRC_BENCH_SHARE_GPU=1 (functional check of the N>1 code path on a one-GPU box, gather bands only:
    # their kernels never wait on each other): ranks share the visible GPUs and the timing collectives
    # run over gloo. Its numbers are not measurements.
    share = os.environ.get("CSRC_BENCH_SHARE_GPU") == "1"
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    coll_dev = "cpu" if share else "cuda"
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dtype = P.DType.f32 if args.dtype == "f32" else P.DType.f64
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    a, x, _ = P.config_matrix(args.config)
    mb = P.model_bytes(a, dtype)
    flops = 2 * a.nnz_full()
    kind = P.StrategyKind[args.kind]
    strat = P.Strategy(kind, P.AccumMethod.interval, p=8, dtype=dtype, device=local)
    flush = 0 if mb > 400e6 else args.flush_mb << 20

    if world == 1:
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
        ms = float(np.mean(tot))
        kms = float(np.mean(ker))
        info = ex.info()
        layout_bytes, row_patterns = int(info.stream_bytes), int(info.row_patterns)
        kernel_name = {1: "k_gather_rows", 2: "k_gather_staged", 3: "k_gather_sell"}.get(
            int(info.gather_form), {"windowed": "k_windowed", "atomic": "k_atomic"}.get(args.kind, args.kind))
        # our kernels per product (the y memset of windowed/atomic is a driver memset, not counted)
        launches_per_step = 1 if args.kind in ("gather", "windowed", "atomic") else info.launches_per_apply
        others = {}
        for name in [k for k in args.compare.split(",") if k and k != args.kind]:
            # gather_explicit: the gather kernel with explicit column indices (row-pattern form off)
            env_off = name == "gather_explicit"
            if env_off:
                os.environ["CSRC_GPU_GPATTERN"] = "0"
            ox = P.GpuSpmv(a, P.Strategy(P.StrategyKind["gather" if env_off else name], P.AccumMethod.interval,
                                          p=8, dtype=dtype, device=local))
            if env_off:
                del os.environ["CSRC_GPU_GPATTERN"]
            for _ in range(3):
                ox.apply_device(xd, yd)
            otot, oker = ox.time_products(xd, yd, min(args.steps, 50), flush)
            ox.close()
            oms = float(np.mean(otot))
            okms = float(np.mean(oker))
            peak_o, _ = load_peaks()
            others[name] = dict(ms_per_step=oms, gflops=flops / (oms / 1e3) / 1e9,
                                effective_gbs=mb / (oms / 1e3) / 1e9, kernel_ms=okms,
                                roofline_achieved_gbs=mb / (okms / 1e3) / 1e9,
                                roofline_frac=mb / (okms / 1e3) / 1e9 / peak_o,
                                reads_csrc_as_stored=name in ("windowed", "atomic"))
        # end to end through the public host API: pinned x -> device, product, y -> pinned host
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        ex.apply(xh.numpy(), yh.numpy())
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ex.apply(xh.numpy(), yh.numpy())
        e2e_s = (time.perf_counter() - t0) / args.steps
        ex.close()
        ms_max = ms
    else:
        others = {}
        layout_bytes, row_patterns = None, 0
        kernel_name = "k_gather_staged" if args.kind == "gather" else "k_" + args.kind
        from paper_1003_0952_b200.dist import DistSpmv
        ds = DistSpmv(a, strat)
        p = ds.plan
        xd = torch.from_numpy(x[p.x_lo:p.x_hi].copy()).to(device="cuda", dtype=tdt)
        yd = torch.zeros(p.row_end - p.y_lo, device="cuda", dtype=tdt)
        dist.barrier()
        for _ in range(args.warmup):
            ds.apply_device(xd, yd)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as cs:
            e0.record()
            for _ in range(args.steps):
                ds.apply_device(xd, yd)
            e1.record()
            torch.cuda.synchronize()
        dist.barrier()
        clocks = cs.summary()
        ms = e0.elapsed_time(e1) / args.steps
        t = torch.tensor([ms], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
        kms = ms
        launches_per_step = 1 if p.mode == "gather" else 3 + len(p.recvs)
        # e2e: host slice in, owned rows out
        xh = torch.from_numpy(x[p.x_lo:p.x_hi].copy()).pin_memory()
        yh = torch.empty(p.row_end - p.row_begin, dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            xd.copy_(xh.to(tdt), non_blocking=True)
            ds.apply_device(xd, yd)
            yh.copy_(yd[p.row_begin - p.y_lo:].to(torch.float64), non_blocking=True)
            torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / args.steps
        te = torch.tensor([e2e_s], device=coll_dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        ds.close()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0
    peak, peak_src = load_peaks()
    gbs = mb / (ms_max / 1e3) / 1e9
    achieved = mb / (kms / 1e3) / 1e9
    elem = 4 if args.dtype == "f32" else 8
    wl = f"{args.config}-{args.dtype}-{args.kind}"
    line = dict(
        metric=METRIC, value=flops / (ms_max / 1e3) / 1e9, unit="GFLOP/s", n_gpus=world, steps=args.steps,
        warmup=args.warmup, ms_per_step=ms_max, higher_is_better=True,
        scaling="strong", vs_baseline=None, dtype=args.dtype,
        data="synthetic (BASELINE config, seeded fixture, DESIGN.md Fixtures)",
        config=workload_config(args, a, world),
        effective_gbs=gbs, roofline_frac_of_measured_hbm=gbs / peak,
        gflops_true=(flops - a.n) / (ms_max / 1e3) / 1e9,
        roofline=dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s", frac=achieved / peak,
                      traffic=load_traffic(wl) if world == 1 else None, peak_source=peak_src,
                      kernel=kernel_name,
                      algorithmic_bytes_per_launch=mb, kernel_ms=kms,
                      layout_bytes_per_launch=layout_bytes,
                      layout_frac=(layout_bytes / (kms / 1e3) / 1e9) / peak if layout_bytes else None,
                      row_patterns=row_patterns),
        e2e=dict(value=flops / e2e_s / 1e9, unit="GFLOP/s", h2d_bytes_per_step=a.n * 8 if world == 1
                 else (p.x_hi - p.x_lo) * 8, d2h_bytes_per_step=a.n * 8 if world == 1
                 else (p.row_end - p.row_begin) * 8, wall_ms_per_step=e2e_s * 1e3),
        gpu_launches=launches_per_step * args.steps,
        clocks=clocks,
    )
    if others:
        line["kernels"] = others
    if world == 1 and not args.no_cpu_baseline:
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
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
