#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/r2_bench_single.json 2> gpurun_out/r2_bench_single.err; echo "bench rc=$?"; cat gpurun_out/r2_bench_single.json; tail -3 gpurun_out/r2_bench_single.err
CSRC_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config c4 --steps 10 --warmup 2 > gpurun_out/r2_bench_share2.json 2> gpurun_out/r2_bench_share2.err; echo "share2 rc=$?"; cat gpurun_out/r2_bench_share2.json; tail -5 gpurun_out/r2_bench_share2.err
CSRC_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config c4 --kind windowed --steps 10 --warmup 2 > gpurun_out/r2_bench_share2w.json 2> gpurun_out/r2_bench_share2w.err; echo "share2w rc=$?"; cat gpurun_out/r2_bench_share2w.json; tail -5 gpurun_out/r2_bench_share2w.err
