#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/r2s7_bench_f32.json 2> gpurun_out/r2s7_bench_f32.err; echo "f32 rc=$?"; tail -c 600 gpurun_out/r2s7_bench_f32.json
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2s7_bench_c4.json 2> gpurun_out/r2s7_bench_c4.err; echo "c4 rc=$?"; tail -c 600 gpurun_out/r2s7_bench_c4.json
timeout 900 python bench.py --kind colorful --no-cpu-baseline --compare "" > gpurun_out/r2s7_bench_colorful.json 2> gpurun_out/r2s7_bench_colorful.err; echo "col rc=$?"; tail -c 900 gpurun_out/r2s7_bench_colorful.json
timeout 900 python bench.py --kind windowed --no-cpu-baseline --compare "" > gpurun_out/r2s7_bench_windowed.json 2> gpurun_out/r2s7_bench_windowed.err; echo "win rc=$?"; tail -c 900 gpurun_out/r2s7_bench_windowed.json
