#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --kind windowed --no-cpu-baseline --compare atomic,local_buffers > gpurun_out/bench_win.json 2> gpurun_out/bench.err; echo "bench win rc=$?"; cat gpurun_out/bench_win.json
timeout 600 python bench.py --kind windowed --dtype f32 --no-cpu-baseline --compare "" > gpurun_out/bench_win32.json 2>> gpurun_out/bench.err; echo "bench win32 rc=$?"; cat gpurun_out/bench_win32.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_windowed -c 1 -o gpurun_out/ncu_win_c5 python tools/prof_one.py c5 windowed 3 > gpurun_out/ncu_win.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_win.log
