#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 python bench.py --kind windowed --no-cpu-baseline --compare atomic,local_buffers > gpurun_out/bench_win.json 2>> gpurun_out/bench.err; echo "bench win rc=$?"; cat gpurun_out/bench_win.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_windowed -c 1 -o gpurun_out/ncu_win_c5 python tools/prof_one.py c5 windowed 3 > gpurun_out/ncu_win.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_win.log
