#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 python bench.py --dtype f32 --no-cpu-baseline --compare "" > gpurun_out/bench_f32.json 2>> gpurun_out/bench.err; echo "bench32 rc=$?"; cat gpurun_out/bench_f32.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_staged -c 1 -o gpurun_out/ncu_gather_c5 python tools/prof_one.py c5 gather 3 > gpurun_out/ncu_gather.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_gather.log
