#!/bin/bash
# last sanity pass over the final build: the whole GPU suite and smoke
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -x > gpurun_out/r2s8_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2s8_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s8_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2s8_smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/r2s8_bench.json 2> gpurun_out/r2s8_bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r2s8_bench.json
