#!/bin/bash
# round 2 GPU check: the new ADVICE tests, then the whole suite, smoke, bench (both arms)
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "smaller_plan or mixing_plan or shapes_fp32" > gpurun_out/r2_pytest_new.log 2>&1; echo "new rc=$?"; tail -3 gpurun_out/r2_pytest_new.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc=$?"; cat gpurun_out/r2_bench_ref.json
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"; cat gpurun_out/r2_bench.json
