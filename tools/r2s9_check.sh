#!/bin/bash
# round 2 (session 3) GPU check of the restored tree: whole GPU suite, smoke, both bench arms, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1700 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2s9_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r2s9_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s9_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2s9_smoke.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2s9_bench_ref.json 2> gpurun_out/r2s9_bench_ref.err; echo "ref rc=$?"; cat gpurun_out/r2s9_bench_ref.json
timeout 900 python bench.py > gpurun_out/r2s9_bench.json 2> gpurun_out/r2s9_bench.err; echo "bench rc=$?"; cat gpurun_out/r2s9_bench.json; tail -3 gpurun_out/r2s9_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2s9_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2s9_ncu_bench.log 2>&1; echo "ncu rc=$?"
