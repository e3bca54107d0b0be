#!/bin/bash
# full GPU parity suite + smoke + benches (c5 f64/f32 headline, c4 sliced form) + ncu of the sliced kernel on c4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2>> gpurun_out/bench.err; echo "bench c4 rc=$?"; cat gpurun_out/bench_c4.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_sell -c 1 -o gpurun_out/ncu_sell_c4 python tools/prof_one.py c4 gather 3 > gpurun_out/ncu_sell.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_sell.log
