mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assemble.py tests/test_gpu_rect.py -x -q > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_new.log
timeout 900 python tools/assemble_bench.py --configs c1,c2,c3,c5 --ref-configs c1,c2,c3 > gpurun_out/assemble.jsonl 2> gpurun_out/assemble.err; echo "asm rc=$?"; cat gpurun_out/assemble.jsonl; tail -5 gpurun_out/assemble.err
