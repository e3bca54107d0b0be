#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assemble.py tests/test_gpu_rect.py tests/test_cli.py tests/test_dropin_cpp.py -m gpu -q > gpurun_out/pytest_asm.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_asm.log
timeout 900 python tools/assemble_bench.py --configs c1,c2,c3,c4,c5 --ref-configs c1,c2,c3 > gpurun_out/assemble.jsonl 2> gpurun_out/assemble.err; echo "asm rc=$?"; cat gpurun_out/assemble.jsonl; tail -3 gpurun_out/assemble.err
ALLBIG=1 NOF32=1 timeout 1500 python tools/gpu_probe.py c2,c3,c4,c5 > gpurun_out/probe_all.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/probe_all.txt
