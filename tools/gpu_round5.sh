#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
KINDS=gather,windowed NOF32=1 timeout 600 python tools/gpu_probe.py c3,c4,c5 > gpurun_out/probe_plan.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/probe_plan.txt
