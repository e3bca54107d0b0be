#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rect.py tests/test_gpu_dropin.py -x -q -m gpu -k "colorful or color or edge or known or rect or accessors or large_configs or c5_fp32" > gpurun_out/r2s8_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s8_tests.txt
V='final:'
REPS=50 timeout 900 python tools/probe_r2.py c5,c4,c3,c2,c1 colorful "$V" > gpurun_out/r2s8_final_colored.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s8_final_colored.txt
DT=f32 REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" >> gpurun_out/r2s8_final_colored.txt 2>&1; tail -2 gpurun_out/r2s8_final_colored.txt
