#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colored_kernel_shapes or edge or known" > gpurun_out/r2s7_r160_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s7_r160_tests.txt
[ $rc -ne 0 ] && exit 1
V='r160:;r160s300:CSRC_GPU_CR_SLACK_PCT=300;r160s500:CSRC_GPU_CR_SLACK_PCT=500'
REPS=50 timeout 900 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s7_r160.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s7_r160.txt
V='r160:'
REPS=50 timeout 900 python tools/probe_r2.py c4,c3,c2 colorful "$V" >> gpurun_out/r2s7_r160.txt 2>&1; echo "rc=$?"; tail -7 gpurun_out/r2s7_r160.txt
DT=f32 REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" >> gpurun_out/r2s7_r160.txt 2>&1; tail -2 gpurun_out/r2s7_r160.txt
