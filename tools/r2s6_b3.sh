#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colored_kernel_shapes" > gpurun_out/r2s6_b3_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s6_b3_tests.txt
[ $rc -ne 0 ] && exit 1
V='b3:;b3c2:CSRC_GPU_CW_CTAS=2;b3s300:CSRC_GPU_CR_SLACK_PCT=300;b3s500:CSRC_GPU_CR_SLACK_PCT=500;b3s600:CSRC_GPU_CR_SLACK_PCT=600;u8:CSRC_GPU_CW_U=8'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s6_b3.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s6_b3.txt
