#!/bin/bash
mkdir -p gpurun_out
timeout 420 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colorful or color" > gpurun_out/r2s4_ring_tests6.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s4_ring_tests6.txt
[ $rc -ne 0 ] && exit 1
V='u8:;u14:CSRC_GPU_CW_U=14;u8h:CSRC_GPU_CR_HINT=1;u14h:CSRC_GPU_CW_U=14,CSRC_GPU_CR_HINT=1;u14s150:CSRC_GPU_CW_U=14,CSRC_GPU_CR_SLACK_PCT=150;u14s300:CSRC_GPU_CW_U=14,CSRC_GPU_CR_SLACK_PCT=300;u14s3:CSRC_GPU_CW_U=14,CSRC_GPU_CR_STAGES=3;u14r2h:CSRC_GPU_CW_U=14,CSRC_GPU_CW_R=2,CSRC_GPU_CR_HINT=1'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s4_ring_sweep6.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2s4_ring_sweep6.txt
