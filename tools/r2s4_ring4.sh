#!/bin/bash
mkdir -p gpurun_out
timeout 420 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colorful or color" > gpurun_out/r2s4_ring_tests4.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s4_ring_tests4.txt
[ $rc -ne 0 ] && exit 1
V='ring:;s100:CSRC_GPU_CR_SLACK_PCT=100;s150:CSRC_GPU_CR_SLACK_PCT=150;s300:CSRC_GPU_CR_SLACK_PCT=300;u14:CSRC_GPU_CW_U=14;u4:CSRC_GPU_CW_U=4;st13x3:CSRC_GPU_CR_STAGES=3;st7x2:CSRC_GPU_CR_STAGES=2,CSRC_GPU_CR_STAGE_BYTES=17920;st7x3:CSRC_GPU_CR_STAGES=3,CSRC_GPU_CR_STAGE_BYTES=17920;st7x4:CSRC_GPU_CR_STAGES=4,CSRC_GPU_CR_STAGE_BYTES=17920;st9x3:CSRC_GPU_CR_STAGES=3,CSRC_GPU_CR_STAGE_BYTES=23040;hint:CSRC_GPU_CR_HINT=1;r2:CSRC_GPU_CW_R=2'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s4_ring_sweep4.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2s4_ring_sweep4.txt
