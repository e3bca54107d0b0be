#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colorful or color" > gpurun_out/r2s4_ring_tests2.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2s4_ring_tests2.txt
V='ring:;old:CSRC_GPU_CW_RING=0;hint:CSRC_GPU_CR_HINT=1;s100:CSRC_GPU_CR_SLACK_PCT=100;s300:CSRC_GPU_CR_SLACK_PCT=300;st13x2:CSRC_GPU_CR_STAGES=2;st7x3:CSRC_GPU_CR_STAGES=3,CSRC_GPU_CR_STAGE_BYTES=17920;st7x2:CSRC_GPU_CR_STAGES=2,CSRC_GPU_CR_STAGE_BYTES=17920;st7x2s100:CSRC_GPU_CR_STAGES=2,CSRC_GPU_CR_STAGE_BYTES=17920,CSRC_GPU_CR_SLACK_PCT=100;u16:CSRC_GPU_CW_U=16;r2:CSRC_GPU_CW_R=2'
REPS=50 timeout 1500 python tools/probe_r2.py c5,c2 colorful "$V" > gpurun_out/r2s4_ring_sweep2.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2s4_ring_sweep2.txt
