#!/bin/bash
mkdir -p gpurun_out
timeout 420 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colorful or color" > gpurun_out/r2s4_ring_tests3.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s4_ring_tests3.txt
[ $rc -ne 0 ] && exit 1
V='ring:;old:CSRC_GPU_CW_RING=0;hint:CSRC_GPU_CR_HINT=1;s100:CSRC_GPU_CR_SLACK_PCT=100;s50:CSRC_GPU_CR_SLACK_PCT=50;s300:CSRC_GPU_CR_SLACK_PCT=300;u8:CSRC_GPU_CW_U=8;u16:CSRC_GPU_CW_U=16;st13x3:CSRC_GPU_CR_STAGES=3;st7x2u8:CSRC_GPU_CR_STAGES=2,CSRC_GPU_CR_STAGE_BYTES=17920,CSRC_GPU_CW_U=8;st7x3u8:CSRC_GPU_CR_STAGES=3,CSRC_GPU_CR_STAGE_BYTES=17920,CSRC_GPU_CW_U=8;r2:CSRC_GPU_CW_R=2;r8:CSRC_GPU_CW_R=8'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s4_ring_sweep3.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2s4_ring_sweep3.txt
REPS=50 timeout 200 python tools/probe_r2.py c2 colorful "$V" >> gpurun_out/r2s4_ring_sweep3.txt 2>&1; echo "probe rc=$?"; tail -14 gpurun_out/r2s4_ring_sweep3.txt
