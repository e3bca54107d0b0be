#!/bin/bash
# ring form of the colored wavefront: parity first (bounded), then a first sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colorful or color or family or mesh or known" > gpurun_out/r2s4_ring_tests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2s4_ring_tests.txt
V='ring:;old:CSRC_GPU_CW_RING=0;hint:CSRC_GPU_CR_HINT=1;s100:CSRC_GPU_CR_SLACK_PCT=100;s300:CSRC_GPU_CR_SLACK_PCT=300;st4:CSRC_GPU_CR_STAGES=4,CSRC_GPU_CR_STAGE_BYTES=25600;u16:CSRC_GPU_CW_U=16;r2:CSRC_GPU_CW_R=2;r8:CSRC_GPU_CW_R=8'
REPS=50 timeout 1500 python tools/probe_r2.py c2,c5 colorful "$V" > gpurun_out/r2s4_ring_sweep1.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2s4_ring_sweep1.txt
