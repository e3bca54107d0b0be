#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colored_kernel_shapes" > gpurun_out/r2s4_ring_tests7.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s4_ring_tests7.txt
[ $rc -ne 0 ] && exit 1
V='u14r2:CSRC_GPU_CW_U=14,CSRC_GPU_CW_R=2;pf3:CSRC_GPU_CW_U=14,CSRC_GPU_CW_R=2,CSRC_GPU_CR_PF=1,CSRC_GPU_CR_STAGES=3;pf2:CSRC_GPU_CW_U=14,CSRC_GPU_CW_R=2,CSRC_GPU_CR_PF=1;s3:CSRC_GPU_CW_U=14,CSRC_GPU_CW_R=2,CSRC_GPU_CR_STAGES=3;pf3u8:CSRC_GPU_CW_R=2,CSRC_GPU_CR_PF=1,CSRC_GPU_CR_STAGES=3;pf2u8:CSRC_GPU_CW_R=2,CSRC_GPU_CR_PF=1;u8r2:CSRC_GPU_CW_R=2;pf3s150:CSRC_GPU_CW_U=14,CSRC_GPU_CW_R=2,CSRC_GPU_CR_PF=1,CSRC_GPU_CR_STAGES=3,CSRC_GPU_CR_SLACK_PCT=150;pf3s300:CSRC_GPU_CW_U=14,CSRC_GPU_CW_R=2,CSRC_GPU_CR_PF=1,CSRC_GPU_CR_STAGES=3,CSRC_GPU_CR_SLACK_PCT=300'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s4_ring_sweep7.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2s4_ring_sweep7.txt
