#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colored_kernel_shapes" > gpurun_out/r2s5_lr2_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s5_lr2_tests.txt
[ $rc -ne 0 ] && exit 1
V='dflt:;lr2:CSRC_GPU_CR_LANES=2;lr2s300:CSRC_GPU_CR_LANES=2,CSRC_GPU_CR_SLACK_PCT=300;lr2s600:CSRC_GPU_CR_LANES=2,CSRC_GPU_CR_SLACK_PCT=600;lr2st3:CSRC_GPU_CR_LANES=2,CSRC_GPU_CR_STAGES=3;lr2c3:CSRC_GPU_CR_LANES=2,CSRC_GPU_CW_CTAS=3;lr2r4:CSRC_GPU_CR_LANES=2,CSRC_GPU_CW_R=4'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s5_lr2.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s5_lr2.txt
