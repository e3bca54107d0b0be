#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colored_kernel_shapes" > gpurun_out/r2s5_claim_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s5_claim_tests.txt
[ $rc -ne 0 ] && exit 1
V='c0s400:CSRC_GPU_CR_SLACK_PCT=400;c1s200:CSRC_GPU_CR_CLAIM=1;c1s300:CSRC_GPU_CR_CLAIM=1,CSRC_GPU_CR_SLACK_PCT=300;c1s400:CSRC_GPU_CR_CLAIM=1,CSRC_GPU_CR_SLACK_PCT=400;c2s200:CSRC_GPU_CR_CLAIM=2;c2s300:CSRC_GPU_CR_CLAIM=2,CSRC_GPU_CR_SLACK_PCT=300;c2s3s200:CSRC_GPU_CR_CLAIM=2,CSRC_GPU_CR_STAGES=3;c2s3s300:CSRC_GPU_CR_CLAIM=2,CSRC_GPU_CR_STAGES=3,CSRC_GPU_CR_SLACK_PCT=300;c1s3s300:CSRC_GPU_CR_CLAIM=1,CSRC_GPU_CR_STAGES=3,CSRC_GPU_CR_SLACK_PCT=300;c1r4s300:CSRC_GPU_CR_CLAIM=1,CSRC_GPU_CW_R=4,CSRC_GPU_CR_SLACK_PCT=300'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s5_claim.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s5_claim.txt
