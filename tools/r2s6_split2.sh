#!/bin/bash
mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colored_kernel_shapes and SPLIT" > gpurun_out/r2s6_split_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s6_split_tests.txt
[ $rc -ne 0 ] && exit 1
V='dflt:;sp14:CSRC_GPU_CR_SPLIT=1;sp8:CSRC_GPU_CR_SPLIT=1,CSRC_GPU_CW_U=8;sp14s300:CSRC_GPU_CR_SPLIT=1,CSRC_GPU_CR_SLACK_PCT=300;sp14s600:CSRC_GPU_CR_SPLIT=1,CSRC_GPU_CR_SLACK_PCT=600'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s6_split2.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s6_split2.txt
