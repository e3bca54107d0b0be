#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colored_kernel_shapes" > gpurun_out/r2s6_coldef_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s6_coldef_tests.txt
[ $rc -ne 0 ] && exit 1
V='base:;mb512:CSRC_GPU_CW_MINB=512;s800:CSRC_GPU_CR_SLACK_PCT=800;mb512s800:CSRC_GPU_CW_MINB=512,CSRC_GPU_CR_SLACK_PCT=800;mb256s800:CSRC_GPU_CW_MINB=256,CSRC_GPU_CR_SLACK_PCT=800;s1200:CSRC_GPU_CR_SLACK_PCT=1200'
REPS=50 timeout 1200 python tools/probe_r2.py c4,c3,c2 colorful "$V" > gpurun_out/r2s6_coldef2.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s6_coldef2.txt
