#!/bin/bash
mkdir -p gpurun_out
V='dflt:;b50:CSRC_GPU_CR_BACKOFF=50;b200:CSRC_GPU_CR_BACKOFF=200;b500:CSRC_GPU_CR_BACKOFF=500;lr2b200:CSRC_GPU_CR_LANES=2,CSRC_GPU_CR_BACKOFF=200;u8b200:CSRC_GPU_CW_U=8,CSRC_GPU_CR_BACKOFF=200'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s5_backoff.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s5_backoff.txt
