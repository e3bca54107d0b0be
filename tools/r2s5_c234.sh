#!/bin/bash
mkdir -p gpurun_out
V='dflt:;s200:CSRC_GPU_CR_SLACK_PCT=200'
REPS=50 timeout 900 python tools/probe_r2.py c2,c4,c3 colorful "$V" > gpurun_out/r2s5_c234.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s5_c234.txt
