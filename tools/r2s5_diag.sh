#!/bin/bash
mkdir -p gpurun_out
V='dflt:;nodep:CSRC_GPU_CR_DIAG_NODEP=1;nodeps100:CSRC_GPU_CR_DIAG_NODEP=1,CSRC_GPU_CR_SLACK_PCT=100;nodeps3:CSRC_GPU_CR_DIAG_NODEP=1,CSRC_GPU_CR_STAGES=3;nodepu8:CSRC_GPU_CR_DIAG_NODEP=1,CSRC_GPU_CW_U=8'
REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s5_diag.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s5_diag.txt
