#!/bin/bash
mkdir -p gpurun_out
V='dflt:;u8r2:CSRC_GPU_CW_U=8;u8r4:CSRC_GPU_CW_U=8,CSRC_GPU_CW_R=4;u14r4:CSRC_GPU_CW_R=4;u4r4:CSRC_GPU_CW_U=4,CSRC_GPU_CW_R=4;old:CSRC_GPU_CW_RING=0'
REPS=50 timeout 900 python tools/probe_r2.py c3,c4 colorful "$V" > gpurun_out/r2s5_c34_colored.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s5_c34_colored.txt
