#!/bin/bash
mkdir -p gpurun_out
V='r4d8:;r4d6:CSRC_GPU_CW_D=6;r4d12:CSRC_GPU_CW_D=12;r4d16:CSRC_GPU_CW_D=16;r2d4:CSRC_GPU_CW_R=2;r2d6:CSRC_GPU_CW_R=2,CSRC_GPU_CW_D=6;r8d16:CSRC_GPU_CW_R=8;r8d24:CSRC_GPU_CW_R=8,CSRC_GPU_CW_D=24;r1d3:CSRC_GPU_CW_R=1,CSRC_GPU_CW_D=3;r4d8u4:CSRC_GPU_CW_U=4;r4d8nt256:CSRC_GPU_CW_NT=256'
REPS=20 timeout 1500 python tools/probe_r2.py c5,c3 colorful "$V" > gpurun_out/r2p3_colored.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p3_colored.txt
REPS=20 timeout 600 python tools/probe_r2.py c4,c2 colorful 'r4d8:;r4d16:CSRC_GPU_CW_D=16;r8d16:CSRC_GPU_CW_R=8' >> gpurun_out/r2p3_colored.txt 2>&1; tail -8 gpurun_out/r2p3_colored.txt
