#!/bin/bash
mkdir -p gpurun_out
V='d16:;pf0:CSRC_GPU_CW_PF=0;pf2:CSRC_GPU_CW_PF=2;keep:CSRC_GPU_CW_KEEP=1;keeppf2:CSRC_GPU_CW_KEEP=1,CSRC_GPU_CW_PF=2;keepd8:CSRC_GPU_CW_KEEP=1,CSRC_GPU_CW_D=8;keepd12:CSRC_GPU_CW_KEEP=1,CSRC_GPU_CW_D=12,CSRC_GPU_CW_PF=2;keepd24:CSRC_GPU_CW_KEEP=1,CSRC_GPU_CW_D=24,CSRC_GPU_CW_PF=2'
REPS=20 timeout 1500 python tools/probe_r2.py c5,c3,c4 colorful "$V" > gpurun_out/r2p5_colored.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p5_colored.txt
