#!/bin/bash
mkdir -p gpurun_out
V='dflt:;lr2:CSRC_GPU_CR_LANES=2;lr2big:CSRC_GPU_CR_LANES=2,CSRC_GPU_CR_STAGE_BYTES=33280;st66:CSRC_GPU_CR_STAGE_BYTES=53760;st20x3:CSRC_GPU_CR_STAGE_BYTES=51200,CSRC_GPU_CR_STAGES=2;u16:CSRC_GPU_CW_U=16;s600:CSRC_GPU_CR_SLACK_PCT=600;r4:CSRC_GPU_CW_R=4;r1:CSRC_GPU_CW_R=1'
REPS=50 timeout 900 python tools/probe_r2.py c4 colorful "$V" > gpurun_out/r2s6_c4col.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s6_c4col.txt
V='dflt:;s600:CSRC_GPU_CR_SLACK_PCT=600;s800:CSRC_GPU_CR_SLACK_PCT=800;r4:CSRC_GPU_CW_R=4;r1:CSRC_GPU_CW_R=1;u16:CSRC_GPU_CW_U=16;lr2:CSRC_GPU_CR_LANES=2'
REPS=50 timeout 600 python tools/probe_r2.py c3 colorful "$V" >> gpurun_out/r2s6_c4col.txt 2>&1; echo "rc=$?"; tail -9 gpurun_out/r2s6_c4col.txt
