#!/bin/bash
mkdir -p gpurun_out
V='s400:;s300:CSRC_GPU_CR_SLACK_PCT=300;s500:CSRC_GPU_CR_SLACK_PCT=500;s600:CSRC_GPU_CR_SLACK_PCT=600;r4s400:CSRC_GPU_CW_R=4;r4s500:CSRC_GPU_CW_R=4,CSRC_GPU_CR_SLACK_PCT=500'
DT=f32 REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s8_slack.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s8_slack.txt
V='s800:;s1200:CSRC_GPU_CR_SLACK_PCT=1200;s1600:CSRC_GPU_CR_SLACK_PCT=1600'
REPS=50 timeout 600 python tools/probe_r2.py c3,c4,c2 colorful "$V" >> gpurun_out/r2s8_slack.txt 2>&1; echo "rc=$?"; tail -12 gpurun_out/r2s8_slack.txt
