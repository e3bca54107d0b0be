#!/bin/bash
mkdir -p gpurun_out
V='b3:;u8:CSRC_GPU_CW_U=8;u16:CSRC_GPU_CW_U=16'
DT=f32 REPS=50 timeout 600 python tools/probe_r2.py c5 colorful "$V" > gpurun_out/r2s6_f32col.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s6_f32col.txt
