#!/bin/bash
mkdir -p gpurun_out
V='base:;comb:CSRC_GPU_WIN_COMBINE=1;l1:CSRC_GPU_LANES=1;l1comb:CSRC_GPU_LANES=1,CSRC_GPU_WIN_COMBINE=1;l4comb:CSRC_GPU_LANES=4,CSRC_GPU_WIN_COMBINE=1'
REPS=50 timeout 1500 python tools/probe_r2.py c5,c3,c4,c2 windowed "$V" > gpurun_out/r2p6_windowed.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p6_windowed.txt
DT=f32 REPS=50 timeout 900 python tools/probe_r2.py c5 windowed "$V" >> gpurun_out/r2p6_windowed.txt 2>&1; tail -6 gpurun_out/r2p6_windowed.txt
