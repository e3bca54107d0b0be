#!/bin/bash
mkdir -p gpurun_out
V='new:;old:CSRC_GPU_MINCTAS=2,CSRC_GPU_RUN_LEN=4;t64:CSRC_GPU_TILE=64;t32:CSRC_GPU_TILE=32;run4:CSRC_GPU_RUN_LEN=4'
REPS=100 timeout 1500 python tools/probe_r2.py c5,c4,c3,c2 windowed,lb_interval "$V" > gpurun_out/r2p8_windowed.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p8_windowed.txt
DT=f32 REPS=100 timeout 900 python tools/probe_r2.py c5 windowed "$V" >> gpurun_out/r2p8_windowed.txt 2>&1; tail -6 gpurun_out/r2p8_windowed.txt
