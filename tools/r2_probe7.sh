#!/bin/bash
mkdir -p gpurun_out
V='base:;st2:CSRC_GPU_STAGES=2;st4:CSRC_GPU_STAGES=4,CSRC_GPU_MINCTAS=1;st3m1:CSRC_GPU_STAGES=3,CSRC_GPU_MINCTAS=1;t64:CSRC_GPU_TILE=64;t64st4:CSRC_GPU_TILE=64,CSRC_GPU_STAGES=4;run8:CSRC_GPU_RUN_LEN=8;run16:CSRC_GPU_RUN_LEN=16;run2:CSRC_GPU_RUN_LEN=2,CSRC_GPU_STAGES=2;m3:CSRC_GPU_MINCTAS=3'
REPS=100 timeout 1500 python tools/probe_r2.py c5,c3 windowed "$V" > gpurun_out/r2p7_windowed.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p7_windowed.txt
