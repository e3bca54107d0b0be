#!/bin/bash
mkdir -p gpurun_out
V='base:;l4:CSRC_GPU_LANES=4;l4t32:CSRC_GPU_LANES=4,CSRC_GPU_TILE=32;l4t32m4:CSRC_GPU_LANES=4,CSRC_GPU_TILE=32,CSRC_GPU_MINCTAS=4;t32m4:CSRC_GPU_TILE=32,CSRC_GPU_MINCTAS=4;l4t64m3:CSRC_GPU_LANES=4,CSRC_GPU_TILE=64,CSRC_GPU_MINCTAS=3;l1t64:CSRC_GPU_LANES=1,CSRC_GPU_TILE=64'
REPS=100 timeout 600 python tools/probe_r2.py c4,c3 windowed "$V" > gpurun_out/r2s5_win34.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s5_win34.txt
