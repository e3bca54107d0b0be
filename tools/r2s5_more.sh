#!/bin/bash
mkdir -p gpurun_out
SPECS="colorful:k_colored_ring:colored_ring" bash tools/r2s4_ncu.sh > gpurun_out/r2s5_ncu_ring.log 2>&1; tail -30 gpurun_out/r2s5_ncu_ring.log
V='base:;t64:CSRC_GPU_TILE=64;t32:CSRC_GPU_TILE=32;t64m4:CSRC_GPU_TILE=64,CSRC_GPU_MINCTAS=4;t32m6:CSRC_GPU_TILE=32,CSRC_GPU_MINCTAS=6;st3:CSRC_GPU_STAGES=3,CSRC_GPU_MINCTAS=2;l1:CSRC_GPU_LANES=1;l4:CSRC_GPU_LANES=4;t64l4:CSRC_GPU_TILE=64,CSRC_GPU_LANES=4'
REPS=200 timeout 300 python tools/probe_r2.py c2,c1 windowed,gather "$V" > gpurun_out/r2s5_small_sweep.txt 2>&1; echo "small rc=$?"; cat gpurun_out/r2s5_small_sweep.txt
timeout 900 python tools/gpu_probe.py c2,c3,c4,c5 > gpurun_out/r2s5_probe_all.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2s5_probe_all.txt
