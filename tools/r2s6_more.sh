#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_dropin_cpp.py tests/test_gpu_bandexec.py -x -q -m gpu > gpurun_out/r2s6_dropin.txt 2>&1; echo "dropin rc=$?"; tail -5 gpurun_out/r2s6_dropin.txt
timeout 60 oracle/_ref/dropin_test; echo "bin rc=$?"
V='base:;l1:CSRC_GPU_LANES=1;l4:CSRC_GPU_LANES=4;t64:CSRC_GPU_TILE=64;m4:CSRC_GPU_MINCTAS=4;st3m2:CSRC_GPU_STAGES=3,CSRC_GPU_MINCTAS=2;run4:CSRC_GPU_RUN_LEN=4'
DT=f32 REPS=100 timeout 600 python tools/probe_r2.py c5 windowed "$V" > gpurun_out/r2s6_win_f32.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s6_win_f32.txt
