#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_dropin_cpp.py -x -q -m gpu > gpurun_out/r2s6_dropin.txt 2>&1; echo "dropin rc=$?"; tail -3 gpurun_out/r2s6_dropin.txt
V='new:;m3:CSRC_GPU_MINCTAS=3'
DT=f32 REPS=100 timeout 600 python tools/probe_r2.py c5,c4,c3,c2 windowed,lb_interval "$V" > gpurun_out/r2s6_win_f32b.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s6_win_f32b.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "f32 or fp32 or windowed or local" > gpurun_out/r2s6_f32_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2s6_f32_tests.txt
