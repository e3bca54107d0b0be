#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rect.py tests/test_gpu_dropin.py -x -q -m gpu -k "colorful or color or edge or known or rect or accessors" > gpurun_out/r2s7_r160_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s7_r160_tests.txt
[ $rc -ne 0 ] && exit 1
V='final:'
REPS=100 timeout 900 python tools/probe_r2.py c5,c4,c3,c2,c1 colorful "$V" > gpurun_out/r2s7_r160b.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s7_r160b.txt
DT=f32 REPS=100 timeout 600 python tools/probe_r2.py c5,c4 colorful "$V" >> gpurun_out/r2s7_r160b.txt 2>&1; tail -4 gpurun_out/r2s7_r160b.txt
SPECS="colorful:k_colored_ring:colored_ring160" bash tools/r2s4_ncu.sh > gpurun_out/r2s7_ncu_ring160.log 2>&1; tail -28 gpurun_out/r2s7_ncu_ring160.log
