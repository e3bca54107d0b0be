#!/bin/bash
mkdir -p gpurun_out
timeout 420 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "colorful or color" > gpurun_out/r2s6_coldef_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s6_coldef_tests.txt
[ $rc -ne 0 ] && exit 1
V='final:'
REPS=50 timeout 1200 python tools/probe_r2.py c5,c4,c3,c2,c1 colorful "$V" > gpurun_out/r2s6_coldef3.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s6_coldef3.txt
DT=f32 REPS=50 timeout 600 python tools/probe_r2.py c5,c4 colorful "$V" >> gpurun_out/r2s6_coldef3.txt 2>&1; tail -4 gpurun_out/r2s6_coldef3.txt
