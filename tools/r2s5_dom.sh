#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csr.py -x -q -m gpu -k "f32 or fp32 or gather or pattern or mesh or family or non_finite or guard or writes" > gpurun_out/r2s5_dom_tests.txt 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2s5_dom_tests.txt
[ $rc -ne 0 ] && exit 1
V='dom:;nodom:CSRC_GPU_GDOM=0'
DT=f32 REPS=200 timeout 600 python tools/probe_r2.py c5,c2,c1 gather "$V" > gpurun_out/r2s5_dom.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s5_dom.txt
DT=f32 REPS=200 timeout 600 python tools/probe_r2.py c5 gather "$V" >> gpurun_out/r2s5_dom.txt 2>&1; tail -3 gpurun_out/r2s5_dom.txt
