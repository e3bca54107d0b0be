#!/bin/bash
mkdir -p gpurun_out
V='r4d8:;r4d12:CSRC_GPU_CW_D=12;r4d16:CSRC_GPU_CW_D=16;r2d6:CSRC_GPU_CW_R=2,CSRC_GPU_CW_D=6;r1d3:CSRC_GPU_CW_R=1,CSRC_GPU_CW_D=3;u4d16:CSRC_GPU_CW_U=4,CSRC_GPU_CW_D=16;nt256d16:CSRC_GPU_CW_NT=256,CSRC_GPU_CW_D=16;u16d16:CSRC_GPU_CW_U=16,CSRC_GPU_CW_D=16'
REPS=20 timeout 1500 python tools/probe_r2.py c5,c3,c4 colorful "$V" > gpurun_out/r2p4_colored.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p4_colored.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colorful or known or family or meshes" > gpurun_out/r2p4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2p4_pytest.log
