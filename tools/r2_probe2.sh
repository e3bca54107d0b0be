#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/probe_r2.py c2,c3,c5 colorful,colorful_exact 'wave:;s8:CSRC_GPU_CW_S=8;s32:CSRC_GPU_CW_S=32;nt256:CSRC_GPU_CW_NT=256;u4:CSRC_GPU_CW_U=4;u16nt256:CSRC_GPU_CW_U=16,CSRC_GPU_CW_NT=256' > gpurun_out/r2p2_colored.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p2_colored.txt
timeout 600 python tools/probe_r2.py c4 colorful 'wave:;s32:CSRC_GPU_CW_S=32;nt256:CSRC_GPU_CW_NT=256' >> gpurun_out/r2p2_colored.txt 2>&1; tail -4 gpurun_out/r2p2_colored.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colorful or lb_ or local_buffers or large" > gpurun_out/r2p2_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2p2_pytest.log
