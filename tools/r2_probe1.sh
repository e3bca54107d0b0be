#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colorful or lb_ or local_buffers or known or meshes or family or mixing or smaller" > gpurun_out/r2p1_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2p1_pytest.log
timeout 900 python tools/probe_r2.py c2,c5 colorful,colorful_exact 'wave:;s8:CSRC_GPU_CW_S=8;s32:CSRC_GPU_CW_S=32;s64:CSRC_GPU_CW_S=64;u4:CSRC_GPU_CW_U=4;old:CSRC_GPU_COLOR_WAVE=0' > gpurun_out/r2p1_colored.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p1_colored.txt
timeout 900 python tools/probe_r2.py c2,c3,c4,c5 windowed,lb_all_in_one,lb_per_buffer,lb_effective,lb_interval,colorful > gpurun_out/r2p1_lb.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2p1_lb.txt
