#!/bin/bash
# SELL gather kernel: parity (gather kinds, drop-in, rect), then a sweep against the staged kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin_cpp.py tests/test_gpu_rect.py -m gpu -x -q -k "gather or sequential or known or dropin or rect" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
CFGS="c5 c4 c3 c2" ./tools/sweep_env.sh 'CSRC_GPU_GSELL=0' 'CSRC_GPU_SELL_L=1 CSRC_GPU_SELL_U=8' 'CSRC_GPU_SELL_L=2 CSRC_GPU_SELL_U=4' 'CSRC_GPU_SELL_L=2 CSRC_GPU_SELL_U=8' 'CSRC_GPU_SELL_L=4 CSRC_GPU_SELL_U=4' 'CSRC_GPU_SELL_L=4 CSRC_GPU_SELL_U=8' > gpurun_out/sweep_sell2.txt 2>&1
cat gpurun_out/sweep_sell2.txt
