#!/bin/bash
mkdir -p gpurun_out
export CSRC_GPU_CW_U=8
python tools/prof_one.py c5 colorful 2 > gpurun_out/r2s4_prof_ring.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_colored_ring -c 1 -o gpurun_out/r2s4_ncu_ring2_c5 python tools/prof_one.py c5 colorful 2 > gpurun_out/r2s4_ncu_ring.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2s4_ncu_ring.log
