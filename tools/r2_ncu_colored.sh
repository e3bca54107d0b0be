#!/bin/bash
mkdir -p gpurun_out
python tools/prof_one.py c5 colorful 2 > gpurun_out/r2_prof_colored.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_colored_wave -c 1 -o gpurun_out/r2_ncu_colored_c5 python tools/prof_one.py c5 colorful 2 > gpurun_out/r2_ncu_colored.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2_ncu_colored.log
