#!/bin/bash
# ncu of the remaining kernel families on C5: colored (one class launch), local-buffers accumulation, atomic
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_colored -c 1 -o gpurun_out/ncu_colored_c5 python tools/prof_one.py c5 colorful 2 > gpurun_out/ncu_col.log 2>&1; echo "col rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_accum -c 1 -o gpurun_out/ncu_accum_c5 python tools/prof_one.py c5 local_buffers 2 > gpurun_out/ncu_acc.log 2>&1; echo "acc rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:k_atomic -c 1 -o gpurun_out/ncu_atomic_c5 python tools/prof_one.py c5 atomic 2 > gpurun_out/ncu_atom.log 2>&1; echo "atom rc=$?"
