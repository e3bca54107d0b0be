#!/bin/bash
# ncu of the remaining kernel families on C5 (colored class launch, local-buffers
# accumulation, atomic), summarised on the box (the reports are too large to ship back)
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none -k regex:k_colored -c 1 -f -o /tmp/ncu/col python tools/prof_one.py c5 colorful 2 > /tmp/ncu/col.log 2>&1; echo "col rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_accum -c 1 -f -o /tmp/ncu/acc python tools/prof_one.py c5 local_buffers 2 > /tmp/ncu/acc.log 2>&1; echo "acc rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:k_atomic -c 1 -f -o /tmp/ncu/atom python tools/prof_one.py c5 atomic 2 > /tmp/ncu/atom.log 2>&1; echo "atom rc=$?"
for r in col acc atom; do python tools/ncu_summary.py /tmp/ncu/$r.ncu-rep > gpurun_out/ncu_${r}_c5_summary.txt 2>&1; head -3 gpurun_out/ncu_${r}_c5_summary.txt; done
