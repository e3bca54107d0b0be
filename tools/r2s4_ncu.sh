#!/bin/bash
# round 2 (session 4): ncu --set full of the round-2 kernels at C5, summarised on the box
# (the reports exceed gpurun's 64 MiB return limit): raw-page summary + SASS hot spots.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for spec in ${SPECS:-"colorful:k_colored_wave:colored_wave" "windowed:k_windowed:windowed3" "local_buffers:k_accum:accum"}; do
  IFS=: read kind kern tag <<< "$spec"
  timeout 600 python tools/prof_one.py ${CFG:-c5} $kind 2 ${DT:-f64} > gpurun_out/r2s4_prof_$tag.log 2>&1; echo "$kind plain rc=$?"
  rep=/tmp/r2s4_ncu_$tag.ncu-rep
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -f -o ${rep%.ncu-rep} python tools/prof_one.py ${CFG:-c5} $kind 2 ${DT:-f64} > gpurun_out/r2s4_ncu_$tag.log 2>&1; echo "$kind ncu rc=$?"
  python tools/ncu_summary.py $rep > gpurun_out/r2s4_ncu_${tag}_summary.txt 2>&1
  ncu -i $rep --page source --csv --print-source sass > /tmp/src_$tag.csv 2>/dev/null && python tools/ncu_sass_hotspots.py /tmp/src_$tag.csv > gpurun_out/r2s4_ncu_${tag}_sass_hotspots.txt 2>&1
  cat gpurun_out/r2s4_ncu_${tag}_summary.txt
done
