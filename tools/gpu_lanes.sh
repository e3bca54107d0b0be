#!/bin/bash
mkdir -p gpurun_out
for v in 'CSRC_GPU_GNT=64' 'CSRC_GPU_GNT=128' 'CSRC_GPU_GNT=64 CSRC_GPU_GU=4' 'CSRC_GPU_GNT=128 CSRC_GPU_GNB=2'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c3 f64,f32 2>&1 | grep -v Warn
done | tee gpurun_out/sweep_gnt64.txt
