#!/bin/bash
mkdir -p gpurun_out
for v in 'CSRC_GPU_GPSMEM=0' 'CSRC_GPU_GPSMEM=1' 'CSRC_GPU_GPSMEM=0' 'CSRC_GPU_GPSMEM=1' 'CSRC_GPU_GPSMEM=1 CSRC_GPU_GSELL=0' 'CSRC_GPU_GPSMEM=0 CSRC_GPU_GSELL=0'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c4,c2 f64,f32 2>&1 | grep -v Warn
done | tee gpurun_out/sweep_psmem.txt
