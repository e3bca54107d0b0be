#!/bin/bash
mkdir -p gpurun_out
for v in 'CSRC_GPU_GMINB=1' 'CSRC_GPU_GMINB=6' 'CSRC_GPU_GMINB=5' 'CSRC_GPU_GMINB=1' 'CSRC_GPU_GMINB=6'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c3,c2 f64,f32 2>&1 | grep -v Warn
done | tee gpurun_out/sweep_minb.txt
