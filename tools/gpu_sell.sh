#!/bin/bash
mkdir -p gpurun_out
for v in 'CSRC_GPU_GSELL=0' 'CSRC_GPU_SELL_L=1 CSRC_GPU_SELL_U=8' 'CSRC_GPU_SELL_L=1 CSRC_GPU_SELL_U=9' 'CSRC_GPU_SELL_L=1 CSRC_GPU_SELL_U=12' 'CSRC_GPU_SELL_L=1 CSRC_GPU_SELL_U=14' 'CSRC_GPU_SELL_L=1 CSRC_GPU_SELL_U=4'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c4,c2 f64,f32 2>&1 | grep -v Warn
done | tee gpurun_out/sweep_sell3.txt
