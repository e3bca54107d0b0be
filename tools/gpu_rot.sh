#!/bin/bash
mkdir -p gpurun_out
for v in 'CSRC_GPU_WIN_ROTATE=0' 'CSRC_GPU_WIN_ROTATE=3' 'CSRC_GPU_WIN_ROTATE=2' 'CSRC_GPU_WIN_ROTATE=3 CSRC_GPU_LANES=1' 'CSRC_GPU_WIN_ROTATE=0 CSRC_GPU_LANES=1'; do
  echo "## $v"
  for cfg in c4 c5 c3 c1; do env $v KINDS=windowed NOF32=1 timeout 300 python tools/gpu_probe.py $cfg 2>&1 | grep -E "^  [a-z]" | sed "s/^/$cfg /"; done
done | tee gpurun_out/sweep_rot.txt
