#!/bin/bash
# windowed-kernel ablation: time with parts disabled (results invalid) -> where time goes
for cfg in ${CFGS:-c5}; do for A in 0 1 2 4 8 5 13 16 31; do
  echo "## cfg=$cfg ablate=$A"
  CSRC_GPU_ABLATE=$A KINDS=windowed NOF32=1 timeout 120 python tools/gpu_probe.py $cfg 2>&1 | grep -E "windowed|FAIL|rror" | sed 's/plan [^ ]* //' | cut -c1-120
done; done
