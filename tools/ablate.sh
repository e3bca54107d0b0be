#!/bin/bash
# windowed-kernel ablation (tuning build only): time with parts disabled
for cfg in ${CFGS:-c5}; do for L in ${LANES:-1}; do for A in ${ABL:-0 13 45 16 32 36}; do
  echo "## cfg=$cfg L=$L ablate=$A"
  CSRC_GPU_LANES=$L CSRC_GPU_ABLATE=$A KINDS=windowed NOF32=1 timeout 120 python tools/gpu_probe.py $cfg 2>&1 | grep -E "windowed|FAIL|rror" | sed 's/plan [^ ]* //; s/hot .*cold / /' | cut -c1-90
done; done; done
