#!/bin/bash
# windowed-kernel tuning sweep: lanes x run length (x stages)
for cfg in ${CFGS:-c5}; do
for L in ${LANES:-2 4}; do for R in ${RUNS:-1 4}; do for S in ${STAGES:-4}; do
  echo "## cfg=$cfg L=$L R=$R S=$S"
  CSRC_GPU_LANES=$L CSRC_GPU_RUN_LEN=$R CSRC_GPU_STAGES=$S KINDS=windowed NOF32=1 timeout 120 python tools/gpu_probe.py $cfg 2>&1 | grep -E "windowed|FAIL|rror" | sed 's/err [^ ]* //; s/plan [^ ]* //'
done; done; done; done
