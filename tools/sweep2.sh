#!/bin/bash
for cfg in ${CFGS:-c5}; do for M in ${MINC:-2}; do for L in ${LANES:-1 2 4}; do for S in ${STAGES:-4}; do for R in ${RUNS:-4}; do
  echo "## cfg=$cfg minctas=$M L=$L S=$S R=$R"
  CSRC_GPU_MINCTAS=$M CSRC_GPU_LANES=$L CSRC_GPU_STAGES=$S CSRC_GPU_RUN_LEN=$R KINDS=windowed NOF32=1 timeout 120 python tools/gpu_probe.py $cfg 2>&1 | grep -E "windowed|FAIL|rror" | sed 's/plan [^ ]* //; s/hot .*cold / /; s/win .*//'
done; done; done; done; done
