#!/bin/bash
# windowed sweep: tile rows x lanes x stages x min CTAs/SM
for cfg in ${CFGS:-c5}; do for T in ${TILES:-64 128}; do for M in ${MINC:-2 3}; do for L in ${LANES:-1 2 4}; do for S in ${STAGES:-2 4 6}; do
  echo "## cfg=$cfg tile=$T minctas=$M L=$L S=$S"
  CSRC_GPU_TILE=$T CSRC_GPU_MINCTAS=$M CSRC_GPU_LANES=$L CSRC_GPU_STAGES=$S KINDS=windowed NOF32=1 timeout 120 python tools/gpu_probe.py $cfg 2>&1 | grep -E "windowed|FAIL|rror" | sed 's/plan [^ ]* //; s/hot .*cold / /; s/win .*//; s/err [^ ]* //'
done; done; done; done; done
