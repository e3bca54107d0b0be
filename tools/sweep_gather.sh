#!/bin/bash
# gather-kernel sweep: CFGS configs x GS (streaming loads) x GU (unroll) x GL (lanes)
for cfg in ${CFGS:-c5}; do for S in ${GS:-0}; do for U in ${GU:-0}; do for G in ${GL:-2 4 8}; do
  echo "## cfg=$cfg stream=$S unroll=$U glanes=$G"
  CSRC_GPU_GUNROLL=$U CSRC_GPU_GSTREAM=$S CSRC_GPU_GLANES=$G KINDS=gather NOF32=${NOF32:-1} timeout 120 python tools/gpu_probe.py $cfg 2>&1 | grep -E "gather|FAIL|rror" | sed 's/plan [^ ]* //; s/win .*//; s/warps.*//'
done; done; done; done
