#!/bin/bash
# usage: CFGS="c5 c3" KINDS=gather tools/sweep_env.sh "ENV1=a ENV2=b" "ENV1=c" ...
# runs tools/gpu_probe.py once per (config, env setting)
for cfg in ${CFGS:-c5}; do for setting in "$@"; do
  echo "## cfg=$cfg $setting"
  env $setting KINDS=${KINDS:-gather} NOF32=${NOF32:-1} timeout 180 python tools/gpu_probe.py $cfg 2>&1 | grep -E "^  [a-z]|FAIL|rror" | sed 's/plan [^ ]* //; s/win .*//; s/warps.*//'
done; done
