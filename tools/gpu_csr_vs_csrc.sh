#!/bin/bash
mkdir -p gpurun_out
for cfg in c5 c4 c3; do
  for args in "--format csr" "--strategy gather" "--strategy windowed" "--strategy atomic"; do
    echo "## $cfg $args"
    timeout 600 ./paper_1003_0952_b200/csrc_bench run --config $cfg $args --reps 200 --runs 3 2>&1 | tail -1
  done
done | tee gpurun_out/csr_vs_csrc.txt
