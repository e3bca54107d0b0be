#!/bin/bash
# one-row-per-thread fp32 gather: default (43 regs, 5 blocks/SM) vs a 6-block __launch_bounds__ (40 regs)
mkdir -p gpurun_out
CSRC_GPU_GMINB=6 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gather_kernel_shapes or known or meshes" > gpurun_out/pytest_minb_l1.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_minb_l1.log
for r in 1 2 3; do
for v in 'X=0' 'CSRC_GPU_GMINB=6'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c3,c4 f32 2>&1 | grep -v Warn
done; done | tee gpurun_out/sweep_minb_l1.txt
