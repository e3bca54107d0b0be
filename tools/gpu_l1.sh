#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gather_kernel_shapes or host_pipeline or known or meshes" > gpurun_out/pytest_l1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_l1.log
for r in 1 2; do
for v in 'X=0' 'CSRC_GPU_GLANES=1' 'CSRC_GPU_GLANES=1 CSRC_GPU_GNT=128' 'CSRC_GPU_GLANES=1 CSRC_GPU_GNT=256' 'CSRC_GPU_GLANES=1 CSRC_GPU_GNT=64'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c3,c2 f64,f32 2>&1 | grep -v Warn
done; done | tee gpurun_out/sweep_l1.txt
