#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin_cpp.py -m gpu -x -q -k "gather or sequential or known or dropin or band or host_pipeline or row_patterns or meshes" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for v in 'CSRC_GPU_GXS=0' 'CSRC_GPU_GXS=1' 'CSRC_GPU_GXS=1 CSRC_GPU_GSELL=0' 'CSRC_GPU_GXS=0 CSRC_GPU_GSELL=0'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c4,c2 f64,f32 2>&1 | grep -v Warn
done | tee gpurun_out/sweep_xs.txt
