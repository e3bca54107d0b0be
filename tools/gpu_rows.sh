#!/bin/bash
# staged row setup (eptr / pbase with the values): parity + A/B against global row-setup loads
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csr.py tests/test_gpu_rect.py tests/test_dropin_cpp.py -m gpu -x -q -k "gather or sequential or known or band or host_pipeline or row_patterns or meshes or csr or rect or fp32 or edge or ragged or outside or dropin or torch_stream or large or family" > gpurun_out/pytest_rows.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_rows.log
for r in 1 2; do
for v in 'CSRC_GPU_GROWS=0' 'CSRC_GPU_GROWS=1'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c4,c3,c2 f64,f32 2>&1 | grep -v Warn
done; done | tee gpurun_out/sweep_rows.txt
