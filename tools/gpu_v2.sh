#!/bin/bash
# staged gather v2 (32-bit column ids, ordered gathers, pipelined row setup): parity + sweep,
# then the host-link contention probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csr.py tests/test_gpu_rect.py -m gpu -x -q -k "gather or sequential or known or band or host_pipeline or row_patterns or meshes or csr or rect or fp32 or edge or ragged or outside" > gpurun_out/pytest_v2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_v2.log
for v in 'X=0' 'CSRC_GPU_GMINB=5' 'CSRC_GPU_GMINB=6' 'CSRC_GPU_GMINB=8' 'CSRC_GPU_GNT=128' 'CSRC_GPU_GNT=256' 'CSRC_GPU_GNT=128 CSRC_GPU_GMINB=8' 'CSRC_GPU_GU=4'; do
  env $v TAG="$v" timeout 300 python tools/gather_probe.py c5,c4,c3 f64,f32 2>&1 | grep -v Warn
done | tee gpurun_out/sweep_v2.txt
timeout 600 python tools/pcie_contention_probe.py > gpurun_out/pcie_contention.txt 2>&1; echo "pcie rc=$?"; cat gpurun_out/pcie_contention.txt | grep -v "^  chunk"
