#!/bin/bash
# final staged-gather build: parity subset, probe, f32 ncu; host-link chunking probe
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csr.py tests/test_gpu_rect.py tests/test_dropin_cpp.py -m gpu -x -q -k "gather or sequential or known or band or host_pipeline or row_patterns or meshes or csr or rect or fp32 or edge or ragged or outside or dropin or torch_stream or large" > gpurun_out/pytest_v3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_v3.log
TAG=final timeout 300 python tools/gather_probe.py c5,c4,c3,c2 f64,f32 2>&1 | grep -v Warn | tee gpurun_out/sweep_v3.txt
timeout 300 python tools/pcie_chunk_probe.py 2>&1 | tee gpurun_out/pcie_chunks.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather -c 1 -f -o /tmp/ncu/g32 python tools/prof_one.py c5 gather 2 f32 > /tmp/ncu/g32.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/ncu/g32.ncu-rep > gpurun_out/ncu_gather_f32_c5_v2_summary.txt 2>&1; head -30 gpurun_out/ncu_gather_f32_c5_v2_summary.txt
ncu -i /tmp/ncu/g32.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_g32v2_source.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather -c 1 -f -o /tmp/ncu/g64 python tools/prof_one.py c5 gather 2 > /tmp/ncu/g64.log 2>&1; echo "ncu64 rc=$?"
python tools/ncu_summary.py /tmp/ncu/g64.ncu-rep > gpurun_out/ncu_gather_f64_c5_v2_summary.txt 2>&1; head -30 gpurun_out/ncu_gather_f64_c5_v2_summary.txt
