#!/bin/bash
# halo-aligned x chunks in the host pipeline: host-path parity, then A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin_cpp.py tests/test_gpu_csr.py -m gpu -x -q -k "host_pipeline or pageable or known or family or meshes or large or csr or dropin or torch_stream" > gpurun_out/pytest_xhalo.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_xhalo.log
timeout 900 python tools/xhalo_probe.py > gpurun_out/xhalo.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/xhalo.txt
