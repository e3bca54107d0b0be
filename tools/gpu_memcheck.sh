#!/bin/bash
# compute-sanitizer memcheck over the small-input GPU tests (out-of-bounds / misaligned accesses)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "known or edge or non_finite or (meshes and not fp32) or sliced or rings or interior" > gpurun_out/memcheck_parity.log 2>&1
echo "memcheck parity rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/memcheck_parity.log | head -20
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_rect.py tests/test_gpu_csr.py tests/test_gpu_assemble.py -m gpu -q -x -p no:cacheprovider \
  -k "not config_round_trip and not host_pipeline" > gpurun_out/memcheck_other.log 2>&1
echo "memcheck other rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/memcheck_other.log | head -20
