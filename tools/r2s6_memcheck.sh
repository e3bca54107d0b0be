#!/bin/bash
# compute-sanitizer memcheck (one tool, one call) over the small-input colored / windowed tests
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "colored_kernel_shapes and (default or PF or LANES or CLAIM or SPLIT or STAGE_BYTES) or known or edge" > gpurun_out/r2s6_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid|closed|not supported|Error" gpurun_out/r2s6_memcheck.log | head -20; tail -5 gpurun_out/r2s6_memcheck.log
