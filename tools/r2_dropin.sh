#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/oneshot_probe.py c5 > gpurun_out/r2_oneshot_c5.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/r2_oneshot_c5.txt
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_dropin_cpp.py tests/test_gpu_rect.py -m gpu -q > gpurun_out/r2_dropin_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2_dropin_pytest.log
