#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin_cpp.py tests/test_gpu_rect.py -m gpu -q -x -k "windowed or lb_ or local or band or rings or dropin or rect or known or meshes" > gpurun_out/pytest_win.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_win.log
for v in 'CSRC_GPU_LANES=4' 'CSRC_GPU_LANES=4 CSRC_GPU_STAGES=2' 'CSRC_GPU_LANES=2' 'CSRC_GPU_LANES=4 CSRC_GPU_MINCTAS=3'; do
  echo "## $v"
  for cfg in c5 c4 c3 c2; do env $v KINDS=windowed,lb_interval NOF32=1 timeout 300 python tools/gpu_probe.py $cfg 2>&1 | grep -E "^  [a-z]" | sed "s/^/$cfg /"; done
done | tee gpurun_out/sweep_win3.txt
