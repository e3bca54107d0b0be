#!/bin/bash
# stream-ordering fix: new ordering test + device/band tests, N>1 bench path on a shared GPU,
# and an ncu capture of the fp32 C5 gather kernel (summarised on the box)
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests -m gpu -q -x -k "torch_stream or band or interior or device_and_graph or pageable" > gpurun_out/pytest_stream.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_stream.log
for spec in "2 c3" "2 c5"; do
  set -- $spec
  CSRC_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 \
    --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus $1 --config $2 --steps 20 --warmup 3 \
    --compare "" > gpurun_out/share_$1_$2.json 2> gpurun_out/share_$1_$2.err
  echo "share n=$1 $2 rc=$?"; python -c "
import json,sys; d=json.load(open('gpurun_out/share_$1_$2.json')); print(d['ms_per_step'], d['value'], d['roofline']['kernel_ms'], d['e2e']['wall_ms_per_step'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather -c 1 -f -o /tmp/ncu/g32 python tools/prof_one.py c5 gather 2 f32 > /tmp/ncu/g32.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/ncu/g32.ncu-rep > gpurun_out/ncu_gather_f32_c5_summary.txt 2>&1; head -40 gpurun_out/ncu_gather_f32_c5_summary.txt
ncu -i /tmp/ncu/g32.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_g32_source.csv 2>/dev/null; ls -la gpurun_out/ncu_g32_source.csv
