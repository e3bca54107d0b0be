#!/bin/bash
# Functional check of bench.py's N>1 path on a one-GPU box: gather bands (no data-path collective),
# ranks share the GPU, timing collectives over gloo (CSRC_BENCH_SHARE_GPU=1). Not measurements.
mkdir -p gpurun_out
run() {  # nproc config extra...
  local n=$1 cfg=$2; shift 2
  CSRC_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n --config $cfg --steps 20 --warmup 3 \
    --compare "" "$@" > gpurun_out/share_${n}_${cfg}.json 2> gpurun_out/share_${n}_${cfg}.err
  echo "n=$n $cfg rc=$?"; tail -c 600 gpurun_out/share_${n}_${cfg}.json; tail -2 gpurun_out/share_${n}_${cfg}.err
}
run 2 c3
run 4 c3
run 8 c2
run 2 c5
free -g | head -2
