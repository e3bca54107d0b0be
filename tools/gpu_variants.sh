#!/bin/bash
# A/B of k_gather_staged build variants (tools/build_gather_variants.sh): each variant library
# is swapped in as the product library of this scratch copy, then the gather probe runs.
mkdir -p gpurun_out
cp paper_1003_0952_b200/libcsrc_b200.so /tmp/lib_current.so
for v in ${VARIANTS:-head o0p0 o1p0 o0p1}; do
  cp tools/_variants/lib_$v.so paper_1003_0952_b200/libcsrc_b200.so
  for e in 'X=0' 'CSRC_GPU_GMINB=6'; do
    env $e TAG="$v $e" timeout 300 python tools/gather_probe.py c5,c4,c3 f64,f32 2>&1 | grep -v Warn
  done
done | tee gpurun_out/sweep_variants.txt
cp /tmp/lib_current.so paper_1003_0952_b200/libcsrc_b200.so
