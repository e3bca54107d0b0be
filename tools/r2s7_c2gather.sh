#!/bin/bash
mkdir -p gpurun_out
V='base:;nb2:CSRC_GPU_GNB=2;nt64:CSRC_GPU_GNT=64;nt64nb2:CSRC_GPU_GNT=64,CSRC_GPU_GNB=2;nt256:CSRC_GPU_GNT=256;l4:CSRC_GPU_GLANES=4;l4nb2:CSRC_GPU_GLANES=4,CSRC_GPU_GNB=2;sell:CSRC_GPU_GSELL=1;nopat:CSRC_GPU_GPATTERN=0;bpsm8:CSRC_GPU_GBPSM=8'
REPS=300 timeout 400 python tools/probe_r2.py c2,c1 gather "$V" > gpurun_out/r2s7_c2gather.txt 2>&1; echo "rc=$?"; cat gpurun_out/r2s7_c2gather.txt
