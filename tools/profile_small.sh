#!/bin/bash
# ncu --set full of the small-field kernels (C2 2D, C1 3D non-TMA) with source.
set -u
TAG=${1:-r2s}
mkdir -p gpurun_out
for cfg in c2 c1; do
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k 'regex:^k_codebook$|^k_quantize|^k_reconstruct|^k_dec4_resolve$|^k_dec4_count$|^k_dec_final9$' -c 6 \
    -f -o gpurun_out/prof_${TAG}_${cfg} python tools/smallprof.py $cfg 1 > gpurun_out/prof_${TAG}_${cfg}.log 2>&1
  ncu -i gpurun_out/prof_${TAG}_${cfg}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_${cfg}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_${TAG}_${cfg}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${TAG}_${cfg}_src.csv 2>/dev/null
done
ls -la gpurun_out/prof_${TAG}_*
