#!/bin/bash
# ncu --set full of the hot kernels on C5q (512x2048x2048: same decode layout
# S=8192 as C5, a quarter of the memory so ncu's save/restore stays cheap).
set -u
TAG=${1:-r1c}
KS=${2:-'regex:k_quantize3d8_tma|k_huff_count_w|k_huff_encode_w|k_dec4_count|k_dec_final9|k_reconstruct3d8'}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k "$KS" -c 6 \
  -f -o gpurun_out/prof_${TAG} \
  python bench.py --config c5q --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > gpurun_out/prof_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
