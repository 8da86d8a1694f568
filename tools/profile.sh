#!/bin/bash
# Round profile (run on the GPU box from the repo root, one GPU):
#  1. launch list of the default bench command (C5), serialised, cold-cache
#  2. one `--set full` capture of each hot kernel on C5q (512x2048x2048: the
#     C5 per-element and decode-layout behaviour at a quarter of the memory
#     ncu has to save/restore per replay)
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/launches_${TAG}_c5.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_quantize3d8_tma|k_huff_count_w|k_huff_encode_w|k_dec_maps3|k_dec_final9|k_reconstruct3d8' -c 6 \
  -f -o gpurun_out/prof_${TAG}_full \
  python bench.py --config c5q --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/prof_${TAG}_full.log 2>&1
ncu -i gpurun_out/prof_${TAG}_full.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_full_raw.csv 2>/dev/null
