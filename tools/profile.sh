#!/bin/bash
# Round profile (run on the GPU box from the repo root, one GPU):
#  1. launch list of the default bench command (C5), serialised, cold-cache
#  2. one `--set full` capture of each hot kernel on C5s (512^3; the C5 run
#     would need ncu to save/restore ~60 GB of device memory per replay)
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/launches_${TAG}_c5.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_quantize3d8|k_huff_count_w|k_huff_encode_w|k_dec_maps2|k_dec_final6|k_reconstruct3d8' -c 6 \
  -f -o gpurun_out/prof_${TAG}_full \
  python bench.py --config c5s --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/prof_${TAG}_full.log 2>&1
ncu -i gpurun_out/prof_${TAG}_full.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_full_raw.csv 2>/dev/null
