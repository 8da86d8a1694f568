#!/bin/bash
# ncu --set full (with source) of chosen kernels of one bench config: TAG CONFIG REGEX [COUNT]
set -u
TAG=$1; CFG=$2; KS=$3; C=${4:-4}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k "$KS" -c $C -f -o gpurun_out/prof_${TAG} \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > gpurun_out/prof_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
ls -la gpurun_out/prof_${TAG}*
