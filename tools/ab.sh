#!/bin/bash
# A/B stage times of two builds of liblzb.so on one box (alternating runs).
# usage: tools/ab.sh ab/liblzb_base.so paper_2105_12912_b200/_lib/liblzb.so [config] [reps]
A=$1; B=$2; CFG=${3:-c5q}; N=${4:-2}
mkdir -p gpurun_out
for i in $(seq $N); do
  for L in $A $B; do
    LZB_LIB=$L python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 2>/dev/null \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['stages_ms'], d['compress_ms'], d['decompress_ms'])"
  done
done
