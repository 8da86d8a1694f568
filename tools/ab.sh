#!/bin/bash
# A/B stage times of builds of liblzb.so on one box (alternating runs).
# usage: CFG=c5q N=2 tools/ab.sh lib1.so lib2.so ...
CFG=${CFG:-c5q}; N=${N:-2}
mkdir -p gpurun_out
for i in $(seq $N); do
  for L in "$@"; do
    LZB_LIB=$L python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 2>/dev/null \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['stages_ms'], d['compress_ms'], d['decompress_ms'])"
  done
done
