#!/bin/bash
# The round's evidence on one B200: default bench (C5), reference arm, C1-C4,
# and the per-launch ncu list (time + DRAM bytes) of one C5 step.  TAG = prefix.
TAG=${1:-r2}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench_c5.jsonl 2> gpurun_out/${TAG}_bench_c5.err
python bench.py --impl reference > gpurun_out/${TAG}_bench_c5_reference.jsonl 2> gpurun_out/${TAG}_ref.err
for c in c1 c2 c3 c4; do
  python bench.py --config $c --e2e-steps 4 >> gpurun_out/${TAG}_bench_c1_c4.jsonl 2>> gpurun_out/${TAG}_c1c4.err
done
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv -k 'regex:lzb|k_' --log-file gpurun_out/${TAG}_launches_c5_raw.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > gpurun_out/${TAG}_launches.log 2>&1
nvidia-smi -q -d CLOCK | head -30 > gpurun_out/${TAG}_clocks_after.txt
