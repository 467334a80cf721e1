#!/bin/bash
# Capture the evidence for profiles/: the launch list of one bench step and full
# ncu reports of the heaviest launches.  Run under gpurun from the repo root.
set -u
out=gpurun_out/prof
mkdir -p $out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --kernel-reps 0 > $out/launches_bench.json 2>&1
for spec in "$@"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:nchw -s 1 -c 1 -o $out/full_$1_$2 \
      python tools/run_layer.py --layer $1 --pass $2 --reps 2 > /dev/null 2>&1
done
