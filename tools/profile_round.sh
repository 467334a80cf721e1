#!/bin/bash
# Capture the evidence for profiles/: the launch list of one bench step (tuned
# plans re-installed from a saved selection, so no tuning launches run under
# ncu) and full ncu reports of chosen launches.  Run under gpurun from the repo root:
#   bash tools/profile_round.sh "<bench args>" "dw2:bwd_filter dw14:fwd ..."
set -u
out=gpurun_out/prof
mkdir -p $out /tmp/prof
rm -f /tmp/prof/plans.json  # a plan selection belongs to one workload: never reuse another run's
args=${1:-}
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --kernel-reps 0 --plans /tmp/prof/plans.json $args > $out/plans_bench.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --kernel-reps 0 \
    --plans /tmp/prof/plans.json $args > $out/launches_bench.json 2>&1
for spec in ${2:-}; do
  set -- ${spec//:/ }
  ncu --set full --clock-control none --import-source on -k regex:"nchw|dbf|nhwc|small_|band_|lane_" -s 1 -c 1 -o /tmp/prof/full_$1_$2 \
      python tools/run_layer.py --layer $1 --pass $2 --reps 2 --plans /tmp/prof/plans.json $args > /dev/null 2>&1
  ncu -i /tmp/prof/full_$1_$2.ncu-rep --page raw --csv > $out/raw_$1_$2.csv 2>&1
done
