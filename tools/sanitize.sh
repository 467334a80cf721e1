#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py); run under gpurun from the repo root.
# Writes gpurun_out/sanitize/<tool>.log (racecheck: grouped summary per case); summaries go to profiles/ by hand.
set -u
out=gpurun_out/sanitize
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_cases.py --all-candidates \
  > $out/memcheck.log 2>&1; echo "memcheck rc=$?" >> $out/memcheck.log
for c in cfg1 small14 small7_bf16 band56_s2 nhwc_tma_s1 nhwc_tma_s2_bf16 k5 k7_nhwc m2 bdmma_k5 small14_s2 small14_s2_bf16 nhwc_gen_k5; do
  timeout 600 $CS --tool racecheck --racecheck-report all --print-limit 100000000 python tools/sanitize_cases.py --all-candidates --only $c \
    2>&1 | python tools/racecheck_summary.py > $out/racecheck_$c.txt
done
# synccheck aborts the process at the tcgen05 candidate (profiles/r2/README.md), so it is run apart
timeout 900 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py --all-candidates \
  --skip-variant nhwc_bdmma > $out/synccheck.log 2>&1; echo "synccheck rc=$?" >> $out/synccheck.log
timeout 300 $CS --tool synccheck python tools/sanitize_cases.py --all-candidates --only bdmma_k5 \
  > $out/synccheck_bdmma.log 2>&1; echo "synccheck rc=$?" >> $out/synccheck_bdmma.log
timeout 900 $CS --tool initcheck --error-exitcode 9 python tools/sanitize_cases.py \
  > $out/initcheck.log 2>&1; echo "initcheck rc=$?" >> $out/initcheck.log
tail -n 3 $out/*.log; head -n 4 $out/racecheck_*.txt
