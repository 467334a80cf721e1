#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py); run under gpurun from the repo root.
# Writes gpurun_out/sanitize/<tool>.log; the summary goes to profiles/ by hand.
set -u
out=gpurun_out/sanitize
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_cases.py --all-candidates \
  > $out/memcheck.log 2>&1; echo "memcheck rc=$?" >> $out/memcheck.log
timeout 1200 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize_cases.py \
  > $out/racecheck.log 2>&1; echo "racecheck rc=$?" >> $out/racecheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py --all-candidates \
  > $out/synccheck.log 2>&1; echo "synccheck rc=$?" >> $out/synccheck.log
timeout 900 $CS --tool initcheck --error-exitcode 9 python tools/sanitize_cases.py \
  > $out/initcheck.log 2>&1; echo "initcheck rc=$?" >> $out/initcheck.log
tail -n 3 $out/*.log
