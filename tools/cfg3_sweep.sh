#!/bin/bash
# configs[2] (Table V shapes): MobileNet-v1 width alpha x resolution R at batch 128, bf16, both
# layouts, each a full tuned bench.py step.  Run under gpurun from the repo root; lines -> gpurun_out/cfg3/.
mkdir -p gpurun_out/cfg3
for lay in nchw nhwc; do
  for a in 0.25 0.5 0.75 1.0; do
    for r in 128 160 192 224; do
      timeout 300 python bench.py --alpha $a --res $r --batch 128 --dtype bf16 --layout $lay --steps 50 --warmup 5 \
        --no-cpu-baseline --e2e-steps 0 --no-b128 --kernel-reps 2 > gpurun_out/cfg3/${lay}_a${a}_r${r}.json 2>&1
    done
  done
done
