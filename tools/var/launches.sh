#!/bin/bash
# Launch list (per-kernel serialized GPU time) of one C5 assembly, FP64 and FP32.
OUT=gpurun_out; mkdir -p $OUT; TAG=${TAG:-cur}
A="--steps 1 --warmup 1 --no-e2e --no-cpu"
for p in double single; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${TAG}_$p.csv python bench.py --precision $p $A > /dev/null 2>&1
  python tools/ncu_summary.py $OUT/launches_${TAG}_$p.csv 2>&1 | head -24
done
