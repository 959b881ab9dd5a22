#!/bin/bash
# Bench lines of every BASELINE.json configuration (C1..C5) and the C3 degree sweep.
mkdir -p gpurun_out
OUT=gpurun_out/${1:-cfg}_configs.jsonl
: > $OUT
for c in C1 C2 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $OUT 2>> gpurun_out/${1:-cfg}_configs.err
done
for p in 2 4 6 8; do
  timeout 600 python bench.py --config C3 --p $p --steps 5 --warmup 3 --no-cpu-baseline >> $OUT 2>> gpurun_out/${1:-cfg}_configs.err
done
wc -l $OUT
