#!/bin/bash
# PDL variants on the launch-bound configurations: implicit trigger (this build) vs PDL off (ES_NO_PDL=1)
mkdir -p gpurun_out
for c in C1 C2 C4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pdl2_bench_$c.json 2> /dev/null
  ES_NO_PDL=1 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/nopdl_bench_$c.json 2> /dev/null
done
