#!/bin/bash
# programmatic dependent launch: GPU tests + bench lines of the small and large configurations
mkdir -p gpurun_out
for c in C1 C2 C4 C5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pdl_bench_$c.json 2> gpurun_out/pdl_bench_$c.err; echo "bench $c rc $?"
done
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/pdl_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pdl_pytest_gpu.log
