#!/bin/bash
# GPU pass of a session: GPU tests, smoke, default bench, ncu --set full of one kernel.
# usage: bash tools/gpu_check.sh TAG [REGEX] [skip-tests]
TAG=${1:-c}; RX=${2:-rhs2_kernel}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
if [ "$3" != "skip-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
  tail -3 gpurun_out/${TAG}_pytest_gpu.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
  tail -1 gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json | head -c 1500
timeout 300 python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 1 -c 1 \
  -o gpurun_out/${TAG}_prof python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?"
