#!/bin/bash
# Quick GPU iteration: GPU parity tests, a short bench, optional ncu --set full of K1/K2 on a small mesh.
# usage: bash tools/gpu_quick.sh TAG [ncu]
TAG=${1:-q}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json | cut -c1-400
if [ "$2" == "ncu" ] && grep -q "pytest rc=0" gpurun_out/${TAG}_pytest_gpu.log; then
  timeout 300 python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rhs2_kernel|project_kernel" -s 2 -c 2 \
    -o gpurun_out/${TAG}_prof python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
